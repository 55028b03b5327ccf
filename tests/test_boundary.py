"""C-ABI boundary tests that need no GPU: the library loads, exports every symbol include/cats.h
declares, validates arguments before touching CUDA, plans shapes, and its host-side calibration
logic (rank rule, window steering, refinement) converges to the oracle's order statistic when the
device histogram pass is emulated with numpy."""
import ctypes
import math
import os
import re
from fractions import Fraction

import numpy as np
import pytest
import torch

import cats_synth
import oracle
import paper_2404_08763_b200 as cats
from paper_2404_08763_b200 import _lib
from tests.conftest import ROOT

lib = _lib.load()
FAKE = 0x10000  # 16-byte aligned non-null "device" pointer; validation never dereferences it


def header_functions():
    src = open(os.path.join(ROOT, "include", "cats.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cats_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    names = header_functions()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.exported_symbols())
    assert lib.cats_version() == 1


def test_status_strings():
    for code, name in enumerate(_lib.STATUS):
        assert lib.cats_status_string(code).decode() == name
    assert lib.cats_status_string(99).decode() == "CATS_E_UNKNOWN"


def test_rank_rule_exact():
    for k in [0.0, 0.1, 0.25, 0.5, 0.7, 0.9, 0.99, 1e-300, 5e-324, 0.9999999999999999]:
        for n in [0, 1, 2, 3, 10, 1000, 2**31 + 7, 11272192000, 2**63 + 5]:
            assert cats.cats_calib_rank(k, n) == math.ceil(Fraction(k) * n), (k, n)
            assert cats.cats_calib_rank(k, n) == oracle.rank(k, n)
    for bad in [1.0, 1.5, -0.1, float("nan")]:
        with pytest.raises(cats.CatsError) as e:
            cats.cats_calib_rank(bad, 10)
        assert e.value.name == "CATS_E_SPARSITY"


def test_plan_without_gpu():
    p = cats.MlpPlan(4096, 14336, max_batch=1, dtype=torch.bfloat16, num_sms=148)
    i = p.info
    assert i["grid"] == 2 * 148 and i["stages"] >= 2 and i["rows_per_tile"] == 6
    assert 2 * (i["smem"] + 1024) <= 228 * 1024      # two K12 CTAs per SM
    assert i["workspace_bytes"] >= 4096 * 8          # int64 y accumulator
    toy = cats.MlpPlan(64, 176, max_batch=1, dtype=torch.float32, num_sms=148)
    assert toy.info["grid"] == 176 // 4 // 2         # small layers: >= 2 tiles per CTA
    small = cats.MlpPlan(64, 5, max_batch=8, dtype=torch.float32, num_sms=148)
    assert small.info["grid"] == 1                  # 2 tiles (m = 5): one CTA
    p13 = cats.MlpPlan(5120, 13824, max_batch=8, num_sms=148)   # Llama2-13B: KA + KB at every batch size
    assert [cats.cats_mlp_kernels_per_call(p13, b) for b in range(1, 9)] == [2] * 8
    for b in range(1, 9):                            # every batch size fits the shared-memory budget
        i = cats.MlpPlan(5120, 13824, max_batch=b, num_sms=148).info
        per_sm = 2 if b == 1 else 1
        assert i["grid"] == 148 * per_sm and per_sm * (i["smem"] + 1024) <= 228 * 1024
    assert cats.MlpPlan(8192, 1000, max_batch=8, num_sms=148).info["stages"] >= 3


@pytest.mark.parametrize("args,err", [
    ((0, 100, 1, torch.bfloat16), "CATS_E_SHAPE"),
    ((64, 0, 1, torch.bfloat16), "CATS_E_SHAPE"),
    ((4100, 100, 1, torch.bfloat16), "CATS_E_ALIGN"),
    ((66, 100, 1, torch.float32), "CATS_E_ALIGN"),
    ((64, 100, 0, torch.bfloat16), "CATS_E_BATCH"),
    ((64, 100, 9, torch.bfloat16), "CATS_E_BATCH"),
    ((65536, 100, 1, torch.bfloat16), "CATS_E_UNSUPPORTED"),
])
def test_plan_errors(args, err):
    with pytest.raises(cats.CatsError) as e:
        cats.MlpPlan(*args, num_sms=148)
    assert e.value.name == err


def _decode_rc(plan, x=FAKE, b=1, wg=FAKE, wu=FAKE, wd=FAKE, t=0.1, y=FAKE, ws=FAKE, wsb=None):
    wsb = plan.workspace_bytes if wsb is None else wsb
    return lib.cats_status_string(lib.cats_mlp_decode(plan.handle, x, b, wg, wu, wd, t, y, ws, wsb, None)).decode()


def test_decode_validation_precedes_cuda():
    p = cats.MlpPlan(256, 512, max_batch=4, dtype=torch.bfloat16, num_sms=148)
    assert _decode_rc(p, x=None) == "CATS_E_NULL"
    assert _decode_rc(p, wd=None) == "CATS_E_NULL"
    assert _decode_rc(p, y=None) == "CATS_E_NULL"
    assert _decode_rc(p, b=0) == "CATS_E_BATCH"
    assert _decode_rc(p, b=5) == "CATS_E_BATCH"
    assert _decode_rc(p, wsb=p.workspace_bytes - 1) == "CATS_E_WORKSPACE"
    assert _decode_rc(p, ws=None) == "CATS_E_WORKSPACE"
    assert _decode_rc(p, x=FAKE + 8) == "CATS_E_ALIGN"
    assert _decode_rc(p, wu=FAKE + 2) == "CATS_E_ALIGN"
    assert _decode_rc(p, t=-0.5) == "CATS_E_THRESHOLD"
    assert _decode_rc(p, t=float("nan")) == "CATS_E_THRESHOLD"
    assert _decode_rc(p, t=float("inf")) == "CATS_E_THRESHOLD"
    if not torch.cuda.is_available():
        # valid arguments reach CUDA, which reports the missing device as a status, not a crash
        assert _decode_rc(p) == "CATS_E_CUDA"
        assert lib.cats_last_cuda_error().decode() != ""
    rc = lib.cats_mlp_dense(p.handle, FAKE, 9, FAKE, FAKE, FAKE, FAKE, FAKE, p.workspace_bytes, None)
    assert lib.cats_status_string(rc).decode() == "CATS_E_BATCH"
    rc = lib.cats_mlp_gate_act(p.handle, None, 1, FAKE, FAKE, FAKE, p.workspace_bytes, None)
    assert lib.cats_status_string(rc).decode() == "CATS_E_NULL"


def test_calibrate_validation():
    t = ctypes.c_float(-1.0)
    wsb = cats.cats_calibrate_workspace_bytes(100, torch.bfloat16)
    assert wsb >= 32768 * 8

    def rc(acts=FAKE, n=100, dt=1, k=0.5, ws=FAKE, wsb=wsb, tout=ctypes.byref(t)):
        return lib.cats_status_string(lib.cats_calibrate_threshold(acts, n, dt, k, ws, wsb, None, tout, None)).decode()

    assert rc(acts=None) == "CATS_E_NULL"
    assert rc(tout=None) == "CATS_E_NULL"
    assert rc(dt=7) == "CATS_E_DTYPE"
    assert rc(k=1.0) == "CATS_E_SPARSITY"
    assert rc(k=-0.1) == "CATS_E_SPARSITY"
    assert rc(k=float("nan")) == "CATS_E_SPARSITY"
    assert rc(n=0) == "CATS_E_EMPTY"
    assert rc(acts=FAKE + 4) == "CATS_E_ALIGN"
    assert rc(wsb=wsb - 1) == "CATS_E_WORKSPACE"
    assert t.value == -1.0  # untouched on error


# ---------------------------------------------------------------- host calibration logic (numpy pass)

def _keys(acts: np.ndarray):
    if acts.dtype == np.uint16:
        return (acts.astype(np.uint32) & 0x7FFF), 0x7F80, 8
    return (acts.view(np.uint32) & 0x7FFFFFFF), 0x7F800000, 4


def emulated_pass(acts: np.ndarray, w):
    """numpy stand-in for the device pass cats_calib_hist (same contract as include/cats.h)."""
    keys, inf, per = _keys(acts)
    if w.sample_stride:
        nvec = acts.size // per
        vsel = np.arange(0, nvec, w.sample_stride)
        keys = keys[: nvec * per].reshape(nvec, per)[vsel].reshape(-1)
    fin = keys < inf
    kf = keys[fin]
    below = int((kf < w.lo).sum())
    above = int((kf > w.hi).sum())
    inw = kf[(kf >= w.lo) & (kf <= w.hi)]
    hist = np.bincount(((inw - w.lo) >> w.shift).astype(np.int64), minlength=w.nbins).astype(np.uint64)
    counts = np.array([below, inw.size, above, int((~fin).sum())], np.uint64)
    return hist, counts


def emulated_calibrate(acts: np.ndarray, k: float):
    dtype = torch.bfloat16 if acts.dtype == np.uint16 else torch.float32
    w = cats.cats_calib_window_init(acts.size, dtype)
    passes = 0
    for _ in range(32):
        hist, counts = emulated_pass(acts, w)
        if not w.sample_stride:
            passes += 1
        done, tb, lt, le = cats.cats_calib_step(hist, counts, acts.size, dtype, k, w)
        if done:
            bits = np.uint32(tb << 16) if dtype == torch.bfloat16 else np.uint32(tb)
            return float(np.array([bits], np.uint32).view(np.float32)[0]), lt, le, passes
    raise AssertionError("no convergence")


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("n", [1, 7, 1000, 50_000, 20_000_000])
def test_host_select_matches_oracle(dtype, n):
    if n > 1_000_000 and dtype == torch.float32:
        n = 9_000_000
    acts_t = cats_synth.calib_acts(n, dtype, seed=n % 97, heavy=(n % 2 == 0))
    acts = cats_synth.to_oracle(acts_t)
    ks = [0.0, 0.5, 0.9] if n > 1_000_000 else [0.0, 0.1, 0.5, 0.7, 0.9, 0.99]
    for k in ks:
        t, lt, le, passes = emulated_calibrate(acts, k)
        if dtype == torch.bfloat16 and n > 1_000_000:
            ref = oracle.calibrate_bf16_counts(oracle.bf16_counts(acts), k)
        else:
            ref = oracle.calibrate_sort(acts, k)
        assert (t, lt, le) == (ref.t, ref.count_lt, ref.count_le), (k, t, ref)
        if dtype == torch.bfloat16:
            assert passes <= 2


def test_host_select_adversarial():
    # all equal, sorted, ties across the window, signed zeros, tiny subnormals
    cases = [np.full(100_000, 0x3E00, np.uint16),
             np.sort(cats_synth.bf16_bits(cats_synth.calib_acts(30_000_000, torch.bfloat16, seed=3))),
             np.repeat(np.array([0x0000, 0x8000, 0x0001, 0x3F80], np.uint16), 5_000_000)]
    for acts in cases:
        for k in [0.0, 0.2, 0.5, 0.75, 0.999]:
            t, lt, le, _ = emulated_calibrate(acts, k)
            ref = oracle.calibrate_bf16_counts(oracle.bf16_counts(acts), k)
            assert (t, lt, le) == (ref.t, ref.count_lt, ref.count_le)


def test_host_select_nonfinite():
    acts = cats_synth.bf16_bits(cats_synth.calib_acts(5000, torch.bfloat16, seed=1)).copy()
    acts[1234] = 0x7FC0  # NaN
    with pytest.raises(cats.CatsError) as e:
        emulated_calibrate(acts, 0.5)
    assert e.value.name == "CATS_E_NONFINITE"


def test_kernels_per_call_path_choice():
    """b = 1 runs the fused K12 (one kernel); b >= 2 the split path KA + KB where it fits shared memory."""
    p = cats.MlpPlan(4096, 11008, max_batch=8, dtype=torch.bfloat16, num_sms=148)
    assert cats.cats_mlp_kernels_per_call(p, 1) == 1
    assert [cats.cats_mlp_kernels_per_call(p, b) for b in range(2, 9)] == [2] * 7
    toy = cats.MlpPlan(64, 176, max_batch=3, dtype=torch.float32, num_sms=148)
    assert cats.cats_mlp_kernels_per_call(toy, 3) == 2
    wide = cats.MlpPlan(8192, 512, max_batch=8, dtype=torch.bfloat16, num_sms=148)
    # x takes 128 KB of KA's shared memory: full-row stages no longer fit, 8 x 1024-column parts do
    assert cats.cats_mlp_kernels_per_call(wide, 8) == 2
    with pytest.raises(cats.CatsError) as e:
        cats.cats_mlp_kernels_per_call(p, 9)
    assert e.value.name == "CATS_E_BATCH"


def _xs_rc(plan, x=FAKE, b=1, W=FAKE, t=0.1, y=FAKE, ws=FAKE, wsb=None):
    wsb = plan.workspace_bytes if wsb is None else wsb
    return lib.cats_status_string(lib.cats_xsparse_gemv(plan.handle, x, b, W, t, y, ws, wsb, None)).decode()


def test_xsparse_plan_and_validation_without_gpu():
    """App. B plan (d_in -> d_out): host-only planning, argument checks before any CUDA call, and the
    two plan kinds rejected by each other's entry points."""
    p = cats.XsparsePlan(4096, 6144, max_batch=8, dtype=torch.bfloat16, num_sms=148)
    assert (p.d, p.m, p.d_in, p.d_out) == (6144, 4096, 4096, 6144)
    assert [cats.cats_mlp_kernels_per_call(p, b) for b in range(1, 9)] == [1] * 8  # kernel XS
    for shape in [(4096, 12288), (5120, 5120), (1001, 264), (64, 64), (8192, 8192)]:
        cats.XsparsePlan(*shape, max_batch=8, dtype=torch.bfloat16, num_sms=148)
    with pytest.raises(cats.CatsError) as e:
        cats.XsparsePlan(4096, 100, max_batch=1, num_sms=148)  # 200-byte rows: not 16-byte aligned
    assert e.value.name == "CATS_E_ALIGN"
    assert _xs_rc(p, x=None) == "CATS_E_NULL"
    assert _xs_rc(p, W=None) == "CATS_E_NULL"
    assert _xs_rc(p, b=0) == "CATS_E_BATCH"
    assert _xs_rc(p, b=9) == "CATS_E_BATCH"
    assert _xs_rc(p, wsb=p.workspace_bytes - 1) == "CATS_E_WORKSPACE"
    assert _xs_rc(p, W=FAKE + 4) == "CATS_E_ALIGN"
    assert _xs_rc(p, t=-1.0) == "CATS_E_THRESHOLD"
    assert _xs_rc(p, t=float("nan")) == "CATS_E_THRESHOLD"
    mp = cats.MlpPlan(4096, 14336, max_batch=1, dtype=torch.bfloat16, num_sms=148)
    assert _xs_rc(mp) == "CATS_E_UNSUPPORTED"
    assert _decode_rc(p) == "CATS_E_UNSUPPORTED"
    rc = lib.cats_mlp_decode_host(p.handle, FAKE, 1, FAKE, FAKE, FAKE, 0.1, FAKE, FAKE, p.workspace_bytes, None)
    assert lib.cats_status_string(rc).decode() == "CATS_E_UNSUPPORTED"
    rc = lib.cats_mlp_gate_act(p.handle, FAKE, 1, FAKE, FAKE, FAKE, p.workspace_bytes, None)
    assert lib.cats_status_string(rc).decode() == "CATS_E_UNSUPPORTED"
    rc = lib.cats_mlp_dense(p.handle, FAKE, 1, FAKE, FAKE, FAKE, FAKE, FAKE, p.workspace_bytes, None)
    assert lib.cats_status_string(rc).decode() == "CATS_E_UNSUPPORTED"
    if not torch.cuda.is_available():
        assert _xs_rc(p) == "CATS_E_CUDA"


def test_plan_options():
    """cats_mlp_plan_options_t: defaults, explicit kernel-path / App. D ablation selection, validation
    (the library reads no environment variables)."""
    o = cats.plan_options()
    assert (o.size, o.path, o.compaction, o.lazy_tail, o.min_tiles, o.xs_mma) == (
        ctypes.sizeof(_lib.PlanOptions), 0, 0, 8, 2, 1)
    auto = cats.MlpPlan(4096, 11008, max_batch=8, num_sms=148)
    assert [cats.cats_mlp_kernels_per_call(auto, b) for b in range(1, 9)] == [1] + [2] * 7
    fused = cats.MlpPlan(4096, 11008, max_batch=8, num_sms=148, path=cats.CATS_PATH_FUSED)
    assert [cats.cats_mlp_kernels_per_call(fused, b) for b in range(1, 9)] == [1] * 8
    pred = cats.MlpPlan(4096, 11008, max_batch=8, num_sms=148, compaction=cats.CATS_COMPACT_PREDICATED)
    assert [cats.cats_mlp_kernels_per_call(pred, b) for b in range(1, 9)] == [1] * 8
    atom = cats.MlpPlan(4096, 11008, max_batch=8, num_sms=148, compaction=cats.CATS_COMPACT_ATOMIC)
    assert [cats.cats_mlp_kernels_per_call(atom, b) for b in range(1, 9)] == [2] * 8  # gate + list kernel
    assert atom.workspace_bytes >= fused.workspace_bytes + 11008 * 4 * 9  # the global idcs list (ids + v)
    assert cats.MlpPlan(5120, 13824, num_sms=148, rows_per_tile=2).info["rows_per_tile"] == 2
    split1 = cats.MlpPlan(5120, 1728, max_batch=8, num_sms=148, path=cats.CATS_PATH_SPLIT)
    assert cats.cats_mlp_kernels_per_call(split1, 1) == 2  # KA + KB at b = 1 (small TP shards)
    # KB's last-64 reduction needs more than 64 SMs: smaller devices take K12 at every batch size
    small = cats.MlpPlan(4096, 11008, max_batch=8, num_sms=64)
    assert [cats.cats_mlp_kernels_per_call(small, b) for b in range(1, 9)] == [1] * 8
    for bad, err in [({"path": 7}, "CATS_E_UNSUPPORTED"), ({"compaction": 3}, "CATS_E_UNSUPPORTED"),
                     ({"rows_per_tile": 3}, "CATS_E_SHAPE"), ({"min_tiles": 0}, "CATS_E_SHAPE"),
                     ({"max_stages": 1}, "CATS_E_SHAPE"), ({"lazy_tail": -1}, "CATS_E_SHAPE")]:
        with pytest.raises(cats.CatsError) as e:
            cats.MlpPlan(4096, 11008, num_sms=148, **bad)
        assert e.value.name == err, bad
    o = cats.plan_options()
    o.size = 4
    h = ctypes.c_void_p()
    rc = lib.cats_mlp_plan_create_ex(64, 64, 1, 1, 0, 148, ctypes.byref(o), ctypes.byref(h))
    assert lib.cats_status_string(rc).decode() == "CATS_E_SHAPE"
    with pytest.raises(TypeError):
        cats.plan_options(no_such_field=1)
    src = open(os.path.join(ROOT, "paper_2404_08763_b200", "csrc", "api.cu")).read()
    assert "getenv" not in src


def test_binding_checks_shapes_before_the_abi():
    """The C ABI carries no sizes: the binding checks every tensor against the plan."""
    p = cats.MlpPlan(256, 512, max_batch=4, dtype=torch.bfloat16, num_sms=148)
    x = torch.zeros(2, 256, dtype=torch.bfloat16)
    w = torch.zeros(512, 256, dtype=torch.bfloat16)
    with pytest.raises(ValueError):   # host tensors are rejected before any call
        cats.cats_mlp_decode(p, x, w, w, w, 0.1, ws=torch.zeros(8, dtype=torch.uint8))
    with pytest.raises(ValueError):
        cats.cats_mlp_decode_host(p, torch.zeros(2, 255, dtype=torch.bfloat16), w, w, w, 0.1)
    with pytest.raises(TypeError):
        cats.cats_mlp_decode_host(p, torch.zeros(2, 256, dtype=torch.float32), w, w, w, 0.1)


def test_tp_comm_validation_without_gpu():
    """The fused TP reduction's host side (cats_tp_*): buffer sizing and argument checks, no device needed."""
    nb = ctypes.c_size_t()
    assert lib.cats_tp_buffer_bytes(4, 5120, ctypes.byref(nb)) == 0
    assert nb.value >= 2 * 4 * 5120 * 4
    for w, n in [(0, 5120), (9, 5120), (4, 0), (4, 5122)]:
        assert lib.cats_status_string(lib.cats_tp_buffer_bytes(w, n, ctypes.byref(nb))).decode() == "CATS_E_SHAPE"
    ptrs = (ctypes.c_void_p * 2)(FAKE, FAKE + 4096)
    h = ctypes.c_void_p()
    assert lib.cats_tp_comm_create(1, 2, 5120, ptrs, 0, ctypes.byref(h)) == 0
    lib.cats_tp_comm_destroy(h)
    assert lib.cats_status_string(lib.cats_tp_comm_create(2, 2, 5120, ptrs, 0, ctypes.byref(h))).decode() == "CATS_E_SHAPE"
    pb = ctypes.c_void_p()
    assert lib.cats_status_string(lib.cats_tp_buffer_alloc(0, 0, ctypes.byref(pb))).decode() == "CATS_E_SHAPE"
    assert lib.cats_status_string(lib.cats_tp_buffer_alloc(64, 0, None)).decode() == "CATS_E_NULL"
    if not torch.cuda.is_available():
        assert lib.cats_status_string(lib.cats_tp_buffer_alloc(1024, 0, ctypes.byref(pb))).decode() == "CATS_E_CUDA"
    bad = (ctypes.c_void_p * 2)(FAKE, FAKE + 4)
    assert lib.cats_status_string(lib.cats_tp_comm_create(0, 2, 5120, bad, 0, ctypes.byref(h))).decode() == "CATS_E_ALIGN"


def test_host_call_validation_before_cuda():
    """cats_mlp_host_call_create validates like cats_mlp_decode_host before touching the device."""
    p = cats.MlpPlan(4096, 14336, max_batch=2, dtype=torch.bfloat16, num_sms=148)
    h = ctypes.c_void_p()

    def rc(*args):
        return lib.cats_status_string(lib.cats_mlp_host_call_create(*args)).decode()

    wsb = p.workspace_bytes
    assert rc(p.handle, FAKE, 1, FAKE, FAKE, FAKE, 0.1, FAKE, FAKE, wsb, None, None) == "CATS_E_NULL"
    assert rc(None, FAKE, 1, FAKE, FAKE, FAKE, 0.1, FAKE, FAKE, wsb, None, ctypes.byref(h)) == "CATS_E_NULL"
    assert rc(p.handle, None, 1, FAKE, FAKE, FAKE, 0.1, FAKE, FAKE, wsb, None, ctypes.byref(h)) == "CATS_E_NULL"
    assert rc(p.handle, FAKE, 3, FAKE, FAKE, FAKE, 0.1, FAKE, FAKE, wsb, None, ctypes.byref(h)) == "CATS_E_BATCH"
    assert rc(p.handle, FAKE, 1, FAKE, FAKE, FAKE, 0.1, FAKE, FAKE, wsb - 1, None, ctypes.byref(h)) == "CATS_E_WORKSPACE"
    assert rc(p.handle, FAKE, 1, FAKE, FAKE, FAKE, -1.0, FAKE, FAKE, wsb, None, ctypes.byref(h)) == "CATS_E_THRESHOLD"
    assert h.value is None
    assert lib.cats_status_string(lib.cats_mlp_host_call_run(None)).decode() == "CATS_E_NULL"
    lib.cats_mlp_host_call_destroy(None)  # no-op
