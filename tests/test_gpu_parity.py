"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on identical seeded inputs.

Acceptance (BASELINE.json north_star):
  * active-neuron sets bit-exact with the oracle except entries with ||SiLU64| - t| <= 1e-3 t;
  * y relative L2 <= 2e-3 vs the oracle recomputed with the GPU's keep decisions substituted on
    those band entries only (reading R9);
  * calibration threshold bit-exact with the oracle's order statistic (and its counts).
"""
import ctypes
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import cats_synth
import oracle
import paper_2404_08763_b200 as cats

pytestmark = pytest.mark.gpu

BAND = 1e-3
Y_TOL = 2e-3
EL_TOL = 1e-4


def _dev(t):
    return t.to("cuda").contiguous()


def _keep_from_gpu(idx, tm, b, m):
    keep = np.zeros((b, m), np.uint8)
    for tk in range(b):
        keep[tk, idx[((tm >> tk) & 1).astype(bool)]] = 1
    return keep


def _rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def oracle_mlp(ox, og, ou, od, t, mode=oracle.SPARSE, keep_in=None):
    """oracle.mlp token by token on host threads (the C oracle releases the GIL; tokens are
    independent, so the results are the identical serial per-token computations)."""
    b = ox.shape[0]
    if b == 1:
        return oracle.mlp(ox, og, ou, od, t=t, mode=mode, keep_in=keep_in)
    def one(i):
        return oracle.mlp(ox[i:i + 1], og, ou, od, t=t, mode=mode,
                          keep_in=None if keep_in is None else keep_in[i:i + 1])
    with ThreadPoolExecutor(max_workers=min(b, os.cpu_count() or 1)) as ex:
        outs = list(ex.map(one, range(b)))
    return tuple(np.concatenate([o[j] for o in outs]) for j in range(3))


def check_y(yg, y_ref):
    """North-star bound (rel-L2 <= 2e-3 per token) and an element-wise bound |y - y_ref| <= 1e-4 rms(y_ref)
    per token (fp32 accumulation over <= 2 m terms: ~sqrt(n) 2^-24 relative, x1 hi/lo split 2^-16 relative
    per term on the b >= 4 tensor-core path). Returns the worst rel-L2."""
    errs = []
    for i in range(y_ref.shape[0]):
        ref = y_ref[i]
        if not np.abs(ref).any():
            assert not np.abs(yg[i]).any(), f"token {i}: y must be exactly 0"
            errs.append(0.0)
            continue
        errs.append(_rel_l2(yg[i], ref))
        rms = float(np.sqrt(np.mean(ref ** 2)))
        worst = float(np.abs(yg[i] - ref).max())
        assert worst <= EL_TOL * rms, f"token {i}: max |dy| {worst:.3g} > {EL_TOL} rms {rms:.3g}"
    assert max(errs) <= Y_TOL, errs
    return max(errs)


def run_parity(d, m, b, dtype, k, seed=0, heavy=False, num_sms=0, check=True, opts=None, wd_scale=1.0,
               x_scale=1.0, same_tokens=False):
    Wg, Wu, Wd = cats_synth.mlp_weights(d, m, dtype, layer=seed, heavy=heavy)
    if wd_scale != 1.0:  # power of two: exact in bf16 / fp32, scales y exactly (mask unchanged)
        Wd = (Wd.float() * wd_scale).to(dtype)
    x = cats_synth.tokens(b, d, dtype, seed=1 + seed, heavy=heavy)
    if x_scale != 1.0:   # power of two: exact; moves u = x W_gate into SiLU's saturated / linear regions
        x = (x.float() * x_scale).to(dtype)
    if same_tokens:      # b copies of one token: identical per-token masks (union = each token's set)
        x = x[:1].repeat(b, 1).contiguous()
    ox, og, ou, od = (cats_synth.to_oracle(a) for a in (x, Wg, Wu, Wd))
    # threshold: Eq. 3 on the oracle's |SiLU| of these tokens (any t >= 0 is a valid test point)
    zero = np.zeros((m, d), og.dtype)
    _, v64, _ = oracle_mlp(ox, og, zero, zero, 0.0, mode=oracle.DENSE)
    t = float(oracle.calibrate_sort(v64.astype(np.float32), k).t) if k > 0 else 0.0

    plan = cats.MlpPlan(d, m, max_batch=b, dtype=dtype, num_sms=num_sms, **(opts or {}))
    ws = plan.workspace()
    dx, dg, du, dd = (_dev(a) for a in (x, Wg, Wu, Wd))
    y = cats.cats_mlp_decode(plan, dx, dg, du, dd, t, ws=ws)
    torch.cuda.synchronize()
    idx, tm, per = cats.cats_mlp_last_active(plan, ws, b)
    assert (np.diff(idx) > 0).all(), "active list must be strictly ascending"
    assert (tm != 0).all()
    keep_gpu = _keep_from_gpu(idx, tm, b, m)
    assert (keep_gpu.sum(1) == per).all()

    keep64 = (np.abs(v64) >= np.float64(t)).astype(np.uint8)
    band = np.abs(np.abs(v64) - t) <= BAND * t
    mism = (keep_gpu != keep64) & ~band
    assert not mism.any(), f"{int(mism.sum())} active-set mismatches outside the band"
    res = {"t": t, "band": int(band.sum()), "flips_in_band": int(((keep_gpu != keep64) & band).sum()),
           "nnz_union": len(idx), "sparsity": 1 - keep_gpu.mean(), "kernels": cats.cats_mlp_kernels_per_call(plan, b)}
    if check:
        keep_sub = np.where(band, keep_gpu, keep64).astype(np.uint8)
        y_ref, _, _ = oracle_mlp(ox, og, ou, od, t, keep_in=keep_sub)
        res["rel_l2_max"] = check_y(y.cpu().numpy().astype(np.float64), y_ref)
    return res, (plan, ws, dx, dg, du, dd, y)


@pytest.mark.parametrize("d,m,b,dtype,k", [
    (64, 176, 1, torch.float32, 0.5),        # BASELINE config 0 (toy)
    (64, 176, 3, torch.float32, 0.7),
    (264, 1000, 1, torch.bfloat16, 0.5),     # ragged: 33 chunks per row, m not a multiple of anything
    (264, 1000, 2, torch.bfloat16, 0.9),
    (512, 3001, 5, torch.bfloat16, 0.7),
    (1024, 4096, 8, torch.bfloat16, 0.5),
    (8192, 512, 1, torch.bfloat16, 0.5),     # widest supported row (4 chunks per K2 thread)
    (8192, 700, 3, torch.bfloat16, 0.7),     # b >= 2 where the split path does not fit: K12 fallback
    (128, 7, 4, torch.bfloat16, 0.5),        # m < number of SMs
    (8, 1, 1, torch.float32, 0.0),           # a single neuron, one 32-byte row
])
def test_parity_small(d, m, b, dtype, k):
    res, _ = run_parity(d, m, b, dtype, k, seed=d + m + b)
    assert res["rel_l2_max"] <= Y_TOL
    if k > 0:  # the same inputs through the App. D ablation modes (Alg. 2 predicated, Alg. 1 atomic idcs)
        for comp in (cats.CATS_COMPACT_PREDICATED, cats.CATS_COMPACT_ATOMIC):
            run_parity(d, m, b, dtype, k, seed=d + m + b, opts={"compaction": comp})


@pytest.mark.parametrize("model,b,k,heavy", [
    ("mistral-7b", 1, 0.5, False),           # BASELINE config 1 (bench workload)
    ("mistral-7b", 8, 0.5, True),
    ("llama2-7b", 1, 0.7, False),            # config 2
    ("llama2-7b", 4, 0.9, True),
    ("llama2-13b", 1, 0.5, False),           # config 3, unsharded
])
def test_parity_full_size(model, b, k, heavy):
    d, m = cats_synth.MODELS[model]
    res, _ = run_parity(d, m, b, torch.bfloat16, k, seed=7, heavy=heavy)
    assert res["rel_l2_max"] <= Y_TOL
    if b == 1:
        assert abs(res["sparsity"] - k) < 0.01


# Every kernel instantiation the planner selects for the BASELINE shapes: per model,
# b = 1 -> K12 at d = 4096, KA + KB at d = 5120; b = 2 -> KA + KB on CUDA cores (6-row tiles at d = 4096);
# b = 3..8 -> KA + KB on bf16 MMA with x in tensor memory (6-row tiles at d = 4096, 4-row at d = 5120; KB
# MT = 4 at d = 4096, MT = 5 at d = 5120). The batch is a template parameter, so each (model, b) is a
# distinct kernel pair.
@pytest.mark.parametrize("model", ["mistral-7b", "llama2-7b", "llama2-13b"])
@pytest.mark.parametrize("b", [2, 3, 4, 5, 6, 7, 8])
def test_parity_every_planned_batch(model, b):
    d, m = cats_synth.MODELS[model]
    k = {2: 0.5, 3: 0.7, 4: 0.5, 5: 0.9, 6: 0.7, 7: 0.5, 8: 0.5}[b]
    res, _ = run_parity(d, m, b, torch.bfloat16, k, seed=50 + b, heavy=(b % 2 == 1))
    # the split path KA + KB (Llama2-13B d = 5120 from b = 6: KA in column parts, 8-row tiles)
    assert res["kernels"] == 2


@pytest.mark.parametrize("d,m", [(5120, 1003), (5120, 77), (5120, 8), (8192, 512), (4096, 1003), (4096, 77),
                                 (4096, 8)])
@pytest.mark.parametrize("b", [4, 6, 8])
def test_parity_ka_column_parts_ragged(d, m, b):
    """KA in column parts (d = 5120, b >= 6: 8-row tiles, each job streamed as 5 stages of 1024 columns;
    d = 8192: 8 parts, two stages per stream next to 128 KB of x) and KA's 6-row tiles with x in tensor
    memory (d = 4096, b >= 4; two (row, token) pairs per producer lane from b = 6) on ragged and tiny
    layers: a last tile of 1-5 rows, fewer tiles than job streams, one tile."""
    res, _ = run_parity(d, m, b, torch.bfloat16, 0.5, seed=90 + m + b)
    assert res["kernels"] == 2


@pytest.mark.parametrize("model,b", [("mistral-7b", 2), ("llama2-7b", 5), ("llama2-13b", 8)])
def test_parity_fused_path_full_size(model, b):
    """K12 at b >= 2 (options.path = FUSED: the fallback the planner takes where KA / KB do not fit)."""
    d, m = cats_synth.MODELS[model]
    res, _ = run_parity(d, m, b, torch.bfloat16, 0.5, seed=60 + b, opts={"path": cats.CATS_PATH_FUSED})
    assert res["kernels"] == 1


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("b", [1, 8])
def test_parity_llama13b_tp_shard(P, b):
    """BASELINE config 3: the per-GPU shard m / P of Llama2-13B (the decode of one rank, b = 1 and 8)."""
    d, m = cats_synth.MODELS["llama2-13b"]
    res, _ = run_parity(d, m // P, b, torch.bfloat16, 0.5, seed=70 + P)
    # d = 5120: KA + KB from b = 1 (planner); b = 8 with 2-row tiles
    assert res["kernels"] == 2


@pytest.mark.parametrize("comp", ["predicated", "atomic"])
@pytest.mark.parametrize("model,b,k", [("mistral-7b", 1, 0.5), ("llama2-7b", 1, 0.9), ("llama2-7b", 4, 0.7)])
def test_parity_app_d_ablation_modes(comp, model, b, k):
    """App. D Alg. 2 (mask-predicated row loads, no compaction) and Alg. 1 (atomic appends to a global idcs
    list, then a list kernel) compute the same CATS y as the default ballot compaction."""
    d, m = cats_synth.MODELS[model]
    c = cats.CATS_COMPACT_PREDICATED if comp == "predicated" else cats.CATS_COMPACT_ATOMIC
    res, (plan, ws, dx, dg, du, dd, y) = run_parity(d, m, b, torch.bfloat16, k, seed=80, opts={"compaction": c})
    assert res["kernels"] == (2 if comp == "atomic" else 1)
    y2 = cats.cats_mlp_decode(plan, dx, dg, du, dd, res["t"], ws=ws)
    if comp == "predicated":
        assert torch.equal(y, y2)  # deterministic (fixed tiles, exact fixed-point split-K)
    else:
        # Alg. 1's idcs order is the order of the atomic appends: the neurons grouped into one fp32
        # sub-sum change from run to run, so y is reproducible only to fp32 rounding (reading R15)
        assert float((y - y2).norm() / y.norm()) < 1e-6


@pytest.mark.parametrize("opts", [{"lazy_tail": 0}, {"lazy_tail": 64}, {"max_stages": 2}, {"eager": 1},
                                  {"min_tiles": 16}, {"l2_prefetch": 4}, {"rows_per_tile": 2},
                                  {"rows_per_tile": 4, "eager": 1, "lazy_tail": 1000}])
@pytest.mark.parametrize("model,b,k", [("mistral-7b", 1, 0.5), ("llama2-7b", 3, 0.7)])
def test_parity_k12_schedule_knobs(opts, model, b, k):
    """K12 under the schedule knobs (tile reservation off / everywhere, shallow ring, eager fill, few CTAs,
    L2 prefetch of static tiles, other tile heights) against the oracle, bit-reproducible: the dynamic
    schedule changes which CTA takes which tile, never y."""
    d, m = cats_synth.MODELS[model]
    res, (plan, ws, dx, dg, du, dd, y) = run_parity(d, m, b, torch.bfloat16, k, seed=85,
                                                    opts={"path": cats.CATS_PATH_FUSED, **opts})
    assert res["kernels"] == 1
    assert torch.equal(y, cats.cats_mlp_decode(plan, dx, dg, du, dd, res["t"], ws=ws))
    res_small, _ = run_parity(264, 1000, b, torch.bfloat16, k, seed=86, opts={"path": cats.CATS_PATH_FUSED, **opts})


@pytest.mark.parametrize("b", [1, 2, 8])
@pytest.mark.parametrize("case", ["saturated", "tiny", "same_tokens"])
def test_parity_extreme_inputs(case, b):
    """x scaled by 2^6 (|u| up to ~10: SiLU's saturated branches, exp(-u) overflowing to inf for very
    negative u), by 2^-6 (u ~ 5e-3: SiLU's linear region near 0, t tiny), and b identical tokens."""
    kw = {"saturated": {"x_scale": 64.0}, "tiny": {"x_scale": 1 / 64}, "same_tokens": {"same_tokens": True}}[case]
    res, _ = run_parity(1024, 3000, b, torch.bfloat16, 0.7, seed=95, **kw)
    if case == "same_tokens" and b > 1:
        assert abs(res["nnz_union"] / 3000 - (1 - res["sparsity"])) < 1e-9  # union = every token's set


@pytest.mark.parametrize("b", [1, 4])
@pytest.mark.parametrize("e", [-16, -8, 8, 16])
def test_parity_output_magnitude_sweep(b, e):
    """W_down scaled by 2^e scales y by 2^e exactly (mask unchanged): exercises the K12 fixed-point
    accumulator (resolution 2^-38, R10) at b = 1 and the fp32 split path at b = 4."""
    res, _ = run_parity(1024, 4096, b, torch.bfloat16, 0.5, seed=90, wd_scale=2.0 ** e)
    assert res["rel_l2_max"] <= Y_TOL


def test_t0_and_dense_path():
    d, m, b = 512, 2000, 3
    res, (plan, ws, dx, dg, du, dd, y) = run_parity(d, m, b, torch.bfloat16, 0.0, seed=3)
    assert res["nnz_union"] == m
    y_dense = cats.cats_mlp_dense(plan, dx, dg, du, dd, ws=ws)
    y0 = cats.cats_mlp_decode(plan, dx, dg, du, dd, 0.0, ws=ws)
    assert torch.equal(y_dense, y0)
    # dense vs oracle Eq. 1
    ox, og, ou, od = (cats_synth.to_oracle(a.cpu()) for a in (dx, dg, du, dd))
    y_ref, _, _ = oracle.mlp(ox, og, ou, od, t=0.0, mode=oracle.DENSE)
    assert _rel_l2(y_dense.cpu().numpy().astype(np.float64), y_ref) < 1e-5


def test_threshold_above_every_activation_gives_zero():
    d, m = 256, 600
    Wg, Wu, Wd = (_dev(a) for a in cats_synth.mlp_weights(d, m, torch.bfloat16))
    x = _dev(cats_synth.tokens(2, d, torch.bfloat16))
    plan = cats.MlpPlan(d, m, max_batch=2)
    ws = plan.workspace()
    y = cats.cats_mlp_decode(plan, x, Wg, Wu, Wd, 1e30, ws=ws)
    idx, tm, per = cats.cats_mlp_last_active(plan, ws, 2)
    assert len(idx) == 0 and not per.any()
    assert not y.any()


def test_deterministic_bitwise():
    d, m = 4096, 14336
    Wg, Wu, Wd = (_dev(a) for a in cats_synth.mlp_weights(d, m, torch.bfloat16))
    plan = cats.MlpPlan(d, m, max_batch=8)
    ws = plan.workspace()
    for b in (1, 8):
        x = _dev(cats_synth.tokens(b, d, torch.bfloat16, seed=11))
        ys = [cats.cats_mlp_decode(plan, x, Wg, Wu, Wd, 0.0994, ws=ws).clone() for _ in range(10)]
        assert all(torch.equal(ys[0], yi) for yi in ys[1:])


def test_gate_act_matches_oracle_silu():
    d, m, b = 4096, 11008, 4
    Wg, Wu, Wd = cats_synth.mlp_weights(d, m, torch.bfloat16)
    x = cats_synth.tokens(b, d, torch.bfloat16, seed=5)
    plan = cats.MlpPlan(d, m, max_batch=b)
    acts = cats.cats_mlp_gate_act(plan, _dev(x), _dev(Wg)).cpu().numpy()
    ox, og = cats_synth.to_oracle(x), cats_synth.to_oracle(Wg)
    z = np.zeros((m, d), np.uint16)
    _, v64, _ = oracle.mlp(ox, og, z, z, t=0.0, mode=oracle.DENSE)
    err = np.abs(acts - v64)
    assert err.max() < 1e-5 * np.abs(v64).max() + 1e-7


def test_decode_host_equals_device_path():
    d, m, b = 4096, 14336, 2
    Wg, Wu, Wd = (_dev(a) for a in cats_synth.mlp_weights(d, m, torch.bfloat16))
    x = cats_synth.tokens(b, d, torch.bfloat16, seed=9)
    plan = cats.MlpPlan(d, m, max_batch=b)
    ws = plan.workspace()
    y_dev = cats.cats_mlp_decode(plan, _dev(x), Wg, Wu, Wd, 0.1, ws=ws).cpu()
    y_host = cats.cats_mlp_decode_host(plan, x.pin_memory(), Wg, Wu, Wd, 0.1, ws=ws)  # kernel writes host y
    assert torch.equal(y_dev, y_host)
    y_pageable = torch.empty((b, d), dtype=torch.float32)                         # device-to-host copy path
    cats.cats_mlp_decode_host(plan, x, Wg, Wu, Wd, 0.1, y_host=y_pageable, ws=ws)
    assert torch.equal(y_dev, y_pageable)
    x1 = x[:1].clone()                                                            # b = 1 (K12), pinned
    y1 = cats.cats_mlp_decode_host(plan, x1.pin_memory(), Wg, Wu, Wd, 0.1, ws=ws)
    assert torch.equal(cats.cats_mlp_decode(plan, _dev(x1), Wg, Wu, Wd, 0.1, ws=ws).cpu(), y1)
    for bb in (b, 1):  # bound call (graph replay of x staging + KA/KB or K12): x re-read on every call
        xp = x[:bb].clone().pin_memory()
        call = cats.BoundDecodeHost(plan, xp, Wg, Wu, Wd, 0.1, ws=ws)
        assert call._call is not None
        for seed in (10, 11, 12):
            x2 = cats_synth.tokens(bb, d, torch.bfloat16, seed=seed)
            xp.copy_(x2)
            assert torch.equal(call().clone(), cats.cats_mlp_decode(plan, _dev(x2), Wg, Wu, Wd, 0.1, ws=ws).cpu())
    h = ctypes.c_void_p()                                                         # pageable buffers: not bindable
    rc = plan._lib.cats_mlp_host_call_create(plan.handle, x.data_ptr(), b, Wg.data_ptr(), Wu.data_ptr(), Wd.data_ptr(),
                                             0.1, y_pageable.data_ptr(), ws.data_ptr(), ws.numel(), None, ctypes.byref(h))
    assert plan._lib.cats_status_string(rc).decode() == "CATS_E_UNSUPPORTED" and h.value is None


def test_tensor_parallel_emulated_on_one_gpu():
    """TP along m: P shard plans with the same layer-global t; the sum of the
    partial y equals the unsharded oracle (the all-reduce is a plain sum)."""
    d, m, b, P = 5120, 13824, 1, 4
    Wg, Wu, Wd = cats_synth.mlp_weights(d, m, torch.bfloat16)
    x = cats_synth.tokens(b, d, torch.bfloat16, seed=13)
    ox, og, ou, od = (cats_synth.to_oracle(a) for a in (x, Wg, Wu, Wd))
    _, v64, _ = oracle.mlp(ox, og, ou, od, t=0.0, mode=oracle.DENSE)
    t = float(oracle.calibrate_sort(v64.astype(np.float32), 0.5).t)
    ysum = torch.zeros(b, d, dtype=torch.float64)
    keep_gpu = np.zeros((b, m), np.uint8)
    ms = m // P
    for r in range(P):
        sl = slice(r * ms, (r + 1) * ms)
        plan = cats.MlpPlan(d, ms, max_batch=b)
        ws = plan.workspace()
        y = cats.cats_mlp_decode(plan, _dev(x), _dev(Wg[sl]), _dev(Wu[sl]), _dev(Wd[sl]), t, ws=ws)
        idx, tm, _ = cats.cats_mlp_last_active(plan, ws, b)
        keep_gpu[:, sl] = _keep_from_gpu(idx, tm, b, ms)
        ysum += y.cpu().double()
    keep64 = (np.abs(v64) >= t).astype(np.uint8)
    band = np.abs(np.abs(v64) - t) <= BAND * t
    assert not ((keep_gpu != keep64) & ~band).any()
    y_ref, _, _ = oracle.mlp(ox, og, ou, od, t=t, keep_in=np.where(band, keep_gpu, keep64).astype(np.uint8))
    assert _rel_l2(ysum.numpy(), y_ref) <= Y_TOL


# ------------------------------------------------------------------------------------ calibration

def _oracle_t(acts_cpu, k):
    a = cats_synth.to_oracle(acts_cpu)
    if a.dtype == np.uint16 and a.size > 2_000_000:
        return oracle.calibrate_bf16_counts(oracle.bf16_counts(a), k)
    return oracle.calibrate_sort(a, k)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("n,heavy", [(1, False), (13, False), (45056, False), (1_000_003, True),
                                     (40_000_001, False)])
def test_calibration_bit_exact(dtype, n, heavy):
    acts = cats_synth.calib_acts(n, dtype, seed=n % 101, heavy=heavy, device="cuda")
    acts_cpu = acts.cpu()
    for k in [0.0, 0.5, 0.7, 0.9, 0.99]:
        t, info = cats.cats_calibrate_threshold(acts, k)
        ref = _oracle_t(acts_cpu, k)
        assert t == ref.t, (k, t, ref.t)
        assert (info["count_lt"], info["count_le"], info["rank_r"]) == (ref.count_lt, ref.count_le, ref.r)
        if dtype == torch.bfloat16 and n > 1000:
            assert info["passes"] <= 2


def test_calibration_adversarial_and_errors():
    dev = "cuda"
    # all equal; signed zeros + subnormals; sorted input (worst case for sampling)
    cases = [torch.full((3_000_000,), 0.7, dtype=torch.bfloat16, device=dev),
             torch.tensor([0.0, -0.0, 1e-40, -1e-39, 1.0] * 2_000_000, dtype=torch.float32, device=dev),
             torch.sort(cats_synth.calib_acts(30_000_000, torch.bfloat16, seed=2, device=dev).abs())[0]]
    for acts in cases:
        for k in [0.0, 0.3, 0.5, 0.999]:
            t, info = cats.cats_calibrate_threshold(acts, k)
            ref = _oracle_t(acts.cpu(), k)
            assert (t, info["count_lt"], info["count_le"]) == (ref.t, ref.count_lt, ref.count_le)
    bad = cats_synth.calib_acts(100_000, torch.bfloat16, device=dev)
    bad[77_777] = float("inf")
    with pytest.raises(cats.CatsError) as e:
        cats.cats_calibrate_threshold(bad, 0.5)
    assert e.value.name == "CATS_E_NONFINITE"
    with pytest.raises(cats.CatsError) as e:
        cats.cats_calibrate_threshold(bad[1:], 0.5)  # misaligned view
    assert e.value.name == "CATS_E_ALIGN"


def test_calibration_achieved_sparsity_on_gpu_activations():
    """Calibrate on GPU-collected |SiLU(x W_gate)| of 256 tokens, then the fraction of zeroed
    entries on the calibration set obeys count_lt < kN <= count_le and held-out tokens reach ~k."""
    d, m = 4096, 11008
    Wg, Wu, Wd = (_dev(a) for a in cats_synth.mlp_weights(d, m, torch.bfloat16))
    plan = cats.MlpPlan(d, m, max_batch=8)
    ws = plan.workspace()
    acts = torch.cat([cats.cats_mlp_gate_act(plan, _dev(cats_synth.tokens(8, d, torch.bfloat16, seed=100 + i)), Wg,
                                             ws=ws) for i in range(32)])
    for k in [0.5, 0.7, 0.9]:
        t, info = cats.cats_calibrate_threshold(acts, k)
        n = acts.numel()
        assert info["count_lt"] < k * n <= info["count_le"]
        assert int((acts.abs() < t).sum()) == info["count_lt"]
        x = _dev(cats_synth.tokens(8, d, torch.bfloat16, seed=999))
        cats.cats_mlp_decode(plan, x, Wg, Wu, Wd, t, ws=ws)
        _, _, per = cats.cats_mlp_last_active(plan, ws, 8)
        assert abs((1 - per / m).mean() - k) < 0.02


@pytest.mark.slow
def test_calibration_full_size_config4():
    """BASELINE config 4: 500 samples x 2048 tokens x 11008 channels of bf16 (22.5 GB) on the GPU;
    oracle = exact multiset order statistic over the identical bytes (streamed to host)."""
    n = 500 * 2048 * 11008
    free, _ = torch.cuda.mem_get_info()
    if free < n * 2 + (4 << 30):
        pytest.skip("not enough device memory")
    acts = cats_synth.calib_acts(n, torch.bfloat16, seed=0, device="cuda")
    counts = np.zeros(65536, np.uint64)
    chunk = 1 << 30
    for s in range(0, n, chunk):
        oracle.bf16_counts(cats_synth.bf16_bits(acts[s:s + chunk].cpu()), counts)
    for k in [0.5, 0.7, 0.9]:
        t, info = cats.cats_calibrate_threshold(acts, k)
        ref = oracle.calibrate_bf16_counts(counts, k)
        assert (t, info["count_lt"], info["count_le"]) == (ref.t, ref.count_lt, ref.count_le)
        assert info["passes"] <= 2
    del acts
    torch.cuda.empty_cache()


@pytest.mark.parametrize("d,m,b,k", [(4096, 11008, 2, 0.5), (4096, 11008, 8, 0.9), (5120, 3456, 5, 0.7),
                                     (264, 1000, 3, 0.5)])
def test_split_path_matches_fused_path(d, m, b, k):
    """b >= 2 runs the split path (KA gate+up, KB down); forcing K12 on the same inputs must give the
    same y within the parity tolerance (the two differ only in fp32 summation order)."""
    Wg, Wu, Wd = (_dev(a) for a in cats_synth.mlp_weights(d, m, torch.bfloat16, layer=b))
    x = _dev(cats_synth.tokens(b, d, torch.bfloat16, seed=21))
    plan_s = cats.MlpPlan(d, m, max_batch=b)
    plan_f = cats.MlpPlan(d, m, max_batch=b, path=cats.CATS_PATH_FUSED)
    t = 0.1 if k < 0.9 else 0.3
    ys = cats.cats_mlp_decode(plan_s, x, Wg, Wu, Wd, t, ws=plan_s.workspace())
    yf = cats.cats_mlp_decode(plan_f, x, Wg, Wu, Wd, t, ws=plan_f.workspace())
    err = (ys.double() - yf.double()).norm() / yf.double().norm().clamp_min(1e-30)
    assert float(err) <= Y_TOL


def test_mixed_batches_share_one_workspace():
    """K12 (b = 1) and the split path (b >= 2) re-arm their counters, accumulators and tile masks for
    each other: alternating batch sizes on one workspace gives the same bits as fresh workspaces."""
    d, m = 4096, 11008
    Wg, Wu, Wd = (_dev(a) for a in cats_synth.mlp_weights(d, m, torch.bfloat16, layer=3))
    plan = cats.MlpPlan(d, m, max_batch=8)
    ws = plan.workspace()
    for i, b in enumerate([1, 8, 2, 1, 5, 4, 1, 3]):
        x = _dev(cats_synth.tokens(b, d, torch.bfloat16, seed=40 + i))
        y_shared = cats.cats_mlp_decode(plan, x, Wg, Wu, Wd, 0.12, ws=ws).clone()
        y_fresh = cats.cats_mlp_decode(plan, x, Wg, Wu, Wd, 0.12, ws=plan.workspace())
        assert torch.equal(y_shared, y_fresh), b
        y_dense = cats.cats_mlp_dense(plan, x, Wg, Wu, Wd, ws=ws)
        assert torch.isfinite(y_dense).all()


@pytest.mark.parametrize("opts", [{"path": cats.CATS_PATH_FUSED}, {"compaction": cats.CATS_COMPACT_ATOMIC}])
def test_k12_alternating_accumulators_across_batches_and_gate_calls(opts):
    """K12's two int64 accumulators alternate per call, and each call zeroes the rows the previous one
    left in the other (a batch-dependent extent): K12 at changing batch sizes, with gate-only
    (calibration collection) launches in between, gives the same bits as fresh workspaces."""
    d, m = 2048, 3000
    Wg, Wu, Wd = (_dev(a) for a in cats_synth.mlp_weights(d, m, torch.bfloat16, layer=5))
    plan = cats.MlpPlan(d, m, max_batch=8, **opts)
    ws = plan.workspace()
    for i, b in enumerate([3, 1, 8, 2, 1, 1, 6]):
        x = _dev(cats_synth.tokens(b, d, torch.bfloat16, seed=70 + i))
        assert cats.cats_mlp_kernels_per_call(plan, b) == (2 if "compaction" in opts else 1)
        y_shared = cats.cats_mlp_decode(plan, x, Wg, Wu, Wd, 0.1, ws=ws).clone()
        y_fresh = cats.cats_mlp_decode(plan, x, Wg, Wu, Wd, 0.1, ws=plan.workspace())
        if "compaction" in opts:  # Alg. 1: append order varies run to run (reading R15)
            assert float((y_shared - y_fresh).norm() / y_fresh.norm()) < 1e-6, b
        else:
            assert torch.equal(y_shared, y_fresh), b
        if i % 2 == 0:
            cats.cats_mlp_gate_act(plan, x, Wg, ws=ws)
