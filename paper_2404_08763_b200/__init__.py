"""paper_2404_08763_b200 -- B200-native CATS (arXiv 2404.08763) decode MLP + threshold calibration.

Thin Python binding over the C ABI in include/cats.h (libcats.so, hand-written CUDA for
sm_100a). Functions keep the C names; they only marshal arguments (torch tensors -> device
pointers, current CUDA stream, workspace allocation). Every step of the method runs in the
library's kernels; there is no CPU or PyTorch fallback.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import (CATS_BF16, CATS_COMPACT_ATOMIC, CATS_COMPACT_BALLOT, CATS_COMPACT_PREDICATED, CATS_F32,
                   CATS_PATH_AUTO, CATS_PATH_FUSED, CATS_PATH_SPLIT, CalibInfo, CalibWindow, PlanInfo, PlanOptions)

__all__ = [
    "CatsError", "MlpPlan", "cats_calib_rank", "cats_calibrate_workspace_bytes", "cats_calibrate_threshold",
    "cats_calib_window_init", "cats_calib_hist", "cats_calib_step", "cats_mlp_decode", "cats_mlp_dense",
    "cats_mlp_decode_profiled",
    "cats_mlp_decode_host", "cats_mlp_gate_act", "cats_mlp_last_active", "cats_mlp_kernels_per_call", "library_path",
    "XsparsePlan", "cats_xsparse_gemv", "BoundDecodeHost", "plan_options", "CATS_PATH_AUTO", "CATS_PATH_FUSED", "CATS_PATH_SPLIT", "CATS_COMPACT_BALLOT",
    "CATS_COMPACT_PREDICATED", "CATS_COMPACT_ATOMIC",
]


class CatsError(RuntimeError):
    def __init__(self, code: int, where: str):
        lib = _lib.load()
        name = lib.cats_status_string(code).decode()
        msg = f"{where}: {name}"
        if name == "CATS_E_CUDA":
            msg += f" ({lib.cats_last_cuda_error().decode()})"
        super().__init__(msg)
        self.code = code
        self.name = name


def _check(rc: int, where: str):
    if rc != 0:
        raise CatsError(rc, where)


def library_path() -> str:
    _lib.load()
    return _lib.LIB_PATH


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return CATS_BF16
    if t.dtype == torch.float32:
        return CATS_F32
    raise TypeError(f"unsupported dtype {t.dtype} (bf16 or fp32)")


def _dev_ptr(t: torch.Tensor, name: str) -> int:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.data_ptr()


def _stream(stream, device) -> int:
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _stream_obj(stream, device):
    """The torch stream a call runs on (allocations for it are made under this stream)."""
    if stream is None:
        return torch.cuda.current_stream(device)
    if isinstance(stream, torch.cuda.Stream):
        return stream
    return torch.cuda.ExternalStream(int(stream), device=device)


def plan_options(**kw) -> PlanOptions:
    """cats_mlp_plan_options_t with the library defaults, fields overridden by keyword
    (path, compaction, trace, rows_per_tile, max_stages, lazy_tail, min_tiles, eager, l2_prefetch,
    xs_cols, xs_ranges, xs_mma, xs_no_shrink)."""
    o = PlanOptions()
    _check(_lib.load().cats_mlp_plan_options_init(ctypes.byref(o)), "cats_mlp_plan_options_init")
    names = {f for f, _ in PlanOptions._fields_} - {"size"}
    for k, v in kw.items():
        if k not in names:
            raise TypeError(f"unknown plan option {k!r}")
        setattr(o, k, int(v))
    return o


# ------------------------------------------------------------------------------- calibration
def cats_calib_rank(k: float, n: int) -> int:
    r = ctypes.c_uint64()
    _check(_lib.load().cats_calib_rank(float(k), int(n), ctypes.byref(r)), "cats_calib_rank")
    return r.value


def cats_calibrate_workspace_bytes(n: int, dtype: torch.dtype = torch.bfloat16) -> int:
    b = ctypes.c_size_t()
    dt = CATS_BF16 if dtype == torch.bfloat16 else CATS_F32
    _check(_lib.load().cats_calibrate_workspace_bytes(int(n), dt, ctypes.byref(b)), "cats_calibrate_workspace_bytes")
    return b.value


def cats_calibrate_threshold(acts: torch.Tensor, k: float, ws: torch.Tensor | None = None, stream=None):
    """Eq. 3 threshold of one MLP block from its activations (device tensor, any shape).

    Returns (t: float, info: dict(n, rank_r, count_lt, count_le, t_bits, passes))."""
    n = acts.numel()
    if ws is None:
        ws = torch.empty(cats_calibrate_workspace_bytes(n, acts.dtype), dtype=torch.uint8, device=acts.device)
    t = ctypes.c_float()
    info = CalibInfo()
    rc = _lib.load().cats_calibrate_threshold(_dev_ptr(acts, "acts") if n else None, n, _dt(acts), float(k),
                                              _dev_ptr(ws, "ws"), ws.numel(), _stream(stream, acts.device),
                                              ctypes.byref(t), ctypes.byref(info))
    _check(rc, "cats_calibrate_threshold")
    return t.value, {f: getattr(info, f) for f, _ in CalibInfo._fields_}


def cats_calib_window_init(n: int, dtype: torch.dtype) -> CalibWindow:
    w = CalibWindow()
    dt = CATS_BF16 if dtype == torch.bfloat16 else CATS_F32
    _check(_lib.load().cats_calib_window_init(int(n), dt, ctypes.byref(w)), "cats_calib_window_init")
    return w


def cats_calib_hist(acts: torch.Tensor, window: CalibWindow, hist_dev: torch.Tensor, counts_dev: torch.Tensor,
                    stream=None):
    """hist_dev (uint64/int64 [>= nbins]) and counts_dev ([CATS_CALIB_COUNTS_LEN = 8]: 4 counts + pass
    scratch) are accumulated into (+=)."""
    if counts_dev.numel() < 8 or hist_dev.numel() < window.nbins:
        raise ValueError("counts_dev needs 8 entries (CATS_CALIB_COUNTS_LEN), hist_dev window.nbins")
    rc = _lib.load().cats_calib_hist(_dev_ptr(acts, "acts"), acts.numel(), _dt(acts), ctypes.byref(window),
                                     _dev_ptr(hist_dev, "hist"), _dev_ptr(counts_dev, "counts"),
                                     _stream(stream, acts.device))
    _check(rc, "cats_calib_hist")


def cats_calib_step(hist_host: np.ndarray, counts_host: np.ndarray, n: int, dtype: torch.dtype, k: float,
                    window: CalibWindow):
    """Returns (done, t_bits, count_lt, count_le); updates `window` in place when not done."""
    hist_host = np.ascontiguousarray(hist_host, dtype=np.uint64)
    counts_host = np.ascontiguousarray(counts_host, dtype=np.uint64)
    done, tb = ctypes.c_int(), ctypes.c_uint32()
    lt, le = ctypes.c_uint64(), ctypes.c_uint64()
    dt = CATS_BF16 if dtype == torch.bfloat16 else CATS_F32
    rc = _lib.load().cats_calib_step(hist_host.ctypes.data, counts_host.ctypes.data, int(n), dt, float(k),
                                     ctypes.byref(window), ctypes.byref(done), ctypes.byref(tb), ctypes.byref(lt),
                                     ctypes.byref(le))
    _check(rc, "cats_calib_step")
    return bool(done.value), tb.value, lt.value, le.value


# ------------------------------------------------------------------------------- decode
class MlpPlan:
    """Host-only plan for one MLP shape (d, m) -- see cats_mlp_plan_create."""

    _create = "cats_mlp_plan_create"

    def __init__(self, d: int, m: int, max_batch: int = 1, dtype: torch.dtype = torch.bfloat16, device: int = 0,
                 num_sms: int = 0, **options):
        """options: cats_mlp_plan_options_t fields (see plan_options); none = the library defaults."""
        self._lib = _lib.load()
        self._h = ctypes.c_void_p()
        self.dtype = dtype
        dt = CATS_BF16 if dtype == torch.bfloat16 else CATS_F32
        args = (int(m), int(d)) if self._create == "cats_xsparse_plan_create" else (int(d), int(m))
        self.options = plan_options(**options)
        fn = self._create + "_ex"
        _check(getattr(self._lib, fn)(*args, int(max_batch), dt, int(device), int(num_sms),
                                      ctypes.byref(self.options), ctypes.byref(self._h)), fn)
        info = PlanInfo()
        _check(self._lib.cats_mlp_plan_info(self._h, ctypes.byref(info)), "cats_mlp_plan_info")
        self.info = {f: getattr(info, f) for f, _ in PlanInfo._fields_}
        self.d, self.m, self.max_batch, self.device = d, m, max_batch, device

    @property
    def handle(self):
        return self._h

    @property
    def workspace_bytes(self) -> int:
        return self.info["workspace_bytes"]

    def workspace(self, stream=None) -> torch.Tensor:
        """Allocate (on `stream`) and initialise (cats_mlp_workspace_init, on `stream`) a decode workspace."""
        st = _stream_obj(stream, torch.device(f"cuda:{self.device}"))
        with torch.cuda.stream(st):
            ws = torch.empty(self.workspace_bytes, dtype=torch.uint8, device=f"cuda:{self.device}")
        rc = self._lib.cats_mlp_workspace_init(self.handle, ws.data_ptr(), ws.numel(), st.cuda_stream)
        _check(rc, "cats_mlp_workspace_init")
        return ws

    def __del__(self, _void_p=ctypes.c_void_p):  # bound early: module globals may be gone at exit
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.cats_mlp_plan_destroy(h)
            self._h = _void_p()


class XsparsePlan(MlpPlan):
    """Host-only plan for one App. B input-sparse projection d_in -> d_out (cats_xsparse_plan_create).
    plan.d = d_out (the output width), plan.m = d_in (the thresholded inputs)."""

    _create = "cats_xsparse_plan_create"

    def __init__(self, d_in: int, d_out: int, max_batch: int = 1, dtype: torch.dtype = torch.bfloat16,
                 device: int = 0, num_sms: int = 0, **options):
        super().__init__(d_out, d_in, max_batch, dtype, device, num_sms, **options)
        self.d_in, self.d_out = d_in, d_out


def _check_tensor(t: torch.Tensor, name: str, shape, dtype, device):
    # cheap checks first (this runs on every call: ~1 us per tensor matters for the e2e path)
    if t.shape != shape:
        raise ValueError(f"{name}: shape {tuple(t.shape)} != {tuple(shape)}")
    if t.dtype is not dtype:
        raise TypeError(f"{name}: dtype {t.dtype} != {dtype}")
    if device.type == "cpu":
        if t.is_cuda:
            raise ValueError(f"{name}: on {t.device}, expected cpu")
    elif not t.is_cuda or t.get_device() != device.index:
        raise ValueError(f"{name}: on {t.device}, expected {device}")


def _prep(plan: MlpPlan, x: torch.Tensor, y, ws, stream, weights=(), wshape=None):
    """Validate shapes / dtypes / devices against the plan (the C ABI carries no sizes), and allocate
    y / the workspace on the stream the call runs on (so the caching allocator and the workspace
    initialisation are ordered with the launch)."""
    if x.dim() == 1:
        x = x.unsqueeze(0)
    b = x.shape[0]
    dev = torch.device(f"cuda:{plan.device}")
    if isinstance(plan, XsparsePlan) != (wshape is not None and len(weights) == 1):
        raise CatsError(12, "plan kind does not match the call")  # CATS_E_UNSUPPORTED, as the C ABI
    _check_tensor(x, "x", (b, plan.m if isinstance(plan, XsparsePlan) else plan.d), plan.dtype, dev)
    for name, w in weights:
        _check_tensor(w, name, wshape, plan.dtype, dev)
    st = _stream_obj(stream, dev)
    with torch.cuda.stream(st):
        if y is None:
            y = torch.empty((b, plan.d), dtype=torch.float32, device=dev)
        if ws is None:
            ws = plan.workspace(stream=st)
    _check_tensor(y, "y", (b, plan.d), torch.float32, dev)
    if ws.dtype != torch.uint8 or ws.numel() < plan.workspace_bytes:
        raise ValueError(f"workspace must be uint8 with >= {plan.workspace_bytes} bytes")
    return x, b, y, ws, st


def _mlp_w(W_gate, W_up, W_down_nm):
    return [("W_gate", W_gate), ("W_up", W_up), ("W_down_nm", W_down_nm)]


def cats_mlp_decode(plan: MlpPlan, x, W_gate, W_up, W_down_nm, t: float, y=None, ws=None, stream=None):
    """y[b][d] (fp32) = CATS_t gated MLP of x[b][d]; weights neuron-major [m][d]."""
    x, b, y, ws, st = _prep(plan, x, y, ws, stream, _mlp_w(W_gate, W_up, W_down_nm), (plan.m, plan.d))
    rc = plan._lib.cats_mlp_decode(plan.handle, _dev_ptr(x, "x"), b, _dev_ptr(W_gate, "W_gate"),
                                   _dev_ptr(W_up, "W_up"), _dev_ptr(W_down_nm, "W_down_nm"), float(t),
                                   _dev_ptr(y, "y"), _dev_ptr(ws, "ws"), ws.numel(), st.cuda_stream)
    _check(rc, "cats_mlp_decode")
    return y


def cats_xsparse_gemv(plan: XsparsePlan, x, W_in_major, t: float, y=None, ws=None, stream=None):
    """y[b][d_out] (fp32) = CATS_t(x) W for x[b][d_in]; W input-major [d_in][d_out] (App. B)."""
    x, b, y, ws, st = _prep(plan, x, y, ws, stream, [("W_in_major", W_in_major)], (plan.m, plan.d))
    rc = plan._lib.cats_xsparse_gemv(plan.handle, _dev_ptr(x, "x"), b, _dev_ptr(W_in_major, "W_in_major"), float(t),
                                     _dev_ptr(y, "y"), _dev_ptr(ws, "ws"), ws.numel(), st.cuda_stream)
    _check(rc, "cats_xsparse_gemv")
    return y


def cats_mlp_decode_profiled(plan: MlpPlan, x, W_gate, W_up, W_down_nm, t: float, events, y=None, ws=None,
                             stream=None):
    """cats_mlp_decode with 3 torch.cuda.Event(enable_timing=True) recorded around K12 and K3."""
    x, b, y, ws, st = _prep(plan, x, y, ws, stream, _mlp_w(W_gate, W_up, W_down_nm), (plan.m, plan.d))
    for e in events:
        if e.cuda_event == 0:
            e.record(st)  # materialise the lazily created event on this device
    arr = (ctypes.c_void_p * 3)(*[e.cuda_event for e in events])
    rc = plan._lib.cats_mlp_decode_profiled(plan.handle, _dev_ptr(x, "x"), b, _dev_ptr(W_gate, "W_gate"),
                                            _dev_ptr(W_up, "W_up"), _dev_ptr(W_down_nm, "W_down_nm"), float(t),
                                            _dev_ptr(y, "y"), _dev_ptr(ws, "ws"), ws.numel(), st.cuda_stream, arr)
    _check(rc, "cats_mlp_decode_profiled")
    return y


def cats_mlp_dense(plan: MlpPlan, x, W_gate, W_up, W_down_nm, y=None, ws=None, stream=None):
    x, b, y, ws, st = _prep(plan, x, y, ws, stream, _mlp_w(W_gate, W_up, W_down_nm), (plan.m, plan.d))
    rc = plan._lib.cats_mlp_dense(plan.handle, _dev_ptr(x, "x"), b, _dev_ptr(W_gate, "W_gate"),
                                  _dev_ptr(W_up, "W_up"), _dev_ptr(W_down_nm, "W_down_nm"), _dev_ptr(y, "y"),
                                  _dev_ptr(ws, "ws"), ws.numel(), st.cuda_stream)
    _check(rc, "cats_mlp_dense")
    return y


def cats_mlp_decode_host(plan: MlpPlan, x_host: torch.Tensor, W_gate, W_up, W_down_nm, t: float, y_host=None,
                         ws=None, stream=None):
    """Host x in (pinned recommended), host y out; blocks on the stream."""
    if x_host.dim() == 1:
        x_host = x_host.unsqueeze(0)
    if x_host.is_cuda or not x_host.is_contiguous():
        raise ValueError("x_host must be a contiguous host tensor")
    b = x_host.shape[0]
    if isinstance(plan, XsparsePlan):
        raise CatsError(12, "cats_mlp_decode_host")
    cpu = torch.device("cpu")
    _check_tensor(x_host, "x_host", (b, plan.d), plan.dtype, cpu)
    dev = torch.device(f"cuda:{plan.device}")
    for name, w in _mlp_w(W_gate, W_up, W_down_nm):
        _check_tensor(w, name, (plan.m, plan.d), plan.dtype, dev)
    st = _stream_obj(stream, dev)
    if y_host is None:
        y_host = torch.empty((b, plan.d), dtype=torch.float32, pin_memory=x_host.is_pinned())
    _check_tensor(y_host, "y_host", (b, plan.d), torch.float32, cpu)
    if not y_host.is_contiguous():
        raise ValueError("y_host must be contiguous")
    if ws is None:
        with torch.cuda.stream(st):
            ws = plan.workspace(stream=st)
    rc = plan._lib.cats_mlp_decode_host(plan.handle, x_host.data_ptr(), b, _dev_ptr(W_gate, "W_gate"),
                                        _dev_ptr(W_up, "W_up"), _dev_ptr(W_down_nm, "W_down_nm"), float(t),
                                        y_host.data_ptr(), _dev_ptr(ws, "ws"), ws.numel(), st.cuda_stream)
    _check(rc, "cats_mlp_decode_host")
    return y_host


class BoundDecodeHost:
    """cats_mlp_decode_host with its arguments validated and marshalled once (a serving loop's per-token
    call): every call copies the CURRENT contents of x_host to the device, decodes and delivers y into
    y_host, blocking on the stream. With pinned x_host and y_host the call is the library's bound host call
    (cats_mlp_host_call_*: one CUDA graph replay per call); otherwise cats_mlp_decode_host per call."""

    def __init__(self, plan: MlpPlan, x_host, W_gate, W_up, W_down_nm, t: float, y_host=None, ws=None, stream=None):
        # one validated call through the regular path (allocates y_host / ws if needed)
        self.y_host = cats_mlp_decode_host(plan, x_host, W_gate, W_up, W_down_nm, t, y_host=y_host, ws=ws,
                                           stream=stream)
        x2 = x_host if x_host.dim() == 2 else x_host.unsqueeze(0)
        ws = ws if ws is not None else plan.workspace(stream=stream)
        st = _stream_obj(stream, torch.device(f"cuda:{plan.device}"))
        self._keep = (plan, x_host, W_gate, W_up, W_down_nm, ws, st)  # lifetimes
        self._lib = plan._lib
        args = (plan.handle, x2.data_ptr(), x2.shape[0], W_gate.data_ptr(), W_up.data_ptr(), W_down_nm.data_ptr(),
                float(t), self.y_host.data_ptr(), ws.data_ptr(), ws.numel(), st.cuda_stream)
        self._call = None
        if x_host.is_pinned() and self.y_host.is_pinned():
            h = ctypes.c_void_p()
            _check(self._lib.cats_mlp_host_call_create(*args, ctypes.byref(h)), "cats_mlp_host_call_create")
            self._call = h
            self._fn, self._args = self._lib.cats_mlp_host_call_run, (h,)
        else:
            self._fn, self._args = self._lib.cats_mlp_decode_host, args

    def __call__(self) -> torch.Tensor:
        _check(self._fn(*self._args), "cats_mlp_host_call_run" if self._call is not None else "cats_mlp_decode_host")
        return self.y_host

    def __del__(self):
        if getattr(self, "_call", None) is not None:
            self._lib.cats_mlp_host_call_destroy(self._call)
            self._call = None


def cats_mlp_gate_act(plan: MlpPlan, x, W_gate, acts=None, ws=None, stream=None):
    """acts[b][m] = SiLU(x W_gate) (fp32) -- calibration data collection."""
    if x.dim() == 1:
        x = x.unsqueeze(0)
    b = x.shape[0]
    dev = torch.device(f"cuda:{plan.device}")
    if isinstance(plan, XsparsePlan):
        raise CatsError(12, "cats_mlp_gate_act")
    _check_tensor(x, "x", (b, plan.d), plan.dtype, dev)
    _check_tensor(W_gate, "W_gate", (plan.m, plan.d), plan.dtype, dev)
    st = _stream_obj(stream, dev)
    with torch.cuda.stream(st):
        if acts is None:
            acts = torch.empty((b, plan.m), dtype=torch.float32, device=dev)
        if ws is None:
            ws = plan.workspace(stream=st)
    _check_tensor(acts, "acts", (b, plan.m), torch.float32, dev)
    rc = plan._lib.cats_mlp_gate_act(plan.handle, _dev_ptr(x, "x"), b, _dev_ptr(W_gate, "W_gate"),
                                     _dev_ptr(acts, "acts"), _dev_ptr(ws, "ws"), ws.numel(), st.cuda_stream)
    _check(rc, "cats_mlp_gate_act")
    return acts


def cats_mlp_kernels_per_call(plan: MlpPlan, b: int) -> int:
    """1 = the fused kernel K12, 2 = the split path KA + KB (b >= 2), for a decode of batch b."""
    n = ctypes.c_int()
    _check(plan._lib.cats_mlp_kernels_per_call(plan.handle, int(b), ctypes.byref(n)), "cats_mlp_kernels_per_call")
    return n.value


def cats_mlp_last_active(plan: MlpPlan, ws: torch.Tensor, b: int, stream=None):
    """(idx int32[nnz] ascending, tokmask uint8[nnz], nnz_per_token uint32[b]) of the last decode."""
    idx = np.zeros(plan.m, np.int32)
    tm = np.zeros(plan.m, np.uint8)
    nnz = ctypes.c_uint32()
    per = np.zeros(b, np.uint32)
    rc = plan._lib.cats_mlp_last_active(plan.handle, _dev_ptr(ws, "ws"), int(b), idx.ctypes.data, tm.ctypes.data,
                                        ctypes.byref(nnz), per.ctypes.data, _stream(stream, ws.device))
    _check(rc, "cats_mlp_last_active")
    return idx[: nnz.value].copy(), tm[: nnz.value].copy(), per
