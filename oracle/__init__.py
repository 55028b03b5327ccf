"""CPU oracle for the CATS hot path (arXiv 2404.08763) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package. It shares no code with the CUDA library in
``paper_2404_08763_b200/`` and never imports it; the product path never imports this.

The arithmetic lives in plain C (``cats_oracle.c``, fp64, ``-ffp-contract=off``) plus the
pure-Python brute force in ``brute.py``. This module only compiles/loads the C library and
marshals numpy arrays. Inputs are numpy ``float32`` arrays (dtype 0) or ``uint16`` arrays
holding bfloat16 bit patterns (dtype 1). Weights are neuron-major ``[m][d]``.

Parity status: every function here is pinned by ``tests/test_oracle_pins.py``
except the paper's real-model statistics (App. C sparsities, "70% <-> t~0.15" on RefinedWeb,
P:236), which are "parity unpinned" because they need the paper's weights and data.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cats_oracle.c")
_LIB_PATH = os.path.join(_HERE, "libcats_oracle.so")
_OMP_PATH = os.path.join(_HERE, "libcats_oracle_omp.so")  # timing build (all cores), same source
_lock = threading.Lock()
_lib = None
_omp = None

F32 = 0
BF16 = 1
SPARSE, MASKED, DENSE = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, fp64, no FMA contraction, no fast-math): the serial
    checker, and the same source with -fopenmp as the all-core timing build."""
    for path, extra in ((_LIB_PATH, []), (_OMP_PATH, ["-fopenmp"])):
        if force or not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(_SRC):
            tmp = path + f".tmp{os.getpid()}"
            subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=gnu11", "-fPIC", "-shared",
                            *extra, _SRC, "-o", tmp, "-lm"], check=True)
            os.replace(tmp, path)
    return _LIB_PATH


def _load(omp: bool = False):
    global _lib, _omp
    with _lock:
        if (_omp if omp else _lib) is None:
            build()
            lib = ctypes.CDLL(_OMP_PATH if omp else _LIB_PATH)
            P = ctypes.c_void_p
            lib.oracle_silu.restype = ctypes.c_double
            lib.oracle_silu.argtypes = [ctypes.c_double]
            lib.oracle_cats_mask.restype = None
            lib.oracle_cats_mask.argtypes = [P, ctypes.c_int64, ctypes.c_double, P]
            lib.oracle_mlp.restype = ctypes.c_int
            lib.oracle_mlp.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                       P, P, P, P, ctypes.c_double, ctypes.c_int, P, P, P, P]
            lib.oracle_xsparse_gemv.restype = ctypes.c_int
            lib.oracle_xsparse_gemv.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, P, P,
                                                ctypes.c_double, P, P]
            lib.oracle_rank.restype = ctypes.c_uint64
            lib.oracle_rank.argtypes = [ctypes.c_double, ctypes.c_uint64]
            lib.oracle_calibrate_sort.restype = ctypes.c_int
            lib.oracle_calibrate_sort.argtypes = [P, ctypes.c_uint64, ctypes.c_int, ctypes.c_double,
                                                  P, P, P, P]
            lib.oracle_bf16_count.restype = None
            lib.oracle_bf16_count.argtypes = [P, ctypes.c_uint64, P]
            lib.oracle_calibrate_bf16_counts.restype = ctypes.c_int
            lib.oracle_calibrate_bf16_counts.argtypes = [P, ctypes.c_double, P, P, P, P, P]
            if omp:
                _omp = lib
            else:
                _lib = lib
    return _omp if omp else _lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def _dtype_code(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return F32
    if a.dtype == np.uint16:
        return BF16
    raise TypeError(f"oracle inputs must be float32 or uint16 (bf16 bits), got {a.dtype}")


def silu(u: float) -> float:
    """Eq. 2, stable two-branch form."""
    return _load().oracle_silu(float(u))


def cats_mask(v: np.ndarray, t: float) -> np.ndarray:
    """Eq. 4: keep iff |v| >= t."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    keep = np.zeros(v.shape[-1], dtype=np.uint8)
    _load().oracle_cats_mask(_ptr(v), v.shape[-1], float(t), _ptr(keep))
    return keep


def mlp(x: np.ndarray, Wg: np.ndarray, Wu: np.ndarray, Wd: np.ndarray, t: float, mode: int = SPARSE,
        keep_in: np.ndarray | None = None, all_cores: bool = False):
    """CATS gated MLP per token (Eq. 1 + Eq. 5, Alg. "MLP using CATS" P:289-298).
    all_cores=True runs the OpenMP build of the same source (timing only; identical results).

    x: [b][d]; Wg, Wu, Wd: neuron-major [m][d]; all float32 or all uint16 (bf16 bits).
    Returns (y [b][d] float64, v [b][m] float64, keep [b][m] uint8).
    """
    x = np.ascontiguousarray(x)
    if x.ndim == 1:
        x = x[None, :]
    Wg, Wu, Wd = (np.ascontiguousarray(w) for w in (Wg, Wu, Wd))
    dt = _dtype_code(x)
    for w in (Wg, Wu, Wd):
        if _dtype_code(w) != dt:
            raise TypeError("x and weights must share a dtype")
    b, d = x.shape
    m = Wg.shape[0]
    assert Wg.shape == (m, d) and Wu.shape == (m, d) and Wd.shape == (m, d)
    y = np.zeros((b, d), dtype=np.float64)
    v = np.zeros((b, m), dtype=np.float64)
    keep = np.zeros((b, m), dtype=np.uint8)
    kp = 0
    if keep_in is not None:
        keep_in = np.ascontiguousarray(keep_in, dtype=np.uint8).reshape(b, m)
        kp = _ptr(keep_in)
    rc = _load(all_cores).oracle_mlp(d, m, b, dt, _ptr(x), _ptr(Wg), _ptr(Wu), _ptr(Wd), float(t), int(mode),
                                     kp, _ptr(y), _ptr(v), _ptr(keep))
    if rc != 0:
        raise ValueError(f"oracle_mlp failed ({rc})")
    return y, v, keep


def xsparse_gemv(x: np.ndarray, W: np.ndarray, t: float):
    """App. B attention-input CATS: y = CATS_t(x) W per token (Eq. 4 on x itself).

    x: [b][d_in]; W: input-major [d_in][d_out]; both float32 or both uint16 (bf16 bits).
    Returns (y [b][d_out] float64, keep [b][d_in] uint8).
    """
    x = np.ascontiguousarray(x)
    if x.ndim == 1:
        x = x[None, :]
    W = np.ascontiguousarray(W)
    dt = _dtype_code(x)
    if _dtype_code(W) != dt:
        raise TypeError("x and W must share a dtype")
    b, d_in = x.shape
    assert W.shape[0] == d_in
    d_out = W.shape[1]
    y = np.zeros((b, d_out), dtype=np.float64)
    keep = np.zeros((b, d_in), dtype=np.uint8)
    rc = _load().oracle_xsparse_gemv(d_in, d_out, b, dt, _ptr(x), _ptr(W), float(t), _ptr(y), _ptr(keep))
    if rc != 0:
        raise ValueError(f"oracle_xsparse_gemv failed ({rc})")
    return y, keep


def rank(k: float, n: int) -> int:
    """r = ceil(k*N) exactly on the binary value of k (Eq. 3, reading G5)."""
    return int(_load().oracle_rank(float(k), int(n)))


class CalibResult(tuple):
    __slots__ = ()
    _fields = ("t", "r", "count_lt", "count_le", "n")

    def __new__(cls, t, r, lt, le, n):
        return super().__new__(cls, (t, r, lt, le, n))

    t = property(lambda s: s[0])
    r = property(lambda s: s[1])
    count_lt = property(lambda s: s[2])
    count_le = property(lambda s: s[3])
    n = property(lambda s: s[4])


def calibrate_sort(acts: np.ndarray, k: float) -> CalibResult:
    """Eq. 3 by full sort of |acts| (float32 or bf16 bits). Raises on NaN/Inf."""
    acts = np.ascontiguousarray(acts).reshape(-1)
    t = ctypes.c_double()
    r, lt, le = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    rc = _load().oracle_calibrate_sort(_ptr(acts), acts.size, _dtype_code(acts), float(k),
                                       ctypes.addressof(t), ctypes.addressof(r), ctypes.addressof(lt),
                                       ctypes.addressof(le))
    if rc == -2:
        raise FloatingPointError("non-finite activation")
    if rc != 0:
        raise ValueError(f"oracle_calibrate_sort failed ({rc})")
    return CalibResult(t.value, r.value, lt.value, le.value, acts.size)


def bf16_counts(acts_u16: np.ndarray, counts: np.ndarray | None = None) -> np.ndarray:
    """Accumulate multiplicities of the 2^16 bf16 bit patterns (call on consecutive chunks)."""
    acts_u16 = np.ascontiguousarray(acts_u16, dtype=np.uint16).reshape(-1)
    if counts is None:
        counts = np.zeros(65536, dtype=np.uint64)
    _load().oracle_bf16_count(_ptr(acts_u16), acts_u16.size, _ptr(counts))
    return counts


def calibrate_bf16_counts(counts: np.ndarray, k: float) -> CalibResult:
    """Eq. 3 from bf16 pattern multiplicities (same answer as sorting the multiset)."""
    counts = np.ascontiguousarray(counts, dtype=np.uint64)
    t = ctypes.c_double()
    r, lt, le, n = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    rc = _load().oracle_calibrate_bf16_counts(_ptr(counts), float(k), ctypes.addressof(t), ctypes.addressof(r),
                                              ctypes.addressof(lt), ctypes.addressof(le), ctypes.addressof(n))
    if rc == -2:
        raise FloatingPointError("non-finite activation")
    if rc != 0:
        raise ValueError(f"oracle_calibrate_bf16_counts failed ({rc})")
    return CalibResult(t.value, r.value, lt.value, le.value, n.value)
