"""Tensor parallelism along the intermediate dimension m.

Rank p of P holds neuron rows [p*m/P, (p+1)*m/P) of W_gate, W_up and the neuron-major W_down. x and the
layer-global scalar t are replicated, so masking needs no communication (Eq. 5 is per neuron); each
rank's cats_mlp_decode yields a partial y_p and one all-reduce (sum, fp32, b x d) combines them.

Calibration shards too: each rank histograms its activation shard with cats_calib_hist, the
histogram and counters are all-reduced between steps, and every rank runs the same cats_calib_step,
so t is bit-identical on all ranks.

This module only sequences library calls and torch.distributed collectives (plumbing).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import CATS_BF16, cats_calib_hist, cats_calib_step, cats_calib_window_init, cats_calibrate_threshold
from . import cats_mlp_decode


def shard_rows(m: int, world: int, rank: int) -> slice:
    if m % world:
        raise ValueError(f"m={m} is not divisible by the TP degree {world}")
    ms = m // world
    return slice(rank * ms, (rank + 1) * ms)


def _bits_to_float(tb: int, dtype: torch.dtype) -> float:
    bits = np.uint32(tb << 16) if dtype == torch.bfloat16 else np.uint32(tb)
    return float(np.array([bits], np.uint32).view(np.float32)[0])


def calibrate_threshold(acts: torch.Tensor, k: float, group=None, hist_fn=None, max_steps: int = 32) -> float:
    """Eq. 3 threshold over the union of every rank's `acts` (device tensors).

    group=None (or a 1-rank group): the single-GPU library call. Otherwise the sharded radix select.
    hist_fn (tests only) replaces the device pass with an equivalent host function."""
    if group is None or dist.get_world_size(group) == 1:
        if hist_fn is None:
            t, _ = cats_calibrate_threshold(acts, k)
            return t
    n_local = acts.numel()
    n_t = torch.tensor([n_local], dtype=torch.int64, device=acts.device if hist_fn is None else "cpu")
    if group is not None:
        dist.all_reduce(n_t, group=group)
    n = int(n_t.item())
    w = cats_calib_window_init(n, acts.dtype)
    dev = acts.device if hist_fn is None else torch.device("cpu")
    hist = torch.zeros(32768, dtype=torch.int64, device=dev)
    counts = torch.zeros(8, dtype=torch.int64, device=dev)  # CATS_CALIB_COUNTS_LEN (4 counts + pass scratch)
    for _ in range(max_steps):
        hist.zero_()
        counts.zero_()
        if hist_fn is None:
            cats_calib_hist(acts, w, hist, counts)
        else:
            h, c = hist_fn(acts, w)
            hist[: w.nbins] += torch.from_numpy(h.astype(np.int64))
            counts[:4] += torch.from_numpy(c.astype(np.int64))
        if group is not None:
            dist.all_reduce(hist, group=group)
            dist.all_reduce(counts, group=group)
        done, tb, _, _ = cats_calib_step(hist[: w.nbins].cpu().numpy().view(np.uint64),
                                         counts[:4].cpu().numpy().view(np.uint64), n, acts.dtype, k, w)
        if done:
            return _bits_to_float(tb, acts.dtype)
    raise RuntimeError("sharded calibration did not converge")


class TpComm:
    """The fused one-shot cross-rank reduction (cats_tp_allreduce) for one process group:
    every rank allocates its symmetric buffer, exports it with CUDA IPC, and opens every peer's (the
    handles travel through torch.distributed, the plumbing; the reduction itself is one library kernel
    that writes and reads peer memory over NVLink)."""

    def __init__(self, n_max: int, group=None, device=None):
        import ctypes
        from . import _lib
        self._lib = _lib.load()
        self.rank = dist.get_rank(group) if group is not None else 0
        self.world = dist.get_world_size(group) if group is not None else 1
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.n_max = int(n_max)
        nb = ctypes.c_size_t()
        _chk(self._lib.cats_tp_buffer_bytes(self.world, self.n_max, ctypes.byref(nb)), "cats_tp_buffer_bytes")
        # the buffer is its own cudaMalloc allocation (not a slice of torch's caching allocator): an IPC
        # handle maps a whole allocation, so peers open exactly this buffer
        self._buf = ctypes.c_void_p()
        _chk(self._lib.cats_tp_buffer_alloc(nb.value, self.device, ctypes.byref(self._buf)), "cats_tp_buffer_alloc")
        h = (ctypes.c_uint8 * 64)()
        _chk(self._lib.cats_ipc_handle_get(self._buf, h), "cats_ipc_handle_get")
        handles = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(handles, bytes(h), group=group)
        else:
            handles = [bytes(h)]
        self._opened = []
        ptrs = (ctypes.c_void_p * self.world)()
        for r, hb in enumerate(handles):
            if r == self.rank:
                ptrs[r] = self._buf.value
                continue
            p = ctypes.c_void_p()
            _chk(self._lib.cats_ipc_handle_open((ctypes.c_uint8 * 64).from_buffer_copy(hb), self.device,
                                                ctypes.byref(p)), "cats_ipc_handle_open")
            self._opened.append(p)
            ptrs[r] = p.value
        self._h = ctypes.c_void_p()
        _chk(self._lib.cats_tp_comm_create(self.rank, self.world, self.n_max, ptrs, self.device, ctypes.byref(self._h)),
             "cats_tp_comm_create")
        if self.world > 1:
            dist.barrier(group=group)

    def allreduce(self, x: torch.Tensor, y: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """y = sum over ranks of x (fp32, fixed rank order, identical on every rank); x and y may alias."""
        y = x if y is None else y
        st = torch.cuda.current_stream(self.device) if stream is None else stream
        _chk(self._lib.cats_tp_allreduce(self._h, x.data_ptr(), y.data_ptr(), x.numel(), st.cuda_stream),
             "cats_tp_allreduce")
        return y

    def __del__(self):
        lib = getattr(self, "_lib", None)
        if lib is None:
            return
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.cats_tp_comm_destroy(h)
        for p in getattr(self, "_opened", []):
            lib.cats_ipc_handle_close(p)
        b = getattr(self, "_buf", None)
        if b is not None and b.value:
            lib.cats_tp_buffer_free(b)


def _chk(rc, where):
    if rc != 0:
        from . import CatsError
        raise CatsError(rc, where)


def tp_decode(plan, x, W_gate_shard, W_up_shard, W_down_shard, t: float, y=None, ws=None, group=None, stream=None,
              comm: TpComm | None = None):
    """y = sum over ranks of the rank-local CATS-MLP partials: the fused one-shot reduction (comm) or one
    NCCL all-reduce (group)."""
    y = cats_mlp_decode(plan, x, W_gate_shard, W_up_shard, W_down_shard, t, y=y, ws=ws, stream=stream)
    if comm is not None and comm.world > 1:
        comm.allreduce(y, stream=stream)
    elif group is not None and dist.get_world_size(group) > 1:
        dist.all_reduce(y, group=group)
    return y





class EmulatedTpComms:
    """P ranks of the fused reduction emulated on ONE device (cats_tp_allreduce_emulated): P symmetric
    buffers on this GPU and P comms over them; allreduce(xs, ys) runs every rank's step in one cooperative
    launch. For testing the exchange protocol where fewer GPUs than ranks are available."""

    def __init__(self, world: int, n_max: int, device=None):
        import ctypes
        from . import _lib
        self._lib = _lib.load()
        self.world, self.n_max = int(world), int(n_max)
        self.device = torch.cuda.current_device() if device is None else int(device)
        nb = ctypes.c_size_t()
        _chk(self._lib.cats_tp_buffer_bytes(self.world, self.n_max, ctypes.byref(nb)), "cats_tp_buffer_bytes")
        self.bufs = [torch.zeros(nb.value, dtype=torch.uint8, device=f"cuda:{self.device}") for _ in range(world)]
        ptrs = (ctypes.c_void_p * world)(*[b.data_ptr() for b in self.bufs])
        self._h = []
        for r in range(world):
            h = ctypes.c_void_p()
            _chk(self._lib.cats_tp_comm_create(r, world, self.n_max, ptrs, self.device, ctypes.byref(h)),
                 "cats_tp_comm_create")
            self._h.append(h)

    def allreduce(self, xs, ys=None, stream=None):
        import ctypes
        ys = xs if ys is None else ys
        n = xs[0].numel()
        st = torch.cuda.current_stream(self.device) if stream is None else stream
        H = (ctypes.c_void_p * self.world)(*[h.value for h in self._h])
        X = (ctypes.c_void_p * self.world)(*[x.data_ptr() for x in xs])
        Y = (ctypes.c_void_p * self.world)(*[y.data_ptr() for y in ys])
        _chk(self._lib.cats_tp_allreduce_emulated(H, self.world, X, Y, n, st.cuda_stream), "cats_tp_allreduce_emulated")
        return ys

    def __del__(self):
        lib = getattr(self, "_lib", None)
        for h in getattr(self, "_h", []):
            if lib is not None and h.value:
                lib.cats_tp_comm_destroy(h)
__all__ = ["shard_rows", "calibrate_threshold", "tp_decode", "TpComm", "EmulatedTpComms", "CATS_BF16"]
