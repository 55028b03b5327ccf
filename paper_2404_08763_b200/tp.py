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


def tp_decode(plan, x, W_gate_shard, W_up_shard, W_down_shard, t: float, y=None, ws=None, group=None, stream=None):
    """y = sum over ranks of the rank-local CATS-MLP partials (one NCCL all-reduce)."""
    y = cats_mlp_decode(plan, x, W_gate_shard, W_up_shard, W_down_shard, t, y=y, ws=ws, stream=stream)
    if group is not None and dist.get_world_size(group) > 1:
        dist.all_reduce(y, group=group)
    return y


__all__ = ["shard_rows", "calibrate_threshold", "tp_decode", "CATS_BF16"]
