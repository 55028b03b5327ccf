"""Per-CTA timeline of the App. B kernel XS (options.trace = 1 globaltimer stamps), one eager call.

    python scripts/trace_xsparse.py [--d-in 4096] [--d-out 6144] [--batch 1] [--k 0.5]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import cats_synth
import paper_2404_08763_b200 as cats

ap = argparse.ArgumentParser()
ap.add_argument("--d-in", type=int, default=4096)
ap.add_argument("--d-out", type=int, default=6144)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--k", type=float, default=0.5)
a = ap.parse_args()
dev = torch.device("cuda:0")
plan = cats.XsparsePlan(a.d_in, a.d_out, max_batch=8, trace=1)
ws = plan.workspace()
off, nbytes = ctypes.c_size_t(), ctypes.c_size_t()
plan._lib.cats_mlp_trace_info(plan.handle, ctypes.byref(off), ctypes.byref(nbytes))
assert nbytes.value > 0
Ws = [cats_synth.attn_weights(a.d_in, a.d_out).to(dev) for _ in range(1)]
Ws += [Ws[0].clone() for _ in range(3)]
t, _ = cats.cats_calibrate_threshold(cats_synth.tokens(256, a.d_in, seed=100).to(dev).reshape(-1), a.k)
x = cats_synth.tokens(a.batch, a.d_in, seed=1).to(dev)
for i in range(20):
    cats.cats_xsparse_gemv(plan, x, Ws[i % 4], t, ws=ws)
torch.cuda.synchronize()
ws[off.value:off.value + nbytes.value].zero_()
cats.cats_xsparse_gemv(plan, x, Ws[1], t, ws=ws)
torch.cuda.synchronize()
tr = ws[off.value:off.value + nbytes.value].cpu().numpy().view(np.uint64).reshape(3, 512, 8).astype(np.int64)
g = int((tr[0, :, 0] > 0).sum())
t0 = tr[0, :g, 0].min()
print(f"XS ({g} CTAs, grid {plan.info['grid']}, R {plan.info['rows_per_tile']}), us from the first CTA start:")
for k, s, nm in [(0, 0, "start"), (0, 5, "x_staged"), (0, 6, "mask_done"), (0, 7, "prefix_done"),
                 (1, 0, "range_found"), (1, 1, "list_written"), (1, 2, "list_synced"), (0, 1, "list_ready"),
                 (0, 2, "rows_done"), (0, 3, "cluster_sync1"), (0, 4, "exit")]:
    v = (tr[k, :g, s] - t0) / 1e3
    print(f"   {nm:14s} min {v.min():7.2f}  p50 {np.median(v):7.2f}  max {v.max():7.2f}")
