"""Graph-timed App. B input-sparse projection (cats_xsparse_gemv) of one shape; one JSON line.

    python scripts/time_xsparse.py [--d-in 4096] [--d-out 6144] [--batch B] [--k K]

Reports the CATS call at sparsity k (t from cats_calibrate_threshold on |x| of 256 calibration
tokens), the same kernels at t = 0 (dense) and cuBLAS (torch.matmul, bf16 -> bf16) on the same
rotated weight copies (>= 400 MB, so every call streams from HBM).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import cats_synth
import paper_2404_08763_b200 as cats

ap = argparse.ArgumentParser()
ap.add_argument("--d-in", type=int, default=4096)
ap.add_argument("--d-out", type=int, default=6144)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--k", type=float, default=0.5)
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--tag", default="")
ap.add_argument("--opt", action="append", default=[],
                help="plan option key=value (cats_mlp_plan_options_t field), repeatable")
a = ap.parse_args()
opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in a.opt}
dev = torch.device("cuda:0")
dt = torch.bfloat16
plan = cats.XsparsePlan(a.d_in, a.d_out, max_batch=8, dtype=dt, **opts)
ws = plan.workspace()
W0 = cats_synth.attn_weights(a.d_in, a.d_out, dt).to(dev)
copies = max(4, -(-400_000_000 // (2 * a.d_in * a.d_out)))
Ws = [W0] + [W0.clone() for _ in range(copies - 1)]
xc = cats_synth.tokens(256, a.d_in, dt, seed=100).to(dev)
t, _ = cats.cats_calibrate_threshold(xc.reshape(-1), a.k)
x = cats_synth.tokens(a.batch, a.d_in, dt, seed=1).to(dev)
y = torch.empty(a.batch, a.d_out, device=dev)


def timed(fn):
    cap = torch.cuda.Stream(dev)
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cap):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cap):
        fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    best = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(a.reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        best.append(1e3 * e0.elapsed_time(e1) / (a.reps * copies))
    return min(best)


us = timed(lambda: [cats.cats_xsparse_gemv(plan, x, W, t, y=y, ws=ws) for W in Ws])
us_t0 = timed(lambda: [cats.cats_xsparse_gemv(plan, x, W, 0.0, y=y, ws=ws) for W in Ws])
us_cublas = timed(lambda: [torch.matmul(x, W) for W in Ws])
cats.cats_xsparse_gemv(plan, x, W0, t, y=y, ws=ws)
idx, tm, per = cats.cats_mlp_last_active(plan, ws, a.batch)
U = len(idx)
esz = 2
moved = U * a.d_out * esz + a.batch * (a.d_in * esz + a.d_out * 4)  # kept W rows + x + y (algorithmic)
print(json.dumps(dict(tag=a.tag, d_in=a.d_in, d_out=a.d_out, b=a.batch, k=a.k, t=t, kept_union=U,
                      kept_frac=round(U / a.d_in, 4), us=round(us, 3), us_t0=round(us_t0, 3),
                      us_cublas=round(us_cublas, 3), speedup_vs_t0=round(us_t0 / us, 3),
                      speedup_vs_cublas=round(us_cublas / us, 3), eff_GBps=round(moved / (us * 1e-6) / 1e9, 1),
                      copies=copies, grid=plan.info["grid"], R=plan.info["rows_per_tile"],
                      clusters=plan.info["stages"], smem=plan.info["smem"])), flush=True)
