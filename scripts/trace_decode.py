"""Per-CTA timeline of one pipelined decode step (options.trace = 1 globaltimer stamps).

    python scripts/trace_decode.py [--model mistral-7b] [--batch 1] [--graph]
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import cats_synth

if "--lib" in sys.argv:  # A/B experiments: load another build of the library (e.g. libcats_ab.so)
    from paper_2404_08763_b200 import _lib as _l
    _l.LIB_PATH = os.path.join(os.path.dirname(_l.LIB_PATH), sys.argv[sys.argv.index("--lib") + 1])
import paper_2404_08763_b200 as cats

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="mistral-7b")
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--k", type=float, default=0.5)
ap.add_argument("--dense", action="store_true")
ap.add_argument("--json")
ap.add_argument("--graph", action="store_true", help="trace a CUDA-graph replay of the step (no host launch gaps)")
ap.add_argument("--m", type=int, default=0, help="override m (e.g. a TP shard)")
ap.add_argument("--opt", action="append", default=[], help="plan option key=value, repeatable")
ap.add_argument("--lib", default="", help="library file name in the package directory (A/B)")
a = ap.parse_args()
opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in a.opt}
d, m = cats_synth.MODELS[a.model]
if a.m:
    m = a.m
dev = torch.device("cuda:0")
W = [w.to(dev) for w in cats_synth.mlp_weights(d, m, torch.bfloat16)]
copies = [W] + [[w.clone() for w in W] for _ in range(3)]
plan = cats.MlpPlan(d, m, max_batch=8, trace=1, **opts)
ws = plan.workspace()
off, nbytes = ctypes.c_size_t(), ctypes.c_size_t()
plan._lib.cats_mlp_trace_info(plan.handle, ctypes.byref(off), ctypes.byref(nbytes))
assert nbytes.value > 0, "tracing off"
xc = cats_synth.tokens(64, d, torch.bfloat16, seed=0).to(dev)
acts = torch.cat([cats.cats_mlp_gate_act(plan, xc[i:i + 8], W[0], ws=ws) for i in range(0, 64, 8)])
t, _ = cats.cats_calibrate_threshold(acts, a.k)
x = cats_synth.tokens(a.batch, d, torch.bfloat16, seed=1).to(dev)
y = torch.empty(a.batch, d, device=dev)


def step(i):
    c = copies[i % 4]
    if a.dense:
        cats.cats_mlp_dense(plan, x, c[0], c[1], c[2], y=y, ws=ws)
    else:
        cats.cats_mlp_decode(plan, x, c[0], c[1], c[2], t, y=y, ws=ws)


for i in range(20):
    step(i)
torch.cuda.synchronize()
if a.graph:  # the traced step as a graph replay: the kernels' launches carry no host latency between them
    side = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        step(20)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=side):
            step(20)
    g.replay()
    torch.cuda.synchronize()
ws[off.value:off.value + nbytes.value].zero_()
if a.graph:
    g.replay()
else:
    step(20)
torch.cuda.synchronize()
tr = ws[off.value:off.value + nbytes.value].cpu().numpy().view(np.uint64).reshape(3, 512, 8).astype(np.int64)
rep = {}
t0 = None
names = {0: ["start", "primed", "jobs_done", "exit", "reduced|KA:pdl_trig", "all_warps_done", "staged", "bulk_done"],
         1: ["start", "list_ready", "jobs_done", "reducer_go", "exit", "masks_read", "prefix_done", "ticket_known"]}
titles = {0: "K12 / KA", 1: "KB"}
for k in range(2):
    g = int((tr[k, :, 0] > 0).sum())  # CTAs that stamped
    if g == 0:
        continue
    if t0 is None:
        t0 = tr[k, :g, 0].min()
    print(f"{titles[k]} ({g} CTAs), us relative to the first CTA start:")
    for sidx, nm in enumerate(names[k]):
        v = (tr[k, :g, sidx] - t0) / 1e3
        v = v[tr[k, :g, sidx] > 0]
        if len(v):
            print(f"   {nm:12s} min {v.min():8.2f}  avg {v.mean():8.2f}  max {v.max():8.2f}")
            rep[f"K{k}.{nm}"] = [float(v.min()), float(v.mean()), float(v.max())]
g = int((tr[0, :, 0] > 0).sum())
gb = int((tr[1, :, 0] > 0).sum())
if gb and tr[2, :gb, 5].max() > 0 and tr[2, :gb, 4].max() == 0:  # KB-only statistics written
    sb = tr[2, :gb, :].astype(np.float64)
    print("KB per-CTA: producer empty-wait ns avg/max", sb[:, 0].mean().round(0), sb[:, 0].max(),
          "| consumer full-wait ns avg/max", sb[:, 3].mean().round(0), sb[:, 3].max(),
          "| chunks avg/min/max", sb[:, 5].mean().round(1), sb[:, 5].min(), sb[:, 5].max(),
          "| claim-wait ns", sb[:, 1].mean().round(0), "| x1-issue ns", sb[:, 2].mean().round(0),
          "| search ns", sb[:, 4].mean().round(0), "| search+bulk ns", sb[:, 6].mean().round(0))
st = tr[2, :g, :7].astype(np.float64)
if st[:, 2].max() > 0:  # K12 producer / consumer statistics
    print("K12 per-CTA stats (avg/min/max):")
    for i, nm in enumerate(["producer wait ns", "producer busy ns", "jobs retired", "consumer wait ns", "gate jobs",
                            "ud jobs", "producer issue ns"]):
        print(f"   {nm:18s} {st[:, i].mean():10.1f} {st[:, i].min():10.1f} {st[:, i].max():10.1f}")
    lg = (tr[2, :g, 7] - t0) / 1e3
    jd = (tr[0, :g, 2] - t0) / 1e3
    ok = tr[2, :g, 7] > 0
    if ok.any():
        print("last GATE issue (us): p10/50/90/max", np.percentile(lg[ok], [10, 50, 90, 100]).round(2))
        print("jobs_done - last GATE issue (us): p10/50/90/max",
              np.percentile((jd - lg)[ok], [10, 50, 90, 100]).round(2))
    print("corr(jobs retired, jobs_done time)", round(float(np.corrcoef(st[:, 2], jd)[0, 1]), 3))
if a.json:
    json.dump(rep, open(a.json, "w"), indent=1)
