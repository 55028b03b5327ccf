"""Graph-timed CATS decode of one layer shape (rotated weight copies defeat L2); one JSON line.

    python scripts/time_decode.py [--model mistral-7b] [--m M] [--batch B] [--k K] [--dense]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

if "--lib" in sys.argv:  # A/B experiments: load another build of the library (e.g. libcats_ab.so)
    from paper_2404_08763_b200 import _lib as _l
    _l.LIB_PATH = os.path.join(os.path.dirname(_l.LIB_PATH), sys.argv[sys.argv.index("--lib") + 1])

import cats_synth
import paper_2404_08763_b200 as cats

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="mistral-7b")
ap.add_argument("--m", type=int, default=0, help="override m (e.g. a TP shard)")
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--k", type=float, default=0.5)
ap.add_argument("--dense", action="store_true")
ap.add_argument("--copies", type=int, default=0, help="weight copies (default: enough for >= 400 MB)")
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--tag", default="")
ap.add_argument("--lib", default="", help="library file name in the package directory (A/B)")
ap.add_argument("--opt", action="append", default=[],
                help="plan option key=value (cats_mlp_plan_options_t field), repeatable")
a = ap.parse_args()
opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in a.opt}
dev = torch.device("cuda:0")
d, m = cats_synth.MODELS[a.model]
m = a.m or m
dt = torch.bfloat16
plan = cats.MlpPlan(d, m, max_batch=8, dtype=dt, **opts)
ws = plan.workspace()
W0 = [w.to(dev) for w in cats_synth.mlp_weights(d, m, dt, layer=0)]
copies = a.copies or max(4, -(-400_000_000 // (3 * 2 * d * m)))
Ws = [W0] + [[w.clone() for w in W0] for _ in range(copies - 1)]
xc = cats_synth.tokens(256, d, dt, seed=100).to(dev)
acts = torch.cat([cats.cats_mlp_gate_act(plan, xc[i:i + 8], W0[0], ws=ws) for i in range(0, 256, 8)])
t, _ = cats.cats_calibrate_threshold(acts, a.k)
x = cats_synth.tokens(a.batch, d, dt, seed=1).to(dev)
y = torch.empty(a.batch, d, device=dev)


def fn():
    for W in Ws:
        if a.dense:
            cats.cats_mlp_dense(plan, x, *W, y=y, ws=ws)
        else:
            cats.cats_mlp_decode(plan, x, *W, t, y=y, ws=ws)


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
# isolated launches: one call bracketed by events, nothing overlapping it
iso = []
for i in range(60):
    W = Ws[i % copies]
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    e0.record()
    if a.dense:
        cats.cats_mlp_dense(plan, x, *W, y=y, ws=ws)
    else:
        cats.cats_mlp_decode(plan, x, *W, t, y=y, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    if i >= 10:
        iso.append(1e3 * e0.elapsed_time(e1))
cats.cats_mlp_decode(plan, x, *W0, t, y=y, ws=ws)
idx, tm, per = cats.cats_mlp_last_active(plan, ws, a.batch)
U = len(idx)
eff = 2 * (d * m + 2 * d * U) if not a.dense else 2 * 3 * d * m
us = min(best)
print(json.dumps(dict(tag=a.tag, model=a.model, d=d, m=m, b=a.batch, k=a.k, dense=a.dense, copies=copies,
                      us=round(us, 3), us_runs=[round(v, 3) for v in best], union=U,
                      iso_us=round(sum(iso) / len(iso), 3),
                      eff_GBps=round(eff / (us * 1e-6) / 1e9, 1), grid=plan.info["grid"],
                      opts=opts)), flush=True)
