"""Small driver for ncu: a few CATS decode steps (and dense steps) at a BASELINE shape."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import cats_synth
import paper_2404_08763_b200 as cats

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="mistral-7b")
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--k", type=float, default=0.5)
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--dense", action="store_true")
a = ap.parse_args()
d, m = cats_synth.MODELS[a.model]
dev = torch.device("cuda:0")
W = [w.to(dev) for w in cats_synth.mlp_weights(d, m, torch.bfloat16)]
copies = [W] + [[w.clone() for w in W] for _ in range(3)]
plan = cats.MlpPlan(d, m, max_batch=8)
ws = plan.workspace()
xc = cats_synth.tokens(64, d, torch.bfloat16, seed=0).to(dev)
acts = torch.cat([cats.cats_mlp_gate_act(plan, xc[i:i + 8], W[0], ws=ws) for i in range(0, 64, 8)])
t, _ = cats.cats_calibrate_threshold(acts, a.k)
x = cats_synth.tokens(a.batch, d, torch.bfloat16, seed=1).to(dev)
y = torch.empty(a.batch, d, device=dev)
for i in range(a.steps):
    c = copies[i % 4]
    cats.cats_mlp_decode(plan, x, c[0], c[1], c[2], t, y=y, ws=ws)
if a.dense:
    for i in range(a.steps):
        c = copies[i % 4]
        cats.cats_mlp_dense(plan, x, c[0], c[1], c[2], y=y, ws=ws)
torch.cuda.synchronize()
print("ok t=", t)
