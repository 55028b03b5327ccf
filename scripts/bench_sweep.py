"""Sweep over the BASELINE.json configurations on one B200 (JSON lines to stdout).

  C0  toy SwiGLU (d=64, m=176, fp32, b=1, k=0.5)
  C1  Mistral-7B layer (4096 x 14336), b=1, k=0.5 (plus the library dense path)
  C2  Llama2-7B 32-layer MLP stack (4096 x 11008, 32 distinct layers = 8.66 GB), per-layer t,
      b in {1,2,4,8}, k in {0.5,0.7,0.9}, Gaussian and heavy-tailed ("hot neuron") inputs;
      graph-captured stack time / 32 = us per token-layer
  C3  Llama2-13B (5120 x 13824) per-GPU shard of a TP = 1/2/4/8 split along m (the all-reduce of
      b x d fp32 is not included: one GPU in this pool)

Every number is CUDA-event timed on the launching stream over CUDA-graph replays; L2 is defeated by
the working set (>= 4 weight copies or the 8.66 GB stack).

    python scripts/bench_sweep.py [--quick]
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
ap.add_argument("--quick", action="store_true")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--only", default="", help="comma-separated config prefixes to run (C0,C1,C2,N3,C3)")
a = ap.parse_args()
dev = torch.device("cuda:0")
torch.cuda.set_device(dev)


def graph_time(fn, reps):
    """us per call of fn() (a sequence of library calls), CUDA graph replays, events."""
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
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / reps


def calibrate(plan, ws, Wg, d, k, dtype, ntok=256, seed=0, heavy=False):
    xc = cats_synth.tokens(ntok, d, dtype, seed=seed, heavy=heavy).to(dev)
    acts = torch.cat([cats.cats_mlp_gate_act(plan, xc[i:i + 8], Wg, ws=ws) for i in range(0, ntok, 8)])
    t, _ = cats.cats_calibrate_threshold(acts, k)
    return t


def emit(**kw):
    print(json.dumps(kw), flush=True)


def want(name):
    return not a.only or any(name.startswith(p) for p in a.only.split(","))


_STACKS = {}


def weights(d, m, layers, copies, heavy, dtype):
    """Device weight list (cached across b / k: generating a 32-layer stack on the host is slow)."""
    key = (d, m, layers, copies, heavy, dtype)
    if key not in _STACKS:
        _STACKS.clear()
        torch.cuda.empty_cache()
        Ws = [[w.to(dev) for w in cats_synth.mlp_weights(d, m, dtype, layer=l, heavy=heavy)] for l in range(layers)]
        if copies > 1:  # rotated copies of a single layer (defeat L2)
            Ws = Ws + [[w.clone() for w in Ws[0]] for _ in range(copies - 1)]
        _STACKS[key] = Ws
    return _STACKS[key]


def run_layers(name, d, m, layers, copies, b, k, heavy, dtype=torch.bfloat16, dense_too=False, optimal=True):
    plan = cats.MlpPlan(d, m, max_batch=8, dtype=dtype)
    ws = plan.workspace()
    Ws = weights(d, m, layers, copies, heavy, dtype)
    ts = [calibrate(plan, ws, W[0], d, k, dtype, seed=100 + l, heavy=heavy) if k > 0 else 0.0
          for l, W in enumerate(Ws[:layers])]
    ts = ts + [ts[0]] * (len(Ws) - len(ts))
    x = cats_synth.tokens(b, d, dtype, seed=1, heavy=heavy).to(dev)
    y = torch.empty(b, d, device=dev)
    n = len(Ws)

    def fn():
        for W, t in zip(Ws, ts):
            cats.cats_mlp_decode(plan, x, W[0], W[1], W[2], t, y=y, ws=ws)

    us = graph_time(fn, a.reps) / n
    # union / per-token activity of one layer
    cats.cats_mlp_decode(plan, x, *Ws[0], ts[0], y=y, ws=ws)
    idx, tm, per = cats.cats_mlp_last_active(plan, ws, b)
    U = len(idx)
    eff = 2 * d * m + 4 * d * U  # algorithmic bytes (bf16 weights only); fp32 toy: x2
    esz = 2 if dtype == torch.bfloat16 else 4
    eff = eff * esz // 2
    rec = dict(config=name, d=d, m=m, b=b, k=k, heavy=heavy, layers=n, us_per_token_layer=round(us / b, 3),
               us_per_step=round(us, 3), union_active=U, union_frac=round(U / m, 4),
               per_token_sparsity=round(1 - float(per.mean()) / m, 4), eff_GBps=round(eff / (us * 1e-6) / 1e9, 1),
               kernels_per_call=cats.cats_mlp_kernels_per_call(plan, b))
    if dense_too:
        def fd():
            for W in Ws:
                cats.cats_mlp_dense(plan, x, W[0], W[1], W[2], y=y, ws=ws)
        ud = graph_time(fd, a.reps) / n
        rec.update(dense_us_per_step=round(ud, 3), speedup_vs_dense=round(ud / us, 4),
                   dense_GBps=round(3 * 2 * d * m * esz // 2 / (ud * 1e-6) / 1e9, 1))
    if optimal and b == 1 and k > 0:
        # the paper's "Optimal" (Fig. 3): a dense MLP with only the (1 - k) m neurons CATS keeps --
        # what a perfect predictor of the active set could at best achieve with the same kernel
        mo = max(8, int(round(m * (1 - k))))
        po = cats.MlpPlan(d, mo, max_batch=8, dtype=dtype)
        wso = po.workspace()
        Wo = [[w[:mo] for w in W] for W in Ws]

        def fo():
            for W in Wo:
                cats.cats_mlp_dense(po, x, W[0], W[1], W[2], y=y, ws=wso)
        uo = graph_time(fo, a.reps) / n
        rec.update(optimal_us_per_step=round(uo, 3), cats_over_optimal=round(us / uo, 4))
    emit(**rec)


def run_chained(name, d, m, layers, b, k, heavy=False, dtype=torch.bfloat16):
    """N3 decode-loop proxy with real layer-to-layer dynamics: layer l's output feeds layer l + 1 the way a
    pre-norm transformer block does, h_l = RMSNorm(x_l) (unit gain), x_{l+1} = bf16(x_l + MLP_l(h_l)) (torch
    ops between the layers: plumbing, not the hot path; attention is not modelled), and each layer's t is
    calibrated on 256 calibration tokens that went through the same chain. Timed as one CUDA graph of the
    whole stack (norm + decode + residual add per layer) / layers."""
    plan = cats.MlpPlan(d, m, max_batch=8, dtype=dtype)
    ws = plan.workspace()
    Ws = weights(d, m, layers, 1, heavy, dtype)
    def rmsnorm(v, out):
        vf = v.float()
        out.copy_(vf * torch.rsqrt(vf.pow(2).mean(-1, keepdim=True) + 1e-6))

    xc = cats_synth.tokens(256, d, dtype, seed=100, heavy=heavy).to(dev)
    hc = torch.empty_like(xc)
    yc = torch.empty(8, d, device=dev)
    ts = []
    for l in range(layers):
        rmsnorm(xc, hc)
        acts = torch.cat([cats.cats_mlp_gate_act(plan, hc[i:i + 8], Ws[l][0], ws=ws) for i in range(0, 256, 8)])
        ts.append(cats.cats_calibrate_threshold(acts, k)[0] if k > 0 else 0.0)
        for i in range(0, 256, 8):
            cats.cats_mlp_decode(plan, hc[i:i + 8], *Ws[l], ts[l], y=yc, ws=ws)
            xc[i:i + 8].add_(yc)
    x0 = cats_synth.tokens(b, d, dtype, seed=1, heavy=heavy).to(dev)
    x = x0.clone()
    h = torch.empty_like(x)
    y = torch.empty(b, d, device=dev)

    def fn():
        x.copy_(x0)
        for W, t in zip(Ws[:layers], ts):
            rmsnorm(x, h)
            cats.cats_mlp_decode(plan, h, W[0], W[1], W[2], t, y=y, ws=ws)
            x.add_(y)

    us = graph_time(fn, a.reps) / layers

    def fn_plumbing():  # the same graph without the decodes: norm + residual add only
        x.copy_(x0)
        for _ in range(layers):
            rmsnorm(x, h)
            x.add_(y)

    us_plumb = graph_time(fn_plumbing, a.reps) / layers
    # realised activity per layer along the chain (eager pass)
    x.copy_(x0)
    unions, spars = [], []
    for W, t in zip(Ws[:layers], ts):
        rmsnorm(x, h)
        cats.cats_mlp_decode(plan, h, W[0], W[1], W[2], t, y=y, ws=ws)
        idx, tm, per = cats.cats_mlp_last_active(plan, ws, b)
        unions.append(len(idx) / m)
        spars.append(1 - float(per.mean()) / m)
        x.add_(y)
    emit(config=name, d=d, m=m, b=b, k=k, heavy=heavy, layers=layers, chained=True,
         us_per_token_layer=round(us / b, 3), us_per_step=round(us, 3),
         us_plumbing_per_layer=round(us_plumb, 3), us_decode_per_token_layer=round((us - us_plumb) / b, 3),
         union_frac_mean=round(sum(unions) / layers, 4), union_frac_min=round(min(unions), 4),
         union_frac_max=round(max(unions), 4), per_token_sparsity_mean=round(sum(spars) / layers, 4),
         t_first=ts[0], t_last=ts[-1])


if want("C0"):
    run_layers("C0-toy", 64, 176, 1, 1, 1, 0.5, False, dtype=torch.float32, dense_too=True)
if want("C1"):
    run_layers("C1-mistral-7b", 4096, 14336, 1, 4, 1, 0.5, False, dense_too=True)
bs = [1, 8] if a.quick else [1, 2, 4, 8]
ks = [0.5, 0.9] if a.quick else [0.5, 0.7, 0.9]
for heavy in ([False] if a.quick else [False, True]) if want("C2") else []:
    for k in ks:
        for b in bs:
            run_layers("C2-llama2-7b-32L", 4096, 11008, 32, 1, b, k, heavy, dense_too=(k == 0.5 and not heavy))
for b in ([1] if a.quick else [1, 8]) if want("N3") else []:
    for k in ([0.5] if a.quick else [0.5, 0.7, 0.9]):
        run_chained("N3-llama2-7b-32L-chained", 4096, 11008, 32, b, k)
for P in [1, 2, 4, 8] if want("C3") else []:
    for b in (1, 8):
        run_layers(f"C3-llama2-13b-TP{P}-shard", 5120, 13824 // P, 1, 4 * P if P > 1 else 4, b, 0.5, False,
                   dense_too=True, optimal=(b == 1))
