"""Calibration benchmark (BASELINE.json config 4): Eq. 3 threshold over 500 samples x 2048 tokens x 11008
channels of synthetic bf16 activations (22.5 GB resident in HBM), GPU radix select vs the CPU oracle.

--source gate (default): acts = bf16(SiLU(x W_gate)) collected by the library's own gate
kernel (cats_mlp_gate_act, fp32 out, rounded to bf16) from synthetic tokens x and a Llama2-7B-shaped
W_gate (sigma_u = 0.30); --source gaussian: i.i.d. N(0, 0.30^2) values rounded to bf16 (round 1).

    python scripts/bench_calib.py [--n N] [--k 0.5 0.7 0.9] [--oracle] [--source gate|gaussian]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import cats_synth
import paper_2404_08763_b200 as cats

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=500 * 2048 * 11008)
ap.add_argument("--k", type=float, nargs="+", default=[0.5, 0.7, 0.9])
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--oracle", action="store_true", help="also run the CPU oracle on the identical bytes")
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--source", default="gate", choices=["gate", "gaussian"])
a = ap.parse_args()
dt = torch.bfloat16 if a.dtype == "bf16" else torch.float32
t0 = time.time()
if a.source == "gaussian":
    acts = cats_synth.calib_acts(a.n, dt, seed=0, device="cuda")
else:
    d, m = cats_synth.MODELS["llama2-7b"]
    assert a.n % m == 0, "--n must be a multiple of m = 11008 (tokens x channels)"
    ntok = a.n // m
    Wg = cats_synth.mlp_weights(d, m, torch.bfloat16)[0].cuda()
    plan = cats.MlpPlan(d, m, max_batch=8)
    wsp = plan.workspace()
    acts = torch.empty(a.n, dtype=dt, device="cuda")
    chunk = 2048  # one calibration sample of 2048 tokens at a time
    buf = torch.empty(chunk, m, dtype=torch.float32, device="cuda")
    for s0 in range(0, ntok, chunk):
        nt = min(chunk, ntok - s0)
        xs = cats_synth.tokens(nt, d, torch.bfloat16, seed=1_000_000 + s0 // chunk).cuda()
        for i in range(0, nt, 8):
            cats.cats_mlp_gate_act(plan, xs[i:i + 8], Wg, acts=buf[i:i + 8], ws=wsp)
        acts[s0 * m:(s0 + nt) * m] = buf[:nt].reshape(-1).to(dt)
    del buf, Wg, wsp
torch.cuda.synchronize()
gen_s = time.time() - t0
ws = torch.empty(cats.cats_calibrate_workspace_bytes(a.n, dt), dtype=torch.uint8, device="cuda")
res = {"n": a.n, "dtype": a.dtype, "source": a.source, "bytes": a.n * acts.element_size(), "gen_s": round(gen_s, 2),
       "k": {}}
for k in a.k:
    t, info = cats.cats_calibrate_threshold(acts, k, ws=ws)  # warm-up
    times = []
    for _ in range(a.reps):
        torch.cuda.synchronize()
        s = time.perf_counter()
        t, info = cats.cats_calibrate_threshold(acts, k, ws=ws)  # blocks until t is on the host
        times.append(time.perf_counter() - s)
    ms = 1e3 * min(times)
    full_pass_bytes = info["passes"] * res["bytes"]
    res["k"][k] = {"t": t, "t_bits": info["t_bits"], "count_lt": info["count_lt"], "count_le": info["count_le"],
                   "passes": info["passes"], "ms_min": round(ms, 3), "ms_median": round(1e3 * sorted(times)[len(times) // 2], 3),
                   "GBps_over_full_passes": round(full_pass_bytes / (ms * 1e-3) / 1e9, 1)}
if a.oracle:
    import oracle
    t0 = time.time()
    counts = np.zeros(65536, np.uint64)
    chunk = 1 << 30
    for s in range(0, a.n, chunk):
        oracle.bf16_counts(cats_synth.bf16_bits(acts[s:s + chunk].cpu()), counts)
    for k in a.k:
        ref = oracle.calibrate_bf16_counts(counts, k)
        r = res["k"][k]
        r["oracle_t"] = ref.t
        r["bit_exact"] = (ref.t == r["t"] and ref.count_lt == r["count_lt"] and ref.count_le == r["count_le"])
    res["oracle_s"] = round(time.time() - t0, 1)
    res["oracle_cores"] = 1
print(json.dumps(res))
