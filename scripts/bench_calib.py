"""Calibration benchmark (BASELINE.json config 4): Eq. 3 threshold over 500 samples x 2048 tokens x 11008
channels of synthetic bf16 activations (22.5 GB resident in HBM), GPU radix select vs the CPU oracle.

    python scripts/bench_calib.py [--n N] [--k 0.5 0.7 0.9] [--oracle]
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
a = ap.parse_args()
dt = torch.bfloat16 if a.dtype == "bf16" else torch.float32
t0 = time.time()
acts = cats_synth.calib_acts(a.n, dt, seed=0, device="cuda")
torch.cuda.synchronize()
gen_s = time.time() - t0
ws = torch.empty(cats.cats_calibrate_workspace_bytes(a.n, dt), dtype=torch.uint8, device="cuda")
res = {"n": a.n, "dtype": a.dtype, "bytes": a.n * acts.element_size(), "gen_s": round(gen_s, 2), "k": {}}
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
