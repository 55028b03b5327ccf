"""Render the DESIGN.md §8.1 sweep table from a bench_sweep.py JSONL file.

    python scripts/sweep_table.py profiles/r01_sweep.jsonl
"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]


def get(cfg, b=1, k=0.5, heavy=False):
    for r in rows:
        if r["config"] == cfg and r["b"] == b and r["k"] == k and r["heavy"] == heavy:
            return r
    return None


def f(x):
    return "–" if x is None else f"{x:.1f}"


print("| config | b | k = 0.5 | k = 0.7 | k = 0.9 | dense | Optimal (b = 1) |")
print("|---|---|---|---|---|---|---|")
c1 = get("C1-mistral-7b")
if c1:
    print(f"| C1 Mistral-7B | 1 | {f(c1['us_per_step'])} µs ({c1['eff_GBps']/1e3:.1f} TB/s) | | | "
          f"{f(c1['dense_us_per_step'])} ({c1['dense_us_per_step']/c1['us_per_step']:.2f}×) | {f(c1.get('optimal_us_per_step'))} / – / – |")
C2 = "C2-llama2-7b-32L"
for b in (1, 2, 4, 8):
    r5, r7, r9 = get(C2, b, 0.5), get(C2, b, 0.7), get(C2, b, 0.9)
    if not r5:
        continue
    name = "C2 Llama2-7B 32 layers, Gaussian x" if b == 1 else ""
    extra = f" = {r5['us_per_token_layer']:.1f} µs/token" if b == 8 else ""
    opt = " / ".join(f(get(C2, 1, k).get("optimal_us_per_step")) for k in (0.5, 0.7, 0.9)) if b == 1 else ""
    dense = r5.get("dense_us_per_step")
    ds = f"{f(dense)} ({dense/r5['us_per_step']:.2f}×)" if dense else ""
    print(f"| {name} | {b} | {f(r5['us_per_step'])} ({r5['eff_GBps']/1e3:.1f} TB/s){extra} | "
          f"{f(r7 and r7['us_per_step'])} | {f(r9 and r9['us_per_step'])} | {ds} | {opt} |")
hv = [" / ".join(f(get(C2, b, k, True) and get(C2, b, k, True)["us_per_step"]) for b in (1, 2, 4, 8)) for k in (0.5, 0.7, 0.9)]
print(f"| C2, heavy-tailed x | 1 / 2 / 4 / 8 | {hv[0]} | {hv[1]} | {hv[2]} | | |")
c3 = [get(f"C3-llama2-13b-TP{p}-shard") for p in (1, 2, 4, 8)]
if all(c3):
    print("| C3 Llama2-13B shard, b = 1 | TP1 / 2 / 4 / 8 | " + " / ".join(f(r["us_per_step"]) for r in c3) + " µs | | | "
          + " / ".join(f(r["dense_us_per_step"]) for r in c3) + " | " + " / ".join(f(r.get("optimal_us_per_step")) for r in c3) + " |")
c0 = get("C0-toy")
if c0:
    print(f"| C0 toy fp32 | 1 | {f(c0['us_per_step'])} (launch-bound) | | | {f(c0['dense_us_per_step'])} | {f(c0.get('optimal_us_per_step'))} |")
