"""Write the committed ncu summaries under profiles/ from a gpurun_out/ capture.

    python scripts/make_profile_summary.py --tag r01 [--rep gpurun_out/r01_prof.ncu-rep]
        [--launches gpurun_out/r01_launches.csv] [--bench gpurun_out/bench.log]

Produces profiles/<tag>_ncu_summary.md (per-kernel metrics + stall reasons), profiles/<tag>_launches.csv
(every launch with device time and DRAM bytes, cold-cache and serialised under ncu: compare shares,
not absolutes) and profiles/ncu_traffic.json (DRAM bytes per launch of the dominant kernel, read by
bench.py for the roofline "traffic" field).
"""
import argparse
import collections
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--bench")
    ap.add_argument("--extra", nargs="*", default=[],
                    help="label::path.ncu-rep of further full-set captures (e.g. the b>=2 split path)")
    a = ap.parse_args()
    rep = a.rep or os.path.join(ROOT, "gpurun_out", f"{a.tag}_prof.ncu-rep")
    lau = a.launches or os.path.join(ROOT, "gpurun_out", f"{a.tag}_launches.csv")
    out = os.path.join(ROOT, "profiles")
    os.makedirs(out, exist_ok=True)
    lines = [f"# ncu summary ({a.tag})", "",
             "Captured with `ncu --set full --clock-control none --import-source on` on one B200 (sm_100a),",
             "command `python scripts/prof_decode.py --steps 8 --dense` (Mistral-7B MLP layer, d=4096, m=14336,",
             "bf16, b=1, k=0.5 threshold calibrated on 64 tokens; 4 rotated weight copies). ncu flushes caches",
             "between replays, so per-launch times are cold-cache and serialised.", ""]
    traffic = {}
    if os.path.exists(rep):
        data = ncu_summary.raw(rep)
        lines += ["## Full-set capture", "",
                  "| kernel | duration | DRAM read | DRAM write | regs | dyn smem | grid x block | top stalls |",
                  "|---|---|---|---|---|---|---|---|"]
        for d in data:
            lines.append(f"| `{d['kernel']}` | {d.get('dur')} {d.get('dur_unit')} | {d.get('dram_rd')} "
                         f"{d.get('dram_rd_unit')} | {d.get('dram_wr')} {d.get('dram_wr_unit')} | {d.get('regs')} | "
                         f"{d.get('dyn_smem')} {d.get('dyn_smem_unit')} | {d.get('grid')} x {d.get('block')} | "
                         f"{', '.join(f'{n} {v}' for v, n in d['stalls'][:4])} |")
        lines += ["", "SM activity (cycles, avg / min / max over SMs vs elapsed):", ""]
        for d in data:
            lines.append(f"- `{d['kernel']}`: active {d.get('sm_active_avg')} / {d.get('sm_active_min')} / "
                         f"{d.get('sm_active_max')} of {d.get('sm_elapsed')} elapsed")
        lines.append("")
    if os.path.exists(lau):
        L = ncu_summary.launches(lau)
        with open(os.path.join(out, f"{a.tag}_launches.csv"), "w") as f:
            f.write("id,kernel,gpu__time_duration.sum_ns,dram__bytes_read.sum,dram__bytes_write.sum\n")
            for x in L:
                f.write(f"{x['id']},\"{x['kernel']}\",{x.get('gpu__time_duration.sum')},"
                        f"{x.get('dram__bytes_read.sum')},{x.get('dram__bytes_write.sum')}\n")
        by = collections.defaultdict(list)
        for x in L:
            name = x["kernel"].replace("void ", "").replace("cats::", "").split("<")[0]
            by[name].append(x)
        lines += ["## Launch list (decode + dense steps)", "",
                  "| kernel | launches | median time (us) | median DRAM read (MB) | median DRAM write (MB) |",
                  "|---|---|---|---|---|"]
        for name, xs in by.items():
            lines.append(f"| `{name}` | {len(xs)} | {statistics.median(x['gpu__time_duration.sum'] for x in xs) / 1e3:.2f} | "
                         f"{statistics.median(x['dram__bytes_read.sum'] for x in xs) / 1e6:.2f} | "
                         f"{statistics.median(x['dram__bytes_write.sum'] for x in xs) / 1e6:.3f} |")
        # dominant kernel traffic per launch: the CATS decode launches of K12 (not the dense ones)
        # (gate-only calibration launches read ~1/3, dense launches all of the layer; the decode
        # launches sit in between)
        k12 = [x for x in by.get("k12_cats_mlp", [])]
        if k12:
            mx = max(x["dram__bytes_read.sum"] for x in k12)
            dec = [x for x in k12 if 0.45 * mx < x["dram__bytes_read.sum"] < 0.9 * mx]
            if dec:
                traffic["K12"] = statistics.median(x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in dec)
                lines.append(f"K12 CATS-decode launches: {len(dec)}, median DRAM traffic {traffic['K12'] / 1e6:.2f} MB "
                             f"per launch, median time {statistics.median(x['gpu__time_duration.sum'] for x in dec) / 1e3:.2f} us")
        lines.append("")
    for item in a.extra:
        label, path = item.split("::", 1)
        if not os.path.exists(path):
            continue
        data = ncu_summary.raw(path)
        lines += [f"## Full-set capture: {label}", "",
                  "| kernel | duration | DRAM read | DRAM write | regs | dyn smem | grid x block | top stalls |",
                  "|---|---|---|---|---|---|---|---|"]
        for d in data:
            lines.append(f"| `{d['kernel']}` | {d.get('dur')} {d.get('dur_unit')} | {d.get('dram_rd')} "
                         f"{d.get('dram_rd_unit')} | {d.get('dram_wr')} {d.get('dram_wr_unit')} | {d.get('regs')} | "
                         f"{d.get('dyn_smem')} {d.get('dyn_smem_unit')} | {d.get('grid')} x {d.get('block')} | "
                         f"{', '.join(f'{n} {v}' for v, n in d['stalls'][:4])} |")
            name = "KA" if "ka_gate_up" in d["kernel"] else "KB" if "kb_down" in d["kernel"] else None
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            if name and "b=2" in label and isinstance(d.get("dram_rd"), float):
                traffic[f"{name}_b2"] = d["dram_rd"] * scale.get(d.get("dram_rd_unit"), 1) + \
                    d["dram_wr"] * scale.get(d.get("dram_wr_unit"), 1)
        lines.append("")
    if a.bench and os.path.exists(a.bench):
        for ln in open(a.bench):
            if ln.startswith("{"):
                lines += ["## bench.py line of the same build", "", "```", ln.strip(), "```", ""]
    with open(os.path.join(out, f"{a.tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic:
        with open(os.path.join(out, "ncu_traffic.json"), "w") as f:
            json.dump(traffic, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
