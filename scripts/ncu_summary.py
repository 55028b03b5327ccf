"""Summarise an ncu report (--set full) or launch-list CSV into a compact table / JSON.

    python scripts/ncu_summary.py gpurun_out/r01_prof.ncu-rep [--json out.json]
    python scripts/ncu_summary.py --launches gpurun_out/r01_launches.csv
"""
import argparse
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "dur"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("sm__cycles_active.avg", "sm_active_avg"),
    ("sm__cycles_active.min", "sm_active_min"),
    ("sm__cycles_active.max", "sm_active_max"),
    ("sm__cycles_elapsed.avg", "sm_elapsed"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block_dynamic", "dyn_smem"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "inst"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0][:70]}
        for k, short in KEYS:
            if k in hdr:
                v = r[hdr.index(k)]
                try:
                    v = float(v.replace(",", ""))
                except ValueError:
                    pass
                d[short] = v
                d[short + "_unit"] = units[hdr.index(k)]
        stalls = []
        for i, c in enumerate(hdr):
            if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio"):
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                if v >= 0.2:
                    stalls.append((round(v, 2), c[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        d["stalls"] = sorted(stalls, reverse=True)[:6]
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            o = dict(zip(hdr, r))
            agg.setdefault((int(o["ID"]), o["Kernel Name"].split("(")[0][:60]), {})[o["Metric Name"]] = \
                float(o["Metric Value"].replace(",", ""))
    return [{"id": i, "kernel": n, **m} for (i, n), m in agg.items()]


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("report", nargs="?")
    ap.add_argument("--launches")
    ap.add_argument("--json")
    a = ap.parse_args()
    if a.launches:
        L = launches(a.launches)
        for x in L:
            print(x)
        data = L
    else:
        data = raw(a.report)
        for d in data:
            print(f"{d['kernel']}")
            print(f"   dur={d.get('dur')}{d.get('dur_unit')} dram_rd={d.get('dram_rd')}{d.get('dram_rd_unit')} "
                  f"dram%={d.get('dram_pct')} sm_active avg/min/max={d.get('sm_active_avg')}/{d.get('sm_active_min')}/"
                  f"{d.get('sm_active_max')} elapsed={d.get('sm_elapsed')} regs={d.get('regs')} "
                  f"smem={d.get('dyn_smem')}{d.get('dyn_smem_unit')} grid={d.get('grid')}x{d.get('block')} "
                  f"occ%={d.get('occupancy_pct')}")
            print(f"   stalls: {d['stalls']}")
    if a.json:
        json.dump(data, open(a.json, "w"), indent=1)
