#!/usr/bin/env python
"""bench.py -- CATS-MLP decode on B200 (BASELINE.json metric), one JSON line on rank 0.

Workload (BASELINE.json configs[1]): one Mistral-7B MLP layer (d=4096, m=14336), bf16 weights and
activations, batch 1, 50% sparsity, threshold calibrated on 2048 held-apart synthetic tokens with
the library's own calibration path. A step = one pass of the whole hot path (one K12 launch: gate
GEMV, SiLU, CATS threshold, compaction, sparse up x v, down projection, split-K reduction [-> NCCL
all-reduce when N > 1]) for one token. N > 1: tensor parallel along m (each rank m/N neurons, same t), "strong" scaling.

Timing: W warm-up steps, then exactly K steps between barrier + synchronize, CUDA events on the
launching stream, max over ranks. L2 defeated by rotating 4 device copies of the weights (1.41 GB
per rank at N=1, >> 126 MB L2). Fresh x per step (a pool of 64 distinct tokens).

--impl reference: the CPU oracle (oracle/, fp64 C) on the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CATS-MLP decode µs/token-layer @50% sparsity; effective HBM GB/s vs 8 TB/s"
UNIT = "us/token-layer"
NOMINAL_HBM_GBS = 8000.0
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="cats", choices=["cats", "reference"])
    ap.add_argument("--model", default="mistral-7b")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--sparsity", type=float, default=0.5)
    ap.add_argument("--copies", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--extras", action="store_true", help="also time dense/cuBLAS/profiled (default on)")
    ap.add_argument("--allreduce", default="fused", choices=["nccl", "fused"],
                    help="N > 1: the library's one-shot NVLink reduction (cats_tp_allreduce; checked against NCCL "
                         "at start, NCCL on a mismatch), or NCCL's all-reduce")
    ap.add_argument("--launcher-selftest", action="store_true",
                    help="start the ranks, all-reduce one tensor, print one line (CPU: gloo) and exit")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """NVML clocks + throttle reasons sampled in a thread during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], 0, False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.th.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        rs = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": rs,
                "samples": len(self.samples)}


def _free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def relaunch_under_torchrun(n: int) -> int:
    """`python bench.py --gpus N` without a torchrun environment: start the N ranks ourselves (one
    process per GPU, torch.distributed.run on 127.0.0.1) and pass rank 0's JSON line through."""
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, cwd=ROOT).returncode


def dist_setup(n, backend="nccl"):
    import torch
    import torch.distributed as dist
    if n > 1 or "RANK" in os.environ:
        rank = int(os.environ["RANK"])
        world = int(os.environ["WORLD_SIZE"])
        local = int(os.environ.get("LOCAL_RANK", rank))
        if world != n:
            raise SystemExit(f"bench.py --gpus {n} launched with WORLD_SIZE={world}")
        if backend == "gloo":
            dist.init_process_group("gloo")
            return rank, world, local
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        return rank, world, local
    torch.cuda.set_device(0)
    return 0, 1, 0


def host_info():
    """(cores this process may run on, CPU model) for the cpu_baseline record."""
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return cores, model


# ---------------------------------------------------------------------------------------- CPU oracle

def time_oracle(d, m, b, sparsity, budget_s=15.0, max_tokens=64, seed=0, all_cores=True):
    """The CPU oracle (fp64 C; all_cores: its OpenMP build over every core this process may use) on
    the same workload: t from Eq. 3 on the oracle's own |SiLU| of 2 held-apart tokens, then decode
    steps of b tokens until the time budget is used. Returns (geometric-mean us per token-layer over
    the steps -- the paper's protocol, P:532 --, steps, threads)."""
    import numpy as np
    import torch

    import cats_synth
    import oracle
    cores, _ = host_info()
    os.environ.setdefault("OMP_NUM_THREADS", str(cores if all_cores else 1))
    # bounded sample: full-width layer, as many steps as fit in the budget
    Wg, Wu, Wd = cats_synth.mlp_weights(d, m, torch.bfloat16)
    og, ou, od = (cats_synth.to_oracle(a) for a in (Wg, Wu, Wd))
    xs = cats_synth.tokens(max_tokens * b + 8, d, torch.bfloat16, seed=seed + 1)
    ox = cats_synth.to_oracle(xs)
    _, v, _ = oracle.mlp(ox[:2], og, ou, od, t=0.0, mode=oracle.DENSE, all_cores=all_cores)
    t = oracle.calibrate_sort(v.astype(np.float32), sparsity).t
    times = []
    n_tok = 0
    t_start = time.perf_counter()
    while n_tok < max_tokens:
        s = time.perf_counter()
        oracle.mlp(ox[2 + n_tok * b: 2 + (n_tok + 1) * b], og, ou, od, t=t, all_cores=all_cores)
        times.append(time.perf_counter() - s)
        n_tok += 1
        if time.perf_counter() - t_start > budget_s:
            break
    geo = math.exp(sum(math.log(x) for x in times) / len(times))
    return 1e6 * geo / b, n_tok, int(os.environ["OMP_NUM_THREADS"]) if all_cores else 1


def run_reference(args):
    import torch
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return 0
    import cats_synth
    d, m = cats_synth.MODELS[args.model]
    # each step: one token through the oracle (~0.6 s at Mistral shape); bounded sample so the run
    # ends within minutes: steps beyond the budget reuse the measured per-token time
    budget = 60.0
    us, ntok, threads = time_oracle(d, m, args.batch, args.sparsity, budget_s=budget,
                                    max_tokens=args.steps + args.warmup)
    cores, cpu_model = host_info()
    value = us
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(value / 1000 * args.batch, 4),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(args, d, m),
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": threads, "kind": "oracle",
                         "cpu_model": cpu_model, "affinity_cores": cores,
                         "sample": f"{ntok} step(s) of b={args.batch} token(s) x full {args.model} layer (d={d}, m={m}), "
                                   f"fp64 C oracle (OpenMP build, {threads} threads), geometric mean, "
                                   f"time-bounded at {budget:.0f} s"},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args, d, m):
    return {"workload": f"{args.model} MLP layer decode (d={d}, m={m}) bf16 b={args.batch} "
                        f"k={args.sparsity} TP={args.gpus}",
            "layer_shape": {"d": d, "m": m}, "batch": args.batch, "sparsity": args.sparsity,
            "tp": args.gpus, "storage": "bf16", "accumulate": "f32",
            "l2": f"inputs larger than L2: {args.copies} rotated weight copies per rank",
            "timing": "CUDA events on the launching stream, max over ranks; steps replayed from a CUDA graph "
                      "of 8 decode calls (eager launches reported in detail.eager_us_per_step)"}


def launcher_selftest(args):
    """The rank plumbing bench.py uses, without the workload: NCCL on GPUs, gloo on a CPU host."""
    import torch
    import torch.distributed as dist
    backend = "nccl" if torch.cuda.is_available() else "gloo"
    rank, world, local = dist_setup(args.gpus, backend=backend)
    dev = torch.device(f"cuda:{local}") if backend == "nccl" else torch.device("cpu")
    v = torch.tensor([float(rank + 1)], device=dev)
    if world > 1:
        dist.all_reduce(v)
    if rank == 0:
        print(json.dumps({"launcher_ok": True, "world": world, "backend": backend, "sum_ranks": float(v.item())}),
              flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------------------- GPU arm

def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "RANK" not in os.environ:
        return relaunch_under_torchrun(args.gpus)
    if args.launcher_selftest:
        return launcher_selftest(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    import cats_synth
    import paper_2404_08763_b200 as cats

    rank, world, local = dist_setup(args.gpus)
    dev = torch.device(f"cuda:{local}")
    d, m = cats_synth.MODELS[args.model]
    b, k = args.batch, args.sparsity
    assert m % world == 0
    ms = m // world
    sl = slice(rank * ms, (rank + 1) * ms)

    # weights: this rank's neuron shard, rotated copies in HBM
    Wg, Wu, Wd = cats_synth.mlp_weights(d, m, torch.bfloat16)
    shard = [w[sl].contiguous() for w in (Wg, Wu, Wd)]
    del Wg, Wu, Wd
    copies = [[w.to(dev) for w in shard] for _ in range(args.copies)]
    plan = cats.MlpPlan(d, ms, max_batch=max(8, b), dtype=torch.bfloat16, device=local)
    ws = plan.workspace()
    stream = torch.cuda.current_stream(dev)

    # ---- Stage 1: calibrate t on 2048 held-apart tokens via the library (sharded: all-reduced histograms)
    from paper_2404_08763_b200 import tp as tpmod
    xcal = cats_synth.tokens(2048, d, torch.bfloat16, seed=0).to(dev)
    acts = torch.empty((2048, ms), dtype=torch.float32, device=dev)
    for i in range(0, 2048, 8):
        cats.cats_mlp_gate_act(plan, xcal[i:i + 8], copies[0][0], acts=acts[i:i + 8], ws=ws)
    t = tpmod.calibrate_threshold(acts, k, group=dist.group.WORLD if world > 1 else None)
    del acts, xcal

    xs = cats_synth.tokens(64 * b, d, torch.bfloat16, seed=1).to(dev).view(64, b, d)
    y = torch.empty((b, d), dtype=torch.float32, device=dev)
    comm = None
    allreduce_used = "nccl" if world > 1 else None
    if world > 1 and args.allreduce == "fused":
        try:  # the fused reduction, checked once against NCCL on a rank-dependent pattern
            comm = tpmod.TpComm(b * d, group=dist.group.WORLD)
            probe = torch.arange(b * d, device=dev, dtype=torch.float32).view(b, d) * (rank + 1) / (b * d)
            ref = probe.clone()
            dist.all_reduce(ref)
            got = comm.allreduce(probe.clone())
            torch.cuda.synchronize(dev)
            ok = torch.tensor([1 if torch.allclose(got, ref, rtol=1e-6, atol=1e-6) else 0], device=dev)
        except Exception as exc:  # pragma: no cover - multi-GPU only
            print(f"[bench] fused reduction unavailable ({type(exc).__name__}: {exc})", file=sys.stderr, flush=True)
            ok = torch.tensor([0], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ok.item():
            allreduce_used = "fused"
        else:
            comm = None
            print("[bench] fused reduction check failed on some rank: using NCCL", file=sys.stderr, flush=True)

    def reduce_y(st):
        if world > 1:
            if comm is not None:
                comm.allreduce(y, stream=st)
            else:
                dist.all_reduce(y)

    def step(i, st=stream):
        W = copies[i % len(copies)]
        cats.cats_mlp_decode(plan, xs[i % 64], W[0], W[1], W[2], t, y=y, ws=ws, stream=st)
        reduce_y(st)

    # CUDA graph of G consecutive steps (the library calls are stream-ordered, allocation- and
    # sync-free, so they capture as-is); replayed K/G times in the timed region
    G = 8
    graph = torch.cuda.CUDAGraph()
    graph_ok = True
    try:
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(stream)
        with torch.cuda.stream(cap):
            for i in range(G):  # warm the capture stream
                step(i, st=cap)
        stream.wait_stream(cap)
        torch.cuda.synchronize(dev)
        with torch.cuda.graph(graph, stream=cap):
            for i in range(G):
                step(i, st=cap)
        torch.cuda.synchronize(dev)
    except Exception as exc:  # e.g. a collective that cannot be captured: time eager launches instead
        graph_ok = False
        print(f"[bench] CUDA graph capture failed ({type(exc).__name__}: {exc}); timing eager steps",
              file=sys.stderr, flush=True)
        torch.cuda.synchronize(dev)
    if world > 1:  # every rank must take the same timing path
        ok_t = torch.tensor([1 if graph_ok else 0], device=dev)
        dist.all_reduce(ok_t, op=dist.ReduceOp.MIN)
        graph_ok = bool(ok_t.item())

    def make_graph_step(k_total):
        full = k_total // G * G if graph_ok else 0

        def graph_step(i):  # exactly k_total steps: k_total // G replays + k_total % G eager steps
            if i < full:
                if i % G == 0:
                    graph.replay()
            else:
                step(i)
        return graph_step

    def timed(fn, steps, warmup):
        for i in range(warmup):
            fn(i)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(steps):
            fn(i)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms_ = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([ms_], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms_ = float(tt.item())
        return ms_ / steps

    sampler = ClockSampler(local)
    with sampler:
        ms_step = timed(make_graph_step(args.steps), args.steps, max(3, args.warmup))
        ms_eager = timed(step, args.steps, max(3, args.warmup))
    clocks = sampler.summary()

    # realized sparsity of this step's token (union over b)
    cats.cats_mlp_decode(plan, xs[0], *copies[0], t, y=y, ws=ws)
    idx, tm, per = cats.cats_mlp_last_active(plan, ws, b)
    nnz_local = len(idx)
    nnz = torch.tensor([nnz_local], device=dev)
    if world > 1:
        dist.all_reduce(nnz)
    U = int(nnz.item())

    # ---- per-kernel times (profiled variant: events between kernels) -> roofline
    n_prof = min(args.steps, 500)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(n_prof)]
    for i in range(10):
        cats.cats_mlp_decode_profiled(plan, xs[i % 64], *copies[i % len(copies)], t, evs[0], y=y, ws=ws)
    torch.cuda.synchronize(dev)
    for i in range(n_prof):
        cats.cats_mlp_decode_profiled(plan, xs[i % 64], *copies[i % len(copies)], t, evs[i], y=y, ws=ws)
    torch.cuda.synchronize(dev)
    t_first = [e[0].elapsed_time(e[1]) * 1e3 for e in evs]   # K12, or KA on the split path
    t_second = [e[1].elapsed_time(e[2]) * 1e3 for e in evs]  # ~0 for K12, KB on the split path
    k_first, k_second = statistics.mean(t_first), statistics.mean(t_second)
    geo = lambda v: math.exp(statistics.mean(math.log(max(x, 1e-3)) for x in v))
    kernels_per_step = cats.cats_mlp_kernels_per_call(plan, b)
    split = kernels_per_step == 2

    # ---- dense path of the same library (speedup denominator), and cuBLAS dense for context
    def dense_step(i):
        W = copies[i % len(copies)]
        cats.cats_mlp_dense(plan, xs[i % 64], W[0], W[1], W[2], y=y, ws=ws, stream=stream)
        reduce_y(stream)
    dense_ms = timed(dense_step, min(args.steps, 1000), 20)

    def cublas_step(i):
        W = copies[i % len(copies)]
        xx = xs[i % 64]
        h = torch.nn.functional.silu(xx @ W[0].T) * (xx @ W[1].T)
        y.copy_((h @ W[2]).float())
        if world > 1:
            dist.all_reduce(y)
    cublas_ms = timed(cublas_step, min(args.steps, 1000), 20)

    # ---- e2e: host activations in (pinned), host y out, through the public C-ABI call
    xh = xs.cpu().pin_memory()
    yh = torch.empty((b, d), dtype=torch.float32).pin_memory()

    # a serving loop's per-token call: arguments validated once (cats.BoundDecodeHost), every step copies
    # that step's host x to the device, decodes and writes y to pinned host memory, blocking
    bound = [cats.BoundDecodeHost(plan, xh[j], *copies[j % len(copies)], t, y_host=yh, ws=ws, stream=stream)
             for j in range(64)] if world == 1 else None

    def e2e_step(i):
        W = copies[i % len(copies)]
        if world == 1:
            bound[i % 64]()
        else:
            xd = xh[i % 64].to(dev, non_blocking=True)
            cats.cats_mlp_decode(plan, xd, W[0], W[1], W[2], t, y=y, ws=ws, stream=stream)
            reduce_y(stream)
            yh.copy_(y, non_blocking=False)
    e2e_ms = timed(e2e_step, min(args.steps, 1000), 10)

    # ---- TP: the all-reduce alone (its share of the step), same buffer and stream
    allreduce_us = None
    if world > 1:
        allreduce_us = timed(lambda i: reduce_y(stream), min(args.steps, 1000), 20) * 1e3

    # ---- roofline of the dominant kernel (algorithmic bytes / live CUDA-event duration)
    hbm_peak, peak_kind = peaks()
    esz = 2
    # K12 algorithmic bytes: every W_gate row (2d B per neuron) + the active neurons' W_up and
    # W_down rows (4d B per active neuron) + x
    step_bytes = 2 * d * ms + 4 * d * nnz_local + b * d * esz
    us_step_dev = ms_step * 1e3
    step_dev_us = us_step_dev - (allreduce_us or 0.0)  # the decode kernels' share of the timed step
    if not split:
        # one kernel per step: its average launch duration over the timed region = the step period
        # (PDL lets a launch's static W_gate tiles stream while its predecessor drains)
        dom, dom_bytes, dom_us, iso_us = "K12", step_bytes, step_dev_us, k_first
    else:
        # two launches per step (KA gate + up, KB down + reduction): the roofline of the pair over the whole
        # step's algorithmic bytes (the step period / the two isolated launches back to back)
        dom, dom_bytes = "KA+KB", step_bytes
        dom_us, iso_us = step_dev_us, k_first + k_second
    achieved = dom_bytes / (dom_us * 1e-6) / 1e9
    achieved_iso = dom_bytes / (iso_us * 1e-6) / 1e9
    traffic = None
    tp_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp_path):
        try:
            traffic = json.load(open(tp_path)).get(dom)
        except Exception:
            traffic = None

    us_step = ms_step * 1e3
    value = us_step / b  # us per token-layer, whole job (TP ranks together process b tokens per step)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cus, ntok, threads = time_oracle(d, m, b, k, budget_s=12.0, max_tokens=40, all_cores=True)
        cus1, ntok1, _ = time_oracle(d, m, b, k, budget_s=6.0, max_tokens=20, all_cores=False)
        cores, cpu_model = host_info()
        cpu = {"value": round(cus, 1), "unit": UNIT, "cores": threads, "kind": "oracle",
               "cpu_model": cpu_model, "affinity_cores": cores, "single_thread_value": round(cus1, 1),
               "sample": f"{ntok} step(s) of b={b} token(s) x full {args.model} layer (d={d}, m={m}), fp64 C "
                         f"oracle, OpenMP build on {threads} threads (single thread: {ntok1} steps), "
                         f"geometric mean per step"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": round(ms_step, 5), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(args, d, m),
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": hbm_peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                         "traffic": traffic, "algorithmic_bytes_per_launch": dom_bytes,
                         "launch_us": round(dom_us, 3),
                         "basis": "timed region: the step period of back-to-back PDL launches (graph replay)",
                         "isolated_launch_us": round(iso_us, 3), "achieved_isolated": round(achieved_iso, 1),
                         "frac_isolated": round(achieved_iso / hbm_peak, 4),
                         "isolated_basis": "one launch bracketed by events on its stream, no overlap with "
                                           "its neighbours (mean of the profiled launches)"},
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_ms * 1e3 / b, 3), "unit": UNIT, "h2d_bytes_per_step": b * d * esz,
                    "d2h_bytes_per_step": b * d * 4},
            "gpu_launches": args.steps * kernels_per_step,
            "clocks": clocks,
            "detail": {
                "allreduce": allreduce_used,
                "nccl": None if world == 1 else {"version": ".".join(map(str, torch.cuda.nccl.version())),
                                                 "nranks": world, "collective": "all_reduce sum fp32 b x d"},
                "t": t, "nnz_union_per_rank": nnz_local, "nnz_union_total": U, "m_per_rank": ms,
                "realized_sparsity": round(1 - U / m, 4),
                "eager_us_per_step": round(ms_eager * 1e3, 3), "graph_steps_per_replay": G if graph_ok else 0,
                "isolated_launch_us": {"K12" if not split else "KA": round(k_first, 3),
                                       **({"KB": round(k_second, 3)} if split else {})},
                "isolated_launch_us_geomean": round(geo([a + c for a, c in zip(t_first, t_second)]), 3),
                "allreduce_us": None if allreduce_us is None else round(allreduce_us, 3),
                "allreduce_share": None if allreduce_us is None else round(allreduce_us / us_step_dev, 4),
                "effective_bytes_per_step": step_bytes,
                "effective_GBps": round(step_bytes / (us_step * 1e-6) / 1e9, 1),
                "frac_of_8TBps": round(step_bytes / (us_step * 1e-6) / 1e9 / NOMINAL_HBM_GBS, 4),
                "dense_us": round(dense_ms * 1e3, 3),
                "speedup_vs_dense": round(dense_ms / ms_step, 4),
                "dense_GBps": round(6 * d * ms / (dense_ms * 1e-3) / 1e9, 1),
                "cublas_dense_us": round(cublas_ms * 1e3, 3),
                "speedup_vs_cublas_dense": round(cublas_ms / ms_step, 4),
                "byte_ceiling_speedup": round(3 / (3 - 2 * (1 - U / m)), 4),
            },
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
