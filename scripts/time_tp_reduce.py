"""Cost of the fused TP reduction's protocol on ONE GPU (emulated ranks: one cooperative launch over P
buffers on the device; no NVLink involved): graph-timed per call, vs torch.distributed-free baselines
(a plain device sum of the P partials). JSON lines.

    python scripts/time_tp_reduce.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2404_08763_b200 import tp


def graph_us(fn, reps=200):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(10):
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
    return 1e3 * e0.elapsed_time(e1) / (reps * 10)


comm = tp.TpComm(5120)  # world = 1: the non-emulated kernel (push to self, flag, sum), no cooperative launch
x1 = torch.randn(5120, device="cuda")
y1 = torch.empty_like(x1)
print(json.dumps({"P": 1, "n": 5120, "real_kernel_world1_us": round(graph_us(lambda: comm.allreduce(x1, y1)), 3)}),
      flush=True)
for P in (2, 4, 8):
    for n in (5120, 8 * 5120):
        em = tp.EmulatedTpComms(P, n)
        xs = [torch.randn(n, device="cuda") for _ in range(P)]
        ys = [torch.empty(n, device="cuda") for _ in range(P)]
        us = graph_us(lambda: em.allreduce(xs, ys))
        st = torch.stack(xs)
        out = torch.empty(n, device="cuda")
        us_sum = graph_us(lambda: torch.sum(st, 0, out=out))
        print(json.dumps({"P": P, "n": n, "fused_emulated_us": round(us, 3), "torch_sum_us": round(us_sum, 3)}),
              flush=True)
