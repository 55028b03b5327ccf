"""Multi-process (world_size 2, gloo, CPU) tests of the tensor-parallel host logic:
  * sharded calibration: per-rank histograms (numpy stand-in for the device pass) all-reduced between
    cats_calib_step calls give the SAME t on every rank, equal to the oracle's t of the union;
  * sharded decode: summing per-rank partial MLP outputs over an m-split (the all-reduce) equals the
    unsharded result, with the layer-global t needing no communication.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import cats_synth
import oracle
from paper_2404_08763_b200 import tp
from tests.test_boundary import emulated_pass


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # pragma: no cover - surfaced to the parent
        q.put((rank, e))
    finally:
        dist.destroy_process_group()


def run_ranks(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return [out[r] for r in range(world)]


N_CAL = 3_000_001


def _calib_rank(rank, world):
    acts = cats_synth.calib_acts(N_CAL, torch.bfloat16, seed=5, heavy=True)
    sl = tp.shard_rows(N_CAL - 1, world, rank)     # even split of the first N-1, last value to rank 0
    mine = acts[sl]
    if rank == 0:
        mine = torch.cat([mine, acts[-1:]])
    res = {}
    for k in (0.0, 0.5, 0.7, 0.9):
        res[k] = tp.calibrate_threshold(mine.contiguous(), k, group=dist.group.WORLD,
                                        hist_fn=lambda a, w: emulated_pass(cats_synth.to_oracle(a), w))
    return res


def test_sharded_calibration_same_t_on_all_ranks():
    outs = run_ranks(_calib_rank)
    acts = cats_synth.to_oracle(cats_synth.calib_acts(N_CAL, torch.bfloat16, seed=5, heavy=True))
    for k, t in outs[0].items():
        assert outs[1][k] == t
        ref = oracle.calibrate_bf16_counts(oracle.bf16_counts(acts), k)
        assert t == ref.t, (k, t, ref.t)


D, M, B = 48, 96, 2


def _decode_rank(rank, world):
    Wg, Wu, Wd = cats_synth.mlp_weights(D, M, torch.float32, layer=2)
    x = cats_synth.tokens(B, D, torch.float32, seed=4)
    t = 0.05
    sl = tp.shard_rows(M, world, rank)
    args = [cats_synth.to_oracle(a) for a in (x, Wg[sl], Wu[sl], Wd[sl])]
    y, _, keep = oracle.mlp(*args, t=t)   # stand-in for the rank's cats_mlp_decode (CPU test)
    yt = torch.from_numpy(y)
    dist.all_reduce(yt)                    # the one exchange step of the TP path
    return yt.numpy(), keep


def test_sharded_decode_sums_to_unsharded():
    outs = run_ranks(_decode_rank)
    Wg, Wu, Wd = cats_synth.mlp_weights(D, M, torch.float32, layer=2)
    x = cats_synth.tokens(B, D, torch.float32, seed=4)
    y, _, keep = oracle.mlp(*[cats_synth.to_oracle(a) for a in (x, Wg, Wu, Wd)], t=0.05)
    np.testing.assert_allclose(outs[0][0], y, rtol=1e-12, atol=1e-15)
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(np.concatenate([outs[0][1], outs[1][1]], axis=1), keep)


def test_shard_rows():
    assert tp.shard_rows(13824, 8, 7) == slice(12096, 13824)
    with pytest.raises(ValueError):
        tp.shard_rows(10, 4, 0)


def test_bench_launcher_starts_n_ranks():
    """`python bench.py --gpus 2` with no torchrun environment starts its own 2 ranks (torch.distributed.run
    on 127.0.0.1); every rank joins the process group (gloo on a CPU host) and one all-reduce sees both."""
    import json
    import subprocess
    import sys
    from tests.conftest import ROOT
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launcher-selftest"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert lines == [{"launcher_ok": True, "world": 2, "backend": "gloo", "sum_ranks": 3.0}]
