"""GPU tests of the tensor-parallel exchange.

This pool lends ONE GPU, so the P-rank fused reduction is exercised as the library's emulation: one
cooperative launch runs every rank's CTAs over P symmetric buffers on the device (the ranks wait on each
other's flags, so they must be co-resident -- the profiling guide's recipe for fewer GPUs than ranks).
The real (non-emulated) kernel runs with world = 1, and the multi-process NCCL / IPC path runs when the
box has >= 2 GPUs (skipped otherwise)."""
import os
import socket

import numpy as np
import pytest
import torch

import cats_synth
import oracle
import paper_2404_08763_b200 as cats
from paper_2404_08763_b200 import tp
from tests.test_gpu_parity import BAND, Y_TOL, _keep_from_gpu, _rel_l2, oracle_mlp

pytestmark = pytest.mark.gpu


def _seq_sum(xs):
    acc = xs[0].cpu().numpy().astype(np.float32).copy()
    for x in xs[1:]:
        acc = (acc + x.cpu().numpy().astype(np.float32)).astype(np.float32)  # fp32, rank order 0..P-1
    return acc


@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_fused_allreduce_emulated_is_the_fixed_order_sum(P):
    n_max = 8 * 5120
    em = tp.EmulatedTpComms(P, n_max)
    g = torch.Generator(device="cuda").manual_seed(P)
    for call, n in enumerate([4, 5120, 8 * 4096, n_max, 1028, 5120, 5120]):  # epochs + both parity slots
        xs = [torch.randn(n, device="cuda", generator=g) * (r + 1) for r in range(P)]
        ys = [torch.full((n,), float("nan"), device="cuda") for _ in range(P)]
        em.allreduce(xs, ys)
        torch.cuda.synchronize()
        want = _seq_sum(xs)
        for r in range(P):
            assert np.array_equal(ys[r].cpu().numpy(), want), (call, n, r)


def test_fused_allreduce_in_place_and_world1_real_path():
    em = tp.EmulatedTpComms(4, 4096)
    xs = [torch.randn(4096, device="cuda") for _ in range(4)]
    want = _seq_sum(xs)
    em.allreduce(xs)  # in place: y aliases x
    torch.cuda.synchronize()
    assert all(np.array_equal(x.cpu().numpy(), want) for x in xs)
    comm = tp.TpComm(4096)  # world = 1: the non-emulated kernel (IPC export, push to self, flags, sum)
    x = torch.randn(4096, device="cuda")
    for _ in range(3):
        y = comm.allreduce(x, torch.empty_like(x))
        torch.cuda.synchronize()
        assert torch.equal(x, y)


@pytest.mark.parametrize("P,b", [(2, 1), (4, 1), (8, 1), (4, 8)])
def test_tp_decode_with_fused_reduction_emulated(P, b):
    """Llama2-13B (BASELINE config 3) split along m over P emulated ranks: every rank's decode partial, then the
    fused reduction; every rank ends with the same y, equal to the unsharded oracle within the tolerance."""
    d, m = cats_synth.MODELS["llama2-13b"]
    Wg, Wu, Wd = cats_synth.mlp_weights(d, m, torch.bfloat16, layer=P)
    x = cats_synth.tokens(b, d, torch.bfloat16, seed=13 + P)
    ox, og, ou, od = (cats_synth.to_oracle(a) for a in (x, Wg, Wu, Wd))
    zero = np.zeros((m, d), np.uint16)
    _, v64, _ = oracle_mlp(ox, og, zero, zero, 0.0, mode=oracle.DENSE)
    t = float(oracle.calibrate_sort(v64.astype(np.float32), 0.5).t)
    ms = m // P
    ys, keep_gpu = [], np.zeros((b, m), np.uint8)
    for r in range(P):
        sl = tp.shard_rows(m, P, r)
        plan = cats.MlpPlan(d, ms, max_batch=b)
        ws = plan.workspace()
        ys.append(cats.cats_mlp_decode(plan, x.cuda(), Wg[sl].cuda(), Wu[sl].cuda(), Wd[sl].cuda(), t, ws=ws))
        idx, tm, _ = cats.cats_mlp_last_active(plan, ws, b)
        keep_gpu[:, sl] = _keep_from_gpu(idx, tm, b, ms)
    parts = [y.clone() for y in ys]
    em = tp.EmulatedTpComms(P, b * d)
    em.allreduce([y.view(-1) for y in ys])
    torch.cuda.synchronize()
    want = _seq_sum([p.view(-1) for p in parts])
    for r in range(P):
        assert np.array_equal(ys[r].view(-1).cpu().numpy(), want)
    keep64 = (np.abs(v64) >= t).astype(np.uint8)
    band = np.abs(np.abs(v64) - t) <= BAND * t
    assert not ((keep_gpu != keep64) & ~band).any()
    y_ref, _, _ = oracle_mlp(ox, og, ou, od, t, keep_in=np.where(band, keep_gpu, keep64).astype(np.uint8))
    yg = ys[0].cpu().numpy().astype(np.float64)
    assert max(_rel_l2(yg[i], y_ref[i]) for i in range(b)) <= Y_TOL


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _mp_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device(f"cuda:{rank}"))
    try:
        d, m, b = 5120, 13824, 1
        Wg, Wu, Wd = cats_synth.mlp_weights(d, m, torch.bfloat16)
        sl = tp.shard_rows(m, world, rank)
        W = [w[sl].contiguous().cuda() for w in (Wg, Wu, Wd)]
        x = cats_synth.tokens(b, d, torch.bfloat16, seed=3).cuda()
        plan = cats.MlpPlan(d, m // world, max_batch=b, device=rank)
        ws = plan.workspace()
        comm = tp.TpComm(b * d, group=dist.group.WORLD)
        y_nccl = tp.tp_decode(plan, x, *W, 0.1, ws=ws, group=dist.group.WORLD).clone()
        y_fused = tp.tp_decode(plan, x, *W, 0.1, ws=ws, comm=comm).clone()
        torch.cuda.synchronize()
        q.put((rank, y_nccl.cpu().numpy(), y_fused.cpu().numpy()))
    except Exception as e:  # pragma: no cover
        q.put((rank, e, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs (this pool lends one)")
def test_tp_decode_nccl_and_fused_on_real_gpus():
    import torch.multiprocessing as mp
    world = min(torch.cuda.device_count(), 8)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict((r, (a, b)) for r, a, b in (q.get(timeout=600) for _ in procs))
    for p in procs:
        p.join(timeout=60)
    for r, (a, b) in out.items():
        assert not isinstance(a, Exception), a
    fused = [out[r][1] for r in range(world)]
    assert all(np.array_equal(fused[0], f) for f in fused[1:])  # bit-identical on every rank
    assert _rel_l2(fused[0].astype(np.float64), out[0][0].astype(np.float64)) < 1e-6
