"""GPU parity of the App. B input-sparse projection (cats_xsparse_gemv) vs oracle.xsparse_gemv.

y = CATS_t(x) W with W input-major (Eq. 4 applied to x itself, reading R14). The keep
decision |x_i| >= t compares two exactly representable values on both sides, so the kept set must be
bit-exact (no band); y within rel-L2 2e-3 of the fp64 oracle (BASELINE north_star tolerance).
"""
import numpy as np
import pytest
import torch

import cats_synth
import oracle
import paper_2404_08763_b200 as cats

pytestmark = pytest.mark.gpu

Y_TOL = 2e-3


def _rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _t_for(x_cal, k):
    """Eq. 3 on |x| of calibration tokens (the oracle's order statistic; a value of x's dtype)."""
    return float(oracle.calibrate_sort(cats_synth.to_oracle(x_cal).ravel(), k).t) if k > 0 else 0.0


def run_xsparse(d_in, d_out, b, dtype, k, seed=0, heavy=False, num_sms=0, plan_b=None):
    W = cats_synth.attn_weights(d_in, d_out, dtype, layer=seed)
    x = cats_synth.tokens(b, d_in, dtype, seed=1 + seed, heavy=heavy)
    t = _t_for(cats_synth.tokens(16, d_in, dtype, seed=100 + seed, heavy=heavy), k)
    y_ref, keep_ref = oracle.xsparse_gemv(cats_synth.to_oracle(x), cats_synth.to_oracle(W), t)
    plan = cats.XsparsePlan(d_in, d_out, max_batch=plan_b or b, dtype=dtype, num_sms=num_sms)
    ws = plan.workspace()
    dx, dW = x.cuda(), W.cuda()
    y = cats.cats_xsparse_gemv(plan, dx, dW, t, ws=ws)
    torch.cuda.synchronize()
    idx, tm, per = cats.cats_mlp_last_active(plan, ws, b)
    assert (np.diff(idx) > 0).all()
    keep = np.zeros((b, d_in), np.uint8)
    for tk in range(b):
        keep[tk, idx[((tm >> tk) & 1).astype(bool)]] = 1
    assert (keep == keep_ref).all(), f"{int((keep != keep_ref).sum())} kept-input mismatches"
    assert (keep.sum(1) == per).all()
    yg = y.cpu().numpy().astype(np.float64)
    for i in range(b):
        if np.abs(y_ref[i]).max() == 0:
            assert np.abs(yg[i]).max() == 0
        else:
            assert _rel_l2(yg[i], y_ref[i]) <= Y_TOL, (i, _rel_l2(yg[i], y_ref[i]))
    return plan, ws, dx, dW, t, y, keep


@pytest.mark.parametrize("d_in,d_out,b,dtype,k", [
    (64, 64, 1, torch.float32, 0.5),           # one tile row of KB parts
    (1001, 264, 3, torch.float32, 0.5),        # ragged d_in (last tile of 1), d_out in 3 column parts
    (1001, 264, 3, torch.bfloat16, 0.7),
    (4096, 6144, 1, torch.bfloat16, 0.5),      # Mistral-7B q|k|v (4096 + 2 x 1024): FFMA, 3 parts
    (4096, 6144, 2, torch.bfloat16, 0.5),
    (4096, 6144, 4, torch.bfloat16, 0.5),      # MMA, 6 parts of 1024 columns
    (4096, 6144, 8, torch.bfloat16, 0.7),
    (4096, 12288, 1, torch.bfloat16, 0.5),     # Llama2-7B q|k|v (3 x 4096)
    (4096, 12288, 5, torch.bfloat16, 0.5),
    (4096, 4096, 8, torch.bfloat16, 0.9),      # o_proj-sized
    (5120, 5120, 3, torch.bfloat16, 0.5),      # Llama2-13B width
    (5120, 5120, 6, torch.bfloat16, 0.5),
    (2048, 2048, 7, torch.float32, 0.5),
])
def test_xsparse_parity(d_in, d_out, b, dtype, k):
    run_xsparse(d_in, d_out, b, dtype, k)


@pytest.mark.parametrize("b", [1, 4])
def test_xsparse_heavy_tails(b):
    run_xsparse(4096, 6144, b, torch.bfloat16, 0.5, seed=3, heavy=True)


def test_xsparse_t0_is_dense_gemv_and_deterministic():
    plan, ws, dx, dW, _, y, keep = run_xsparse(4096, 6144, 4, torch.bfloat16, 0.0)
    assert keep.all()  # |x_i| >= 0 always: every input kept (ties kept, reading G1)
    y_dense = (dx.double() @ dW.double()).cpu().numpy()
    assert _rel_l2(y.cpu().numpy().astype(np.float64), y_dense) <= Y_TOL
    y2 = cats.cats_xsparse_gemv(plan, dx, dW, 0.0, ws=ws)
    torch.cuda.synchronize()
    assert torch.equal(y, y2)


def test_xsparse_nothing_kept_gives_zero():
    plan = cats.XsparsePlan(4096, 6144, max_batch=2)
    ws = plan.workspace()
    x = cats_synth.tokens(2, 4096, torch.bfloat16, seed=1).cuda()
    W = cats_synth.attn_weights(4096, 6144).cuda()
    y = cats.cats_xsparse_gemv(plan, x, W, 1e6, ws=ws)
    torch.cuda.synchronize()
    assert torch.count_nonzero(y) == 0
    idx, _, _ = cats.cats_mlp_last_active(plan, ws, 2)
    assert len(idx) == 0
    # and the workspace is left clean for the next, non-empty call
    run = cats.cats_xsparse_gemv(plan, x, W, 0.5, ws=ws)
    torch.cuda.synchronize()
    y_ref, _ = oracle.xsparse_gemv(cats_synth.to_oracle(x.cpu()), cats_synth.to_oracle(W.cpu()), 0.5)
    assert _rel_l2(run.cpu().numpy().astype(np.float64), y_ref) <= Y_TOL


def test_xsparse_mixed_batches_one_workspace():
    d_in, d_out = 4096, 6144
    plan = cats.XsparsePlan(d_in, d_out, max_batch=8)
    ws = plan.workspace()
    W = cats_synth.attn_weights(d_in, d_out)
    dW = W.cuda()
    for b in (3, 8, 1, 5, 2, 8, 1):
        x = cats_synth.tokens(b, d_in, seed=b)
        y = cats.cats_xsparse_gemv(plan, x.cuda(), dW, 0.6, ws=ws)
        torch.cuda.synchronize()
        y_ref, _ = oracle.xsparse_gemv(cats_synth.to_oracle(x), cats_synth.to_oracle(W), 0.6)
        for i in range(b):
            assert _rel_l2(y[i].cpu().numpy().astype(np.float64), y_ref[i]) <= Y_TOL, (b, i)


def test_xsparse_plan_kinds_are_not_interchangeable():
    xp = cats.XsparsePlan(4096, 6144, max_batch=1)
    mp = cats.MlpPlan(4096, 14336, max_batch=1)
    x = torch.zeros(1, 4096, dtype=torch.bfloat16, device="cuda")
    W = torch.zeros(4096, 6144, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(cats.CatsError, match="UNSUPPORTED"):
        cats.cats_xsparse_gemv(mp, x, W, 0.1, ws=mp.workspace())
    with pytest.raises(cats.CatsError, match="UNSUPPORTED"):
        cats.cats_mlp_decode(xp, x, W, W, W, 0.1, ws=xp.workspace())
