"""Pins for the CPU oracle (oracle/) against what the paper and mathematics fix.

None of these compares the oracle with itself or with a retyped copy of its loops: each
check is a worked value printed in the paper/SPEC (tests/golden/, cited), a closed form, a
special case that reduces to a library routine (numpy BLAS, scipy), brute force on tiny
inputs with exact rationals, or an invariant chosen so that a dropped term, a wrong sign,
a wrong index or a transposed operand fails. CPU only.
"""
import math
from fractions import Fraction

import numpy as np
import pytest
import torch

import cats_synth
import oracle
from oracle import brute
from tests.conftest import golden_lines


# ----------------------------------------------------------------------------- SiLU (Eq. 2)

def test_silu_golden_values():
    n = 0
    for line in golden_lines("silu_examples.txt"):
        u, want, tol = (float(s) for s in line.split())
        got = oracle.silu(u)
        assert abs(got - want) <= tol, (u, got, want)
        n += 1
    assert n == 4
    assert 19.9999 <= oracle.silu(20.0) <= 20.0


def test_silu_minimum_is_lambert_w():
    from scipy.optimize import minimize_scalar
    from scipy.special import lambertw
    w = lambertw(1 / math.e).real
    ustar = -(1 + w)
    assert abs(oracle.silu(ustar) + w) < 1e-15
    # it is the minimum: an independent numerical minimiser lands on the same point
    res = minimize_scalar(oracle.silu, bounds=(-5, 0), method="bounded", options={"xatol": 1e-10})
    assert abs(res.x - ustar) < 1e-6


def test_silu_extremes_and_sign():
    assert oracle.silu(800.0) == 800.0
    v = oracle.silu(-800.0)
    assert v == 0.0 and not math.isnan(v)
    for u in np.linspace(-30, 30, 601):
        s = oracle.silu(float(u))
        # sign(SiLU(u)) = sign(u); SiLU(u) <= u for u >= 0 and >= u for u < 0
        assert (s > 0) == (u > 0) or u == 0
        assert (s <= u) if u >= 0 else (s >= u)
        # SiLU(u) - SiLU(-u) = u  (sigmoid(u) + sigmoid(-u) = 1)
        assert abs((s - oracle.silu(float(-u))) - u) <= 1e-12 * max(1.0, abs(u))


# ----------------------------------------------------------------------------- CATS (Eq. 4)

def test_cats_mask_spec_example():
    lines = dict(l.split(None, 1) for l in golden_lines("cats_mask_example.txt"))
    t = float(lines["t"])
    v = np.array([float(s) for s in lines["v"].split()])
    want = [int(s) for s in lines["mask"].split()]
    keep = oracle.cats_mask(v, t)
    assert keep.tolist() == want and keep.sum() == 2
    # ties are kept (Eq. 4 uses >=, reading G1); t = 0 keeps everything, even -0.0
    assert oracle.cats_mask(np.array([0.15, -0.15]), 0.15).tolist() == [1, 1]
    assert oracle.cats_mask(np.array([0.0, -0.0, 1e-300]), 0.0).tolist() == [1, 1, 1]
    assert oracle.cats_mask(np.zeros(5), 0.1).tolist() == [0] * 5


# ----------------------------------------------------------------------------- MLP (Eq. 1/5)

def _np_silu(u):
    return u / (1.0 + np.exp(-u))


def _np_mlp(x, Wg, Wu, Wd, keep=None):
    """Textbook SwiGLU through numpy's BLAS (float64), neuron-major weights."""
    v = _np_silu(x @ Wg.T)
    if keep is not None:
        v = np.where(keep.astype(bool), v, 0.0)
    return (v * (x @ Wu.T)) @ Wd, _np_silu(x @ Wg.T)


def _widen(a):
    if a.dtype == np.uint16:
        return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return a.astype(np.float64)


def _case(d, m, b, dtype, seed=0, heavy=False):
    Wg, Wu, Wd = cats_synth.mlp_weights(d, m, dtype, layer=seed, heavy=heavy)
    x = cats_synth.tokens(b, d, dtype, seed=1 + seed, heavy=heavy)
    return [cats_synth.to_oracle(a) for a in (x, Wg, Wu, Wd)]


def test_scalar_mlp_golden():
    for line in golden_lines("scalar_mlp.txt"):
        x, wg, wu, wd, want = (float(s) for s in line.split())
        args = [np.array([[v]], dtype=np.float32) for v in (x, wg, wu, wd)]
        y, v, keep = oracle.mlp(args[0], *args[1:], t=0.0)
        assert abs(y[0, 0] - want) <= 1e-14 * want
        # threshold just below / above |SiLU(2)| = 1.7615941559557646
        y, _, keep = oracle.mlp(args[0], *args[1:], t=1.76)
        assert keep[0, 0] == 1 and abs(y[0, 0] - want) <= 1e-14 * want
        y, _, keep = oracle.mlp(args[0], *args[1:], t=1.77)
        assert keep[0, 0] == 0 and y[0, 0] == 0.0


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("d,m,b", [(64, 176, 1), (24, 40, 3), (3, 5, 2), (96, 33, 8)])
def test_dense_matches_numpy_blas(dtype, d, m, b):
    x, Wg, Wu, Wd = _case(d, m, b, dtype)
    y, v, keep = oracle.mlp(x, Wg, Wu, Wd, t=0.0, mode=oracle.DENSE)
    y_np, v_np = _np_mlp(*(_widen(a) for a in (x, Wg, Wu, Wd)))
    assert keep.all()
    np.testing.assert_allclose(v, v_np, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(y, y_np, rtol=1e-11, atol=1e-14 * np.abs(y_np).max())


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("k", [0.5, 0.7, 0.9])
def test_cats_matches_numpy_masked(dtype, k):
    d, m, b = 48, 200, 4
    x, Wg, Wu, Wd = _case(d, m, b, dtype, seed=3)
    xs = [_widen(a) for a in (x, Wg, Wu, Wd)]
    _, v_np = _np_mlp(*xs)
    t = float(np.quantile(np.abs(v_np), k))
    y, v, keep = oracle.mlp(x, Wg, Wu, Wd, t=t)
    keep_np = (np.abs(v_np) >= t)
    assert (keep.astype(bool) == keep_np).all()
    assert 0 < keep.sum() < keep.size
    y_np, _ = _np_mlp(*xs, keep=keep_np)
    np.testing.assert_allclose(y, y_np, rtol=1e-11, atol=1e-14 * np.abs(y_np).max())


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_t0_is_dense_bit_exact(dtype):
    x, Wg, Wu, Wd = _case(64, 176, 3, dtype, seed=5)
    y0, v0, k0 = oracle.mlp(x, Wg, Wu, Wd, t=0.0, mode=oracle.SPARSE)
    yd, vd, kd = oracle.mlp(x, Wg, Wu, Wd, t=0.0, mode=oracle.DENSE)
    assert np.array_equal(y0, yd) and np.array_equal(v0, vd) and k0.all()


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("k", [0.3, 0.5, 0.9, 0.99])
def test_masked_dense_equals_sparse_gather_bit_exact(dtype, k):
    x, Wg, Wu, Wd = _case(40, 300, 2, dtype, seed=7)
    _, v, _ = oracle.mlp(x, Wg, Wu, Wd, t=0.0, mode=oracle.DENSE)
    t = float(np.quantile(np.abs(v), k))
    ys, vs, ks = oracle.mlp(x, Wg, Wu, Wd, t=t, mode=oracle.SPARSE)
    ym, vm, km = oracle.mlp(x, Wg, Wu, Wd, t=t, mode=oracle.MASKED)
    assert np.array_equal(ks, km)
    # adding exact zeros in the same ascending order changes nothing (up to the sign of 0)
    assert np.array_equal(ys, ym)


def test_single_active_neuron_closed_form():
    x, Wg, Wu, Wd = _case(32, 50, 1, torch.float32, seed=11)
    _, v, _ = oracle.mlp(x, Wg, Wu, Wd, t=0.0, mode=oracle.DENSE)
    a = np.sort(np.abs(v[0]))
    t = (a[-1] + a[-2]) / 2  # only the largest |v| survives
    y, _, keep = oracle.mlp(x, Wg, Wu, Wd, t=t)
    j = int(np.argmax(np.abs(v[0])))
    assert keep[0].sum() == 1 and keep[0, j] == 1
    xs, wu, wd = _widen(x)[0], _widen(Wu)[j], _widen(Wd)[j]
    want = v[0, j] * float(np.dot(xs, wu)) * wd
    np.testing.assert_allclose(y[0], want, rtol=1e-13, atol=1e-16)
    # t above every |v|: y = 0 and no neuron active
    y, _, keep = oracle.mlp(x, Wg, Wu, Wd, t=float(a[-1]) * 1.0001)
    assert keep.sum() == 0 and not y.any()


def test_power_of_two_scaling_is_exact_and_mask_invariant():
    x, Wg, Wu, Wd = _case(32, 64, 2, torch.float32, seed=13)
    _, v, _ = oracle.mlp(x, Wg, Wu, Wd, t=0.0, mode=oracle.DENSE)
    t = float(np.median(np.abs(v)))
    y, _, keep = oracle.mlp(x, Wg, Wu, Wd, t=t)
    y2, _, keep2 = oracle.mlp(x, Wg, (Wu * 4).astype(np.float32), Wd, t=t)
    y3, _, keep3 = oracle.mlp(x, Wg, Wu, (Wd * 0.5).astype(np.float32), t=t)
    assert np.array_equal(keep, keep2) and np.array_equal(keep, keep3)
    assert np.array_equal(y2, 4 * y) and np.array_equal(y3, 0.5 * y)


def test_neuron_permutation_invariance():
    # catches any mix-up between neuron j of W_gate / W_up / W_down
    x, Wg, Wu, Wd = _case(32, 80, 2, torch.bfloat16, seed=17)
    _, v, _ = oracle.mlp(x, Wg, Wu, Wd, t=0.0, mode=oracle.DENSE)
    t = float(np.quantile(np.abs(v), 0.6))
    y, v, keep = oracle.mlp(x, Wg, Wu, Wd, t=t)
    p = np.random.default_rng(0).permutation(80)
    yp, vp, keepp = oracle.mlp(x, Wg[p], Wu[p], Wd[p], t=t)
    assert np.array_equal(keepp, keep[:, p]) and np.array_equal(vp, v[:, p])
    np.testing.assert_allclose(yp, y, rtol=1e-12, atol=1e-15)
    # swapping roles of W_up and W_down (a transposed-operand bug) must change y
    ys, _, _ = oracle.mlp(x, Wg, Wd, Wu, t=t)
    assert np.abs(ys - y).max() > 1e-3 * np.abs(y).max()


def test_batch_equals_independent_tokens():
    x, Wg, Wu, Wd = _case(40, 120, 5, torch.bfloat16, seed=19)
    _, v, _ = oracle.mlp(x, Wg, Wu, Wd, t=0.0, mode=oracle.DENSE)
    t = float(np.quantile(np.abs(v), 0.5))
    y, v, keep = oracle.mlp(x, Wg, Wu, Wd, t=t)
    for i in range(5):
        yi, vi, ki = oracle.mlp(x[i:i + 1], Wg, Wu, Wd, t=t)
        assert np.array_equal(yi[0], y[i]) and np.array_equal(ki[0], keep[i])


def test_active_sets_monotone_in_t():
    x, Wg, Wu, Wd = _case(32, 200, 2, torch.float32, seed=23)
    prev = None
    for t in [0.0, 0.01, 0.05, 0.1, 0.2, 0.5]:
        _, _, keep = oracle.mlp(x, Wg, Wu, Wd, t=t)
        if prev is not None:
            assert not (keep & ~prev).any()  # active(t2) subset of active(t1) for t1 <= t2
        prev = keep


def test_keep_override_is_used():
    x, Wg, Wu, Wd = _case(16, 30, 1, torch.float32, seed=29)
    keep = np.zeros((1, 30), np.uint8)
    keep[0, [3, 7]] = 1
    y, v, k = oracle.mlp(x, Wg, Wu, Wd, t=0.0, keep_in=keep)
    assert np.array_equal(k, keep)
    want = sum(v[0, j] * float(np.dot(_widen(x)[0], _widen(Wu)[j])) * _widen(Wd)[j] for j in (3, 7))
    np.testing.assert_allclose(y[0], want, rtol=1e-13)


def test_tiny_pure_python_agrees():
    x, Wg, Wu, Wd = _case(6, 9, 1, torch.float32, seed=31)
    xs, g, u, dd = (_widen(a).tolist() for a in (x, Wg, Wu, Wd))
    _, v, _ = oracle.mlp(x, Wg, Wu, Wd, t=0.0, mode=oracle.DENSE)
    t = float(np.median(np.abs(v)))
    y, _, keep = oracle.mlp(x, Wg, Wu, Wd, t=t)
    yb, kb = brute.cats_mlp_tiny(xs[0], g, u, dd, t)
    assert keep[0].tolist() == kb
    np.testing.assert_allclose(y[0], yb, rtol=1e-13, atol=1e-16)


# ----------------------------------------------------------------------------- calibration (Eq. 3)

def test_rank_exact_rational():
    rng = np.random.default_rng(1)
    ks = [0.1, 0.2, 0.25, 0.3, 0.5, 0.7, 0.9, 0.99, 1e-9, 0.999999999]
    for k in ks:
        for n in list(range(1, 200)) + [int(x) for x in rng.integers(1, 2**40, 50)] + [11272192000]:
            assert oracle.rank(k, n) == math.ceil(Fraction(k) * n), (k, n)
    assert oracle.rank(0.1, 10) == 2          # Appendix A.3 disagreeing case
    assert oracle.rank(0.0, 12345) == 0
    assert oracle.rank(0.5, 11272192000) == 5636096000


def test_calibration_golden_examples():
    n = 0
    for line in golden_lines("calibration_examples.txt"):
        k, vals, want = (s.strip() for s in line.split("|"))
        acts = np.array([float(s) for s in vals.split()], dtype=np.float32)
        res = oracle.calibrate_sort(acts, float(k))
        assert res.t == float(np.float32(float(want))), (line, res)
        assert res.t == brute.fit_threshold(acts.astype(np.float64), float(k))
        n += 1
    assert n == 5
    # S:218
    assert brute.empirical_cdf([0.05, 0.1, 0.2, 0.3], 0.1) == Fraction(1, 2)


def _check_invariant(res, k):
    # count_lt < k N <= count_le  (exact integers / rationals; reading G16)
    kN = Fraction(k) * res.n
    if res.r == 0:
        assert res.t == 0.0
    else:
        assert res.count_lt < kN <= res.count_le


@pytest.mark.parametrize("dtype", [np.float32, np.uint16])
def test_calibrate_sort_vs_bruteforce(dtype):
    rng = np.random.default_rng(2)
    for it in range(100):
        n = int(rng.integers(1, 150))
        if dtype == np.uint16:
            vals = torch.from_numpy(rng.normal(0, 0.3, n).astype(np.float32)).to(torch.bfloat16)
            if it % 3 == 0:   # heavy ties
                vals = torch.from_numpy(rng.integers(-3, 4, n).astype(np.float32) / 8).to(torch.bfloat16)
            acts = cats_synth.bf16_bits(vals)
        else:
            acts = rng.normal(0, 1, n).astype(np.float32)
            if it % 4 == 0:
                acts = np.round(acts * 2).astype(np.float32) / 2   # ties incl. -0.0
        wide = _widen(acts)
        for k in [0.0, 0.25, 0.5, 0.7, 0.9]:
            res = oracle.calibrate_sort(acts, k)
            assert res.t == brute.fit_threshold(wide, k), (it, k)
            assert res.r == brute.rank_exact(k, n)
            _check_invariant(res, k)
            mags = np.abs(wide)
            assert res.count_lt == int((mags < res.t).sum()) and res.count_le == int((mags <= res.t).sum())


def test_calibration_monotone_in_k():
    acts = cats_synth.to_oracle(cats_synth.calib_acts(20000, torch.bfloat16, seed=3))
    ts = [oracle.calibrate_sort(acts, k).t for k in np.linspace(0, 0.99, 40)]
    assert all(a <= b for a, b in zip(ts, ts[1:]))


def test_gaussian_quantile_closed_form():
    from scipy.stats import norm
    n = 2_000_000
    acts = cats_synth.to_oracle(cats_synth.calib_acts(n, torch.float32, seed=4, sigma=1.0))
    for k in [0.5, 0.7, 0.9]:
        res = oracle.calibrate_sort(acts, k)
        want = norm.ppf((1 + k) / 2)     # |N(0,1)| quantile
        sd = math.sqrt(k * (1 - k) / n) / (2 * norm.pdf(want))
        assert abs(res.t - want) < 6 * sd + 1e-6, (k, res.t, want)
        _check_invariant(res, k)


def _silu_abs_cdf(t, sigma):
    """P(|SiLU(u)| <= t) for u ~ N(0, sigma^2), from the level sets of SiLU (scipy roots)."""
    from scipy.optimize import brentq
    from scipy.stats import norm
    silu = lambda u: u / (1 + math.exp(-u))
    ustar, smin = -1.278464542761074, -0.2784645427610738
    c = brentq(lambda u: silu(u) - t, 0, 50)                 # positive branch
    F = norm.cdf(c / sigma) - 0.5
    if t < -smin:                                             # two negative-branch roots
        a = brentq(lambda u: silu(u) + t, -60, ustar)
        bb = brentq(lambda u: silu(u) + t, ustar, 0)
        F += norm.cdf(a / sigma) + (0.5 - norm.cdf(bb / sigma))
    else:
        F += 0.5
    return F


def test_silu_gaussian_quantile_closed_form():
    """Eq. 3 applied to |SiLU(u)|, u ~ N(0,1): the oracle's SiLU + quantile against the analytic
    level-set CDF (t_0.5 = 0.25431967, t_0.7 = 0.32941591, t_0.9 = 1.00308806)."""
    from scipy.optimize import brentq
    n = 1_000_000
    u = cats_synth.calib_acts(n, torch.float32, seed=5, sigma=1.0).numpy()
    # the oracle's own SiLU, via a d=1 MLP whose gate weights are the samples
    _, v, _ = oracle.mlp(np.ones((1, 1), np.float32), u.reshape(n, 1), np.zeros((n, 1), np.float32),
                         np.zeros((n, 1), np.float32), t=0.0, mode=oracle.DENSE)
    acts = v[0].astype(np.float32)
    for k, pinned in [(0.5, 0.25431967), (0.7, 0.32941591), (0.9, 1.00308806)]:
        want = brentq(lambda t: _silu_abs_cdf(t, 1.0) - k, 1e-6, 10)
        assert abs(want - pinned) < 1e-7
        res = oracle.calibrate_sort(acts, k)
        assert abs(res.t - want) < 2e-3, (k, res.t, want)


def test_paper_anchor_sigma():
    """70% sparsity <-> t ~ 0.15. With u ~ N(0, 0.30^2) (the synthetic recipe) the
    analytic t_0.7 is 0.1494 (bf16 sample gives 0x3e19 ~ 0.1494)."""
    from scipy.optimize import brentq
    t7 = brentq(lambda t: _silu_abs_cdf(t, 0.30) - 0.7, 1e-6, 5)
    assert abs(t7 - 0.15) < 0.002


def test_bf16_counts_equals_sort():
    rng = np.random.default_rng(6)
    for it in range(6):
        n = int(rng.integers(1000, 50000))
        vals = torch.from_numpy(rng.normal(0, 0.3, n).astype(np.float32)).to(torch.bfloat16)
        acts = cats_synth.bf16_bits(vals).copy()
        acts[: n // 50] = 0x8000 if it % 2 else 0x0000      # signed zeros
        counts = np.zeros(65536, np.uint64)
        for s in range(0, n, 7777):                          # chunked accumulation
            oracle.bf16_counts(acts[s:s + 7777], counts)
        for k in [0.0, 0.3, 0.5, 0.7, 0.9, 0.999]:
            a = oracle.calibrate_sort(acts, k)
            b = oracle.calibrate_bf16_counts(counts, k)
            assert tuple(a) == tuple(b), (k, a, b)


def test_nonfinite_rejected():
    acts = np.array([0.1, np.inf, 0.2], np.float32)
    with pytest.raises(FloatingPointError):
        oracle.calibrate_sort(acts, 0.5)
    bits = cats_synth.bf16_bits(torch.tensor([0.5, float("nan")], dtype=torch.bfloat16))
    with pytest.raises(FloatingPointError):
        oracle.calibrate_bf16_counts(oracle.bf16_counts(bits), 0.5)


# ------------------------------------------------------ App. B: CATS before the attention projections

def test_xsparse_gemv_worked_example():
    """CATS_t(x) (Eq. 4, applied to the hidden vector, App. B) then x W: with
    x = (1, -0.2, 0.5, 0.05), t = 0.3 only inputs 0 and 2 survive, so y = W[0] + 0.5 W[2]
    (computed by hand for W[i][n] = 3 i + n)."""
    x = np.array([[1.0, -0.2, 0.5, 0.05]], np.float32)
    W = np.arange(12, dtype=np.float32).reshape(4, 3)
    y, keep = oracle.xsparse_gemv(x, W, 0.3)
    assert keep.tolist() == [[1, 0, 1, 0]]
    assert y.tolist() == [[3.0, 4.5, 6.0]]
    y_tie, keep_tie = oracle.xsparse_gemv(x, W, 0.5)   # |x_2| = t: kept (ties, reading G1)
    assert keep_tie.tolist() == [[1, 0, 1, 0]]


def test_xsparse_gemv_t0_is_the_dense_product_and_masking_is_exact():
    rng = np.random.default_rng(5)
    x = rng.standard_normal((3, 40)).astype(np.float32)
    W = rng.standard_normal((40, 24)).astype(np.float32)
    y0, k0 = oracle.xsparse_gemv(x, W, 0.0)
    assert k0.all()
    np.testing.assert_allclose(y0, x.astype(np.float64) @ W.astype(np.float64), rtol=1e-12, atol=1e-12)
    t = 0.8
    y, keep = oracle.xsparse_gemv(x, W, t)
    assert (keep == (np.abs(x.astype(np.float64)) >= t)).all()
    np.testing.assert_allclose(y, (x.astype(np.float64) * keep) @ W.astype(np.float64), rtol=1e-12, atol=1e-12)
    y_hi, k_hi = oracle.xsparse_gemv(x, W, float(np.abs(x).max()) * 2)
    assert not k_hi.any() and not y_hi.any()


def test_xsparse_gemv_brute_force_rationals():
    from fractions import Fraction
    rng = np.random.default_rng(6)
    for _ in range(20):
        x = (rng.integers(-8, 9, size=(2, 5)) / 8).astype(np.float32)
        W = (rng.integers(-8, 9, size=(5, 3)) / 4).astype(np.float32)
        t = float(rng.integers(0, 8) / 8)
        y, _ = oracle.xsparse_gemv(x, W, t)
        for bt in range(2):
            for n in range(3):
                exact = sum((Fraction(float(x[bt, i])) * Fraction(float(W[i, n])) for i in range(5)
                             if abs(Fraction(float(x[bt, i]))) >= Fraction(t)), Fraction(0))
                assert Fraction(y[bt, n]) == exact


def test_oracle_bf16_widening_matches_torch_for_every_finite_pattern():
    """The oracle's bf16 -> double widening (cats_oracle.c `widen`) pinned against torch's own
    bfloat16 -> float32 conversion for all 65 280 finite bit patterns (incl. subnormals and -0):
    y = CATS_0(x) I through oracle.xsparse_gemv returns each x_c times 1 plus exact zeros."""
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    finite = (bits & 0x7F80) != 0x7F80
    bits = bits[finite]
    ref = torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16).float().double().numpy()
    n = 256
    eye = np.zeros((n, n), np.uint16)
    eye[np.arange(n), np.arange(n)] = 0x3F80  # bf16 1.0
    pad = (-len(bits)) % n
    xb = np.concatenate([bits, np.zeros(pad, np.uint16)]).reshape(-1, n)
    got = np.concatenate([oracle.xsparse_gemv(xb[i:i + 1], eye, 0.0)[0][0] for i in range(xb.shape[0])])[:len(bits)]
    assert np.array_equal(got, ref)  # -0 == +0; every other value bit-exact
    assert np.array_equal(np.signbit(got[ref != 0]), np.signbit(ref[ref != 0]))
    # the same widening seen through Eq. 3: the r-th smallest |a| is returned exactly as torch widens it
    a = bits[np.random.default_rng(0).permutation(len(bits))[:5001]]
    at = np.abs(torch.from_numpy(a.view(np.int16).copy()).view(torch.bfloat16).float().double().numpy())
    for k in (0.1, 0.5, 0.9):
        r = oracle.rank(k, len(a))
        assert oracle.calibrate_sort(a, k).t == np.sort(at)[r - 1]


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_openmp_timing_build_is_bit_identical(dtype):
    """The all-core timing build (same source, -fopenmp) returns exactly the serial checker's bits."""
    x, Wg, Wu, Wd = _case(136, 417, 3, dtype, seed=4)
    for mode, t in ((oracle.SPARSE, 0.05), (oracle.MASKED, 0.05), (oracle.DENSE, 0.0)):
        a = oracle.mlp(x, Wg, Wu, Wd, t=t, mode=mode)
        b = oracle.mlp(x, Wg, Wu, Wd, t=t, mode=mode, all_cores=True)
        for u, v in zip(a, b):
            assert np.array_equal(u, v)
