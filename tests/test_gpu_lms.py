"""GPU parity of the LMS path (a7 residual GEMM on tcgen05, a8 batched selection) against the oracle.

Bars: S from the split-TF32 tensor-core GEMM within the 3xTF32 error bound of the
fp64 residuals; every per-column median bit-exact against the sort-based oracle on the GPU's own
S column; the LMS objective within max_i |S_gpu,i - S_fp64,i| of the fp64 objective (order
statistics are 1-Lipschitz in the sup norm)."""
import numpy as np
import pytest

import datagen
import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cp():
    import torch
    assert torch.cuda.is_available()
    import paper_1104_2732_b200 as cp
    cp.load()
    return cp


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def residual_bound(X, y, th):
    """|r_gpu - r_fp64| bound for 3xTF32 products (each ~2^-21 relative) with fp32 accumulation
    over K=16 terms: 2^-19 * (sum_l |x_il theta_lj| + |y_i|), generous by ~4x."""
    A = np.abs(X.astype(np.float64)) @ np.abs(th.astype(np.float64)).T + np.abs(y.astype(np.float64))[:, None]
    return 2.0 ** -19 * A


@pytest.mark.parametrize("n,p,C", [(1, 1, 1), (7, 3, 5), (128, 10, 256), (1000, 10, 300), (12_345, 16, 777),
                                   (100_003, 10, 64)])
def test_residuals_match_fp64(cp, n, p, C):
    rng = np.random.default_rng(n + p + C)
    X = rng.standard_normal((n, p)).astype(np.float32)
    y = (rng.standard_normal(n) * 3).astype(np.float32)
    th = rng.standard_normal((C, p)).astype(np.float32)
    S = cp.lms_residuals(dev(X), dev(y), dev(th)).cpu().numpy()        # (C, n)
    R64 = X.astype(np.float64) @ th.astype(np.float64).T - y.astype(np.float64)[:, None]
    ref = (R64 * R64).T
    rb = residual_bound(X, y, th).T
    err = np.abs(S.astype(np.float64) - ref)
    tol = rb * (2 * np.sqrt(ref) + rb) + 2.0 ** -23 * ref + 1e-30
    assert np.all(err <= tol), float(np.max(err / tol))


@pytest.mark.parametrize("dist", ["uniform", "normal", "dup256", "halfnormal", "mix3"])
def test_batched_select_bit_exact(cp, dist):
    """a8 on arbitrary columns: every column's k-th smallest bit-exact vs the oracle."""
    n, C = 50_001, 96
    S = datagen.make(dist, n * C, "f32").reshape(C, n)
    S[5, :] = 3.0                       # a constant column
    S[6, : n // 2] = -0.0               # signed zeros
    S[6, n // 2:] = 0.0
    Sd = dev(S)
    for k in (1, 2, n // 10, O.median_rank(n), n - 1, n):
        got = cp.select_kth_batched(Sd, k).cpu().numpy()
        for j in range(C):
            want = O.order_statistic(S[j], k)
            assert got[j] == want, (dist, k, j, got[j], want)


def test_batched_select_small_and_ragged(cp):
    rng = np.random.default_rng(9)
    for n in (1, 2, 3, 31, 33, 1000):
        C = 37
        S = rng.standard_normal((C, n)).astype(np.float32)
        S[:, ::3] = S[:, :1]          # duplicates
        Sd = dev(S)
        for k in sorted({1, (n + 1) // 2, n}):
            got = cp.select_kth_batched(Sd, k).cpu().numpy()
            want = np.array([O.order_statistic(S[j], k) for j in range(C)], np.float32)
            assert np.array_equal(got, want)


def test_lms_objective_vs_oracle(cp):
    X, y, th, theta_star = datagen.lms_problem(n=200_001, p=10, C=512)
    got, info = cp.lms_objective(dev(X), dev(y), dev(th), return_info=True)
    got = got.cpu().numpy()
    # bit-exact median of the GPU's own S column
    S = cp.lms_residuals(dev(X), dev(y), dev(th)).cpu().numpy()
    k = O.median_rank(X.shape[0])
    for j in range(0, 512, 7):
        assert got[j] == O.order_statistic(S[j], k)
    # within the Lipschitz bound of the fp64 objective
    ref = O.lms_objective(X, y, th)
    S64 = O.lms_residuals_sq(X, y, th).T
    for j in range(0, 512, 7):
        assert abs(float(got[j]) - ref[j]) <= np.max(np.abs(S[j].astype(np.float64) - S64[j])) + 1e-30


def test_lms_config4_full_size(cp):
    """BASELINE configs[4]: n=1e6, p=10, 4096 candidates; sampled columns checked against the
    oracle on the GPU's S, and the true theta* ranks best among the candidates near it."""
    import torch
    X, y, th, theta_star = datagen.lms_problem()
    Xd, yd, thd = dev(X), dev(y), dev(th)
    got, info = cp.lms_objective(Xd, yd, thd, return_info=True)
    got = got.cpu().numpy()
    assert np.all(np.isfinite(got)) and got.shape == (4096,)
    S = cp.lms_residuals(Xd, yd, thd)
    k = O.median_rank(X.shape[0])
    rng = np.random.default_rng(0)
    for j in rng.choice(4096, 24, replace=False):
        col = S[j].cpu().numpy()
        assert got[j] == O.order_statistic(col, k)
    del S
    torch.cuda.empty_cache()
    # candidates with the smallest perturbations (sigma ~ 1e-3) fit far better than sigma ~ 1
    assert got[:64].max() < got[-64:].min()


@pytest.mark.parametrize("h_rule", ["half", "n_plus_p"])
def test_lts_objective_vs_oracle(cp, h_rule):
    """NEXT row LTS: per candidate the sum of the h smallest squared residuals of the GPU's own S
    (oracle rho/a,b form, fp64) within fp64 rounding, and the h-th smallest bit-exact; and the
    true theta* fits far better than the sigma ~ 1 candidates."""
    X, y, th, theta_star = datagen.lms_problem(n=100_003, p=10, C=300)
    n, p = X.shape
    h = (n + 1) // 2 if h_rule == "half" else (n + p) // 2      # R20: both readings
    Xd, yd, thd = dev(X), dev(y), dev(th)
    F, m = cp.lts_objective(Xd, yd, thd, h)
    F, m = F.cpu().numpy(), m.cpu().numpy()
    S = cp.lms_residuals(Xd, yd, thd).cpu().numpy()
    for j in range(0, 300, 11):
        assert m[j] == O.order_statistic(S[j], h)
        ref = O.lts_objective(S[j].astype(np.float64), h)
        assert F[j] == pytest.approx(ref, rel=1e-11), (j, F[j], ref)   # fp64 sums, different order
    assert F[:16].max() < F[-16:].min()


# ---------------------------------------------------------------------------------- fused path
# §8f-2: with lms_fused=1 (default, n >= 16384) S is never stored: the residuals are recomputed in
# the tcgen05 epilogue of one fused pass.  cpsel_lms_residuals returns the S of that same kernel
# (store mode), so every selected value must be an order statistic of it, bit-exact.

def _fused_problem(n=60_013, C=333, seed=5):
    X, y, th, _ = datagen.lms_problem(n=n, p=10, C=C)
    return X, y, th


@pytest.mark.parametrize("which", ["k1", "tenth", "median", "n_minus_1", "n"])
def test_fused_kth_every_column_bit_exact(cp, which):
    """every column, ranks at both ends and the middle (k via the LTS entry point, whose m_j is
    the fused k-th order statistic), against the oracle on the fused kernel's own S."""
    X, y, th = _fused_problem()
    n = X.shape[0]
    h = {"k1": 1, "tenth": n // 10, "median": O.median_rank(n), "n_minus_1": n - 1, "n": n}[which]
    Xd, yd, thd = dev(X), dev(y), dev(th)
    F, m = cp.lts_objective(Xd, yd, thd, h)
    m, F = m.cpu().numpy(), F.cpu().numpy()
    S = cp.lms_residuals(Xd, yd, thd).cpu().numpy()
    for j in range(th.shape[0]):
        assert m[j] == O.order_statistic(S[j], h), (which, j)
    for j in range(0, th.shape[0], 17):
        ref = O.lts_objective(S[j].astype(np.float64), h)
        assert F[j] == pytest.approx(ref, rel=1e-11), (j, F[j], ref)


def test_fused_matches_unfused_path(cp):
    """lms_fused=0 (S stored by the row-major residual kernel, then the batched select) and
    lms_fused=1 agree within the 3xTF32 bound; each is bit-exact on its own S."""
    X, y, th = _fused_problem(n=70_001, C=260)
    Xd, yd, thd = dev(X), dev(y), dev(th)
    k = O.median_rank(X.shape[0])
    try:
        cp.set_config(lms_fused=0)
        g0 = cp.lms_objective(Xd, yd, thd).cpu().numpy()
        S0 = cp.lms_residuals(Xd, yd, thd).cpu().numpy()
    finally:
        cp.set_config(lms_fused=1)
    g1 = cp.lms_objective(Xd, yd, thd).cpu().numpy()
    S1 = cp.lms_residuals(Xd, yd, thd).cpu().numpy()
    for j in range(0, 260, 13):
        assert g0[j] == O.order_statistic(S0[j], k)
        assert g1[j] == O.order_statistic(S1[j], k)
    assert np.all(np.abs(g0.astype(np.float64) - g1) <= np.max(np.abs(S0.astype(np.float64) - S1), axis=1) + 1e-30)


def test_fused_fallback_columns(cp):
    """Adversarial sample rows: y is huge exactly at the rows the cut stage samples (16384 evenly
    strided rows per candidate tile of 128, phase (tile * 2654435761) mod stride), so every
    column's sample cuts lie far above its median; the fused copy cannot finish any column and all
    of them must go through the stored-S fallback — still bit-exact."""
    X, y, th = _fused_problem(n=200_000, C=130)
    n = X.shape[0]
    ms = 16384                                                          # kLmsSamples
    stride = n // ms
    y = y.copy()
    for ct in range((th.shape[0] + 127) // 128):
        rows = (np.arange(ms, dtype=np.int64) * n) // ms + (ct * 2654435761) % stride
        y[rows] = 1e4
    Xd, yd, thd = dev(X), dev(y), dev(th)
    got, info = cp.lms_objective(Xd, yd, thd, return_info=True)
    got = got.cpu().numpy()
    assert info["fallback_steps"] == th.shape[0]
    S = cp.lms_residuals(Xd, yd, thd).cpu().numpy()
    k = O.median_rank(n)
    for j in range(th.shape[0]):
        assert got[j] == O.order_statistic(S[j], k), j


def test_fused_nonfinite_rejected(cp):
    X, y, th = _fused_problem(n=20_000, C=40)
    y = y.copy()
    y[777] = np.nan
    with pytest.raises(ValueError, match="NaN or Inf"):
        cp.lms_objective(dev(X), dev(y), dev(th))


@pytest.mark.parametrize("p,C", [(1, 1), (3, 129), (16, 200), (10, 1)])
def test_fused_shapes(cp, p, C):
    """Fused path for other predictor counts (K padding 1..16) and candidate counts (one column, a
    ragged last candidate tile): every column bit-exact on the fused kernel's own S, and that S
    within the 3xTF32 bound of fp64."""
    n = 20_011                                                    # >= 16384: fused; ragged row tile
    rng = np.random.default_rng(p * 1000 + C)
    X = rng.standard_normal((n, p)).astype(np.float32)
    y = (rng.standard_normal(n) * 2).astype(np.float32)
    th = rng.standard_normal((C, p)).astype(np.float32)
    Xd, yd, thd = dev(X), dev(y), dev(th)
    got = cp.lms_objective(Xd, yd, thd).cpu().numpy()
    S = cp.lms_residuals(Xd, yd, thd).cpu().numpy()
    k = O.median_rank(n)
    for j in range(C):
        assert got[j] == O.order_statistic(S[j], k), j
    R64 = X.astype(np.float64) @ th.astype(np.float64).T - y.astype(np.float64)[:, None]
    ref = (R64 * R64).T
    rb = residual_bound(X, y, th).T
    assert np.all(np.abs(S.astype(np.float64) - ref) <= rb * (2 * np.sqrt(ref) + rb) + 2.0 ** -23 * ref + 1e-30)
