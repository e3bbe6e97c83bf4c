"""Pins for the CPU oracle (-m "not gpu").

Each test ties an oracle function to something other than the oracle itself:
brute force over the rank definition, exact-rational finite differences, the
paper's printed closed forms, hand-derived golden examples, the Appendix-A
identity in exact rationals, or a claim the paper makes about the method.
"""
import itertools
import math
import random
from fractions import Fraction

import numpy as np
import pytest

import datagen
import oracle as O


# ----------------------------------------------------------------------------- brute force
def brute_kth(xs, k):
    """Rank definition, pure Python: the v in xs with #{x<v} <= k-1 < #{x<=v}."""
    for v in xs:
        lt = sum(1 for a in xs if a < v)
        le = sum(1 for a in xs if a <= v)
        if lt <= k - 1 < le:
            return v
    raise AssertionError("no element satisfies the rank definition")


def frac_F(xs, y, k):
    """F_k(y) in exact rationals, from Eq. 2's u with paper-k = n-k+1 (R2), written as
    positive/negative parts: (k-1/2) sum (x-y)^+ + (n-k+1/2) sum (y-x)^+."""
    n = len(xs)
    y = Fraction(y)
    P = sum((Fraction(a) - y for a in xs if a > y), Fraction(0))
    N = sum((y - Fraction(a) for a in xs if a < y), Fraction(0))
    return (k - Fraction(1, 2)) * P + (n - k + Fraction(1, 2)) * N


def tiny_samples(rng, count, nmax=12):
    vals = [0.0, -0.0, 1.0, -1.0, 2.5, 1e9, -1e9, 3.0, 3.0, 0.5]
    for _ in range(count):
        n = rng.randint(1, nmax)
        if rng.random() < 0.5:
            xs = [rng.choice(vals) for _ in range(n)]
        else:
            xs = [float(np.float32(rng.uniform(-5, 5))) for _ in range(n)]
        yield xs


# ----------------------------------------------------------------------------- golden (SPEC / paper)
def test_golden_median_rank(golden):
    for g in golden["median_rank"]:
        assert O.median_rank(g["n"]) == g["k"], g["cite"]


def test_golden_objective_eq1(golden):
    for g in golden["f_median"]:
        x = np.array(g["x"], dtype=np.float64)
        assert float(O.f_median(x, g["y"])) == g["f"], g["cite"]
        assert tuple(O.subdiff_median(x, g["y"])) == tuple(g["subdiff"]), g["cite"]


def test_golden_eq2_direction(golden):
    """Reading R2: Eq. 2's printed k selects the k-th LARGEST."""
    for g in golden["f_paper_eq2"]:
        x = np.array(g["x"], dtype=np.float64)
        n = x.size
        f = float(np.sum(O.u_paper(x - g["y"], n, g["paper_k"])))
        assert f == g["f"], g["cite"]
        vals = [float(np.sum(O.u_paper(x - v, n, g["paper_k"]))) for v in x]
        assert x[int(np.argmin(vals))] == g["argmin"], g["cite"]
        # and the API's k-th smallest with k = n - paper_k + 1 gives the same objective
        assert float(O.f_os(x, g["y"], n - g["paper_k"] + 1)) == g["f"]


def test_golden_bracket_init(golden):
    """P:L194 closed forms, Eq. 1 scaling (F_k at the median of odd n is (n/2) f)."""
    for g in golden["bracket_init_eq1"]:
        x = np.array(g["x"], dtype=np.float64)
        rec = O.init_record(x)
        n = x.size
        assert rec["min"] == g["y_L"] and rec["max"] == g["y_R"]
        assert float(rec["sum"] - n * g["y_L"]) == g["f_L"]
        assert float(n * g["y_R"] - rec["sum"]) == g["f_R"]
        assert O.subdiff_median(x, g["y_L"])[1] == g["g_L"]      # right derivative at y_L
        assert O.subdiff_median(x, g["y_R"])[0] == g["g_R"]      # left derivative at y_R


def test_golden_cutting_plane(golden):
    for g in golden["cutting_plane"]:
        x = np.array(g["x"], dtype=np.float64)
        r = O.cutting_plane(x, g["k"])
        assert r["value"] == g["value"] and r["iterations"] == g["iterations"], g["cite"]
        if "t1" in g:
            assert r["trace"][0][0] == g["t1"]


def test_golden_exact_finish(golden):
    for g in golden["exact_finish"]:
        x = np.array(g["x"], dtype=np.float64)
        s = O.pass_stats(x, g["y"] + 1e-9, -math.inf, math.inf)
        # largest x_i <= y~ is pred of a query just above y~ (P:L192 footnote)
        assert s["pred"] == g["value"], g["cite"]


def test_golden_lms_lts(golden):
    for g in golden["lms"]:
        r = np.array(g["r"], dtype=np.float64)
        X = np.ones((r.size, 1))
        assert O.lms_objective(X, -r, np.zeros((1, 1)))[0] == g["lms"], g["cite"]
    for g in golden["lts"]:
        assert O.lts_objective(np.array(g["rsq"], float), g["h"]) == g["lts"], g["cite"]


# ----------------------------------------------------------------------------- plain definition
def test_order_statistic_vs_brute_force_all_permutations():
    rng = random.Random(1)
    for n in range(1, 7):
        base = [rng.choice([0.0, 1.0, 1.0, 2.0, -3.0, 1e9]) for _ in range(n)]
        for perm in set(itertools.permutations(base)):
            x = np.array(perm, dtype=np.float64)
            for k in range(1, n + 1):
                assert O.order_statistic(x, k) == brute_kth(list(perm), k)


def test_order_statistic_vs_brute_force_random_tiny():
    rng = random.Random(2)
    for xs in tiny_samples(rng, 400):
        for dt in (np.float32, np.float64):
            x = np.array(xs, dtype=dt)
            for k in range(1, len(xs) + 1):
                v = O.order_statistic(x, k)
                assert v == brute_kth([dt(a) for a in xs], k)
                assert O.order_statistic_sorted(x, k) == v
                assert not (v == 0 and math.copysign(1.0, float(v)) < 0)  # canonical +0 (R13)


def test_rank_invariant_large():
    """#{x < x_(k)} <= k-1 < #{x <= x_(k)} (north_star) on every distribution."""
    for dist in datagen.ALL_DISTS:
        x = datagen.make(dist, 100_003, "f32")
        n = x.size
        for k in (1, 2, n // 10, O.median_rank(n), n - 1, n):
            v = O.order_statistic(x, k)
            c_lt, c_eq = O.rank_counts(x, v)
            assert c_lt <= k - 1 < c_lt + c_eq


def test_check_input_errors():
    with pytest.raises(ValueError):
        O.order_statistic(np.array([], np.float32), 1)
    with pytest.raises(ValueError):
        O.order_statistic(np.array([1.0]), 2)
    with pytest.raises(ValueError):
        O.order_statistic(np.array([1.0, np.nan]), 1)
    with pytest.raises(ValueError):
        O.cutting_plane(np.array([1.0, np.inf]), 1)


# ----------------------------------------------------------------------------- objectives / subgradients
def test_subdiff_equals_exact_finite_difference_off_grid():
    """off the data grid dF is a point equal to the central finite difference
    (computed here in exact rationals from F's values, not from counts)."""
    rng = random.Random(3)
    for xs in tiny_samples(rng, 300, nmax=9):
        xs = [float(a) for a in xs]
        x = np.array(xs)
        n = len(xs)
        grid = sorted(set(xs))
        pts = [grid[0] - 1.0, grid[-1] + 1.0] + [(a + b) / 2 for a, b in zip(grid, grid[1:])]
        for y in pts:
            gap = min(abs(Fraction(y) - Fraction(a)) for a in xs)
            h = gap / 2
            for k in range(1, n + 1):
                fd = (frac_F(xs, Fraction(y) + h, k) - frac_F(xs, Fraction(y) - h, k)) / (2 * h)
                lo, hi = O.subdiff_os(x, y, k)
                assert lo == hi == fd
            fd1 = sum((1 if Fraction(y) + h > a else -1) for a in xs)  # slope of sum|x-y| just right
            lo1, hi1 = O.subdiff_median(x, y)
            assert lo1 == hi1 == fd1


def test_subdiff_at_kinks_are_one_sided_derivatives():
    """At a data point the interval ends are the one-sided derivatives (Clarke)."""
    rng = random.Random(4)
    for xs in tiny_samples(rng, 200, nmax=8):
        xs = [float(a) for a in xs]
        x = np.array(xs)
        n = len(xs)
        gaps = [abs(Fraction(a) - Fraction(b)) for a in xs for b in xs if a != b]
        h = (min(gaps) / 4) if gaps else Fraction(1)
        for y in set(xs):
            for k in range(1, n + 1):
                lo, hi = O.subdiff_os(x, y, k)
                assert hi == (frac_F(xs, Fraction(y) + h, k) - frac_F(xs, y, k)) / h
                assert lo == (frac_F(xs, y, k) - frac_F(xs, Fraction(y) - h, k)) / h


def test_paper_g_is_negated_subdifferential_R1():
    """Reading R1: P:L130's g as printed is -df of Eq. 1."""
    rng = random.Random(5)
    for xs in tiny_samples(rng, 100):
        x = np.array(xs, dtype=np.float64)
        for y in list(x) + [0.25]:
            lo, hi = O.g_paper(x, y)
            dlo, dhi = O.subdiff_median(x, y)
            assert (lo, hi) == (-dhi, -dlo)


def test_eq2_minimizer_is_kth_smallest_with_mapped_k():
    """Brute force: argmin over the data of F_k (R2 mapping) is the k-th smallest; the optimality
    condition 0 in dF_k(y) holds exactly at y = x_(k)."""
    rng = random.Random(6)
    for xs in tiny_samples(rng, 200, nmax=9):
        x = np.array(xs, dtype=np.float64)
        n = x.size
        for k in range(1, n + 1):
            vals = [frac_F([float(a) for a in xs], float(v), k) for v in x]
            best = min(vals)
            argmins = {float(v) for v, f in zip(x, vals) if f == best}
            target = brute_kth([float(a) for a in xs], k)
            assert argmins == {target}
            lo, hi = O.subdiff_os(x, target, k)
            assert lo <= 0 <= hi
            assert float(O.f_os(x, target, k)) == pytest.approx(float(best), rel=1e-15, abs=1e-12)


def test_eq2_reduces_to_eq1_at_median_of_odd_n():
    """odd n, k=(n+1)/2 -> F_k = (n/2) * f (Eq. 1)."""
    x = datagen.make("normal", 1001, "f64")
    k = O.median_rank(x.size)
    for y in (-1.0, 0.0, 0.3, 2.0):
        assert float(O.f_os(x, y, k)) == pytest.approx(x.size / 2 * float(O.f_median(x, y)), rel=1e-15)


def test_paper_closed_forms_at_the_extremes():
    """with unique extremes g(y_L)=-n+2, g(y_R)=n-2, f(y_L)=sum x - n y_L,
    f(y_R)=n y_R - sum x (Eq. 1); the k-weighted version scales by (k-1/2) / (n-k+1/2)."""
    x = datagen.make("normal", 4097, "f64")
    n = x.size
    rec = O.init_record(x)
    assert rec["cnt_min"] == rec["cnt_max"] == 1
    assert O.subdiff_median(x, rec["min"])[1] == -n + 2
    assert O.subdiff_median(x, rec["max"])[0] == n - 2
    S = float(rec["sum"])
    assert float(O.f_median(x, rec["min"])) == pytest.approx(S - n * float(rec["min"]), rel=1e-13)
    assert float(O.f_median(x, rec["max"])) == pytest.approx(n * float(rec["max"]) - S, rel=1e-13)
    for k in (1, 7, 2049, n):
        assert float(O.f_os(x, rec["min"], k)) == pytest.approx((k - .5) * (S - n * float(rec["min"])), rel=1e-13)
        assert float(O.f_os(x, rec["max"], k)) == pytest.approx((n - k + .5) * (n * float(rec["max"]) - S), rel=1e-13)


def test_convexity_and_permutation_invariance():
    x = datagen.make("mix1", 2000, "f64")
    k = 777
    ys = np.sort(np.random.default_rng(0).uniform(-3, 103, 60))
    F = [float(O.f_os(x, y, k)) for y in ys]
    for i in range(1, len(ys) - 1):
        y0, y1, y2 = ys[i - 1], ys[i], ys[i + 1]
        interp = ((y2 - y1) * F[i - 1] + (y1 - y0) * F[i + 1]) / (y2 - y0)
        assert F[i] <= interp * (1 + 1e-12)
    xp = x[np.random.default_rng(1).permutation(x.size)]
    assert float(O.f_os(xp, 50.0, k)) == pytest.approx(float(O.f_os(x, 50.0, k)), rel=1e-15)
    assert O.cutting_plane(xp, k)["value"] == O.cutting_plane(x, k)["value"]


def test_pass_stats_identities():
    """Appendix-A positive-term identities tie pass_stats' local sums to the direct P and N:
    P(t) = P(y_R) + #{x>=y_R}(y_R-t) + L_hi,  N(t) = N(y_L) + #{x<=y_L}(t-y_L) + L_lo."""
    x = datagen.make("normal", 50_001, "f64")
    yL, t, yR = -0.5, 0.1, 0.9
    s = O.pass_stats(x, t, yL, yR)
    sL = O.pass_stats(x, yL, -math.inf, math.inf)
    sR = O.pass_stats(x, yR, -math.inf, math.inf)
    c_le_L = sL["c_lt"] + sL["c_eq"]
    c_ge_R = x.size - sR["c_lt"]
    assert float(s["P"]) == pytest.approx(float(sR["P"] + c_ge_R * O.LD(yR - t) + s["L_hi"]), rel=1e-14)
    assert float(s["N"]) == pytest.approx(float(sL["N"] + c_le_L * O.LD(t - yL) + s["L_lo"]), rel=1e-14)
    assert s["c_lo"] == s["c_lt"] - c_le_L
    assert s["pred"] == x[(x > yL) & (x < t)].max() and s["succ"] == x[(x > t) & (x < yR)].min()


def _grid_samples(rng, count):
    """Small integer-valued samples with heavy duplication: every sum below is exact in float64,
    and data values (kinks of F) are plentiful so brackets and queries land ON the grid."""
    for _ in range(count):
        n = rng.randint(2, 14)
        yield [float(rng.randint(-4, 4)) for _ in range(n)]


def test_F_from_PN_matches_eq2_and_exact_rationals():
    """oracle.F_from_PN / eval_at()['F'] against two independent forms of Eq. 2:
    the exact-rational F_k (frac_F, itself pinned to the rank definition by
    test_eq2_minimizer_is_kth_smallest_with_mapped_k) and oracle.f_os (the penalty u exactly as
    printed, with paper-k = n-k+1).  Queries on and off the data grid, every k: the weights
    (k-1/2) on P and (n-k+1/2) on N are not symmetric for k != (n+1)/2, so swapping them fails."""
    rng = random.Random(11)
    for xs in _grid_samples(rng, 150):
        x = np.array(xs)
        n = x.size
        grid = sorted(set(xs))
        ys = grid + [grid[0] - 0.75, grid[-1] + 1.25] + [(a + b) / 2 for a, b in zip(grid, grid[1:])]
        for y in ys:
            for k in range(1, n + 1):
                e = O.eval_at(x, k, y, -math.inf, math.inf)
                exact = frac_F(xs, y, k)
                assert Fraction(float(e["F"])) == exact, (xs, y, k)
                assert float(O.F_from_PN(n, k, e["P"], e["N"])) == float(exact)
                assert float(O.f_os(x, y, k)) == float(exact)


def test_F_from_PN_minimizer_is_kth_smallest():
    """Brute force: over the data values, the F assembled by eval_at (F_from_PN of the pass's P and
    N) is minimised exactly at x_(k) (rank definition), and nowhere else (the 1/2 offsets make the
    minimiser unique, reading R6)."""
    rng = random.Random(12)
    for xs in _grid_samples(rng, 150):
        x = np.array(xs)
        for k in range(1, x.size + 1):
            vals = {v: float(O.eval_at(x, k, v, -math.inf, math.inf)["F"]) for v in set(xs)}
            best = min(vals.values())
            assert {v for v, f in vals.items() if f == best} == {brute_kth(xs, k)}


def test_pass_stats_strict_bracket_on_grid():
    """pass_stats' bracket is OPEN at both ends (P:L196 'y_L < x_i < y_R'), checked with y_L, t,
    y_R ON data values that carry duplicates, against properties fixed by the mathematics:
      c_lo = #{x<t} - #{x<=y_L},  c_hi = #{x<y_R} - #{x<=t}          (counts, brute force)
      N(t) = N(y_L) + #{x<=y_L}(t-y_L) + L_lo                        (App. A, exact here)
      P(t) = P(y_R) + #{x>=y_R}(y_R-t) + L_hi
      pred = x_(#{x<t}) if any element lies in ]y_L,t[ else -inf     (order statistics of
      succ = x_(#{x<=t}+1) if any element lies in ]t,y_R[ else +inf   a sorted copy)
    An inclusive end double-counts the elements equal to y_L / y_R in c_lo / L_lo (resp. c_hi /
    L_hi) and reports pred = y_L on an empty ]y_L, t[."""
    rng = random.Random(13)
    cases = 0
    for xs in _grid_samples(rng, 400):
        grid = sorted(set(xs))
        if len(grid) < 3:
            continue
        x = np.array(xs)
        srt = sorted(xs)
        for i in range(len(grid)):
            for j in range(i + 1, len(grid)):
                for q in range(i + 1, j):
                    yL, t, yR = grid[i], grid[q], grid[j]
                    s = O.pass_stats(x, t, yL, yR)
                    lt_t = sum(a < t for a in xs)
                    le_t = sum(a <= t for a in xs)
                    le_L = sum(a <= yL for a in xs)
                    lt_R = sum(a < yR for a in xs)
                    ge_R = len(xs) - lt_R
                    assert s["c_lo"] == lt_t - le_L and s["c_hi"] == lt_R - le_t
                    NL = sum(yL - a for a in xs if a < yL)
                    PR = sum(a - yR for a in xs if a > yR)
                    assert float(s["N"]) == NL + le_L * (t - yL) + float(s["L_lo"])
                    assert float(s["P"]) == PR + ge_R * (yR - t) + float(s["L_hi"])
                    assert s["pred"] == (srt[lt_t - 1] if lt_t > le_L else -math.inf)
                    assert s["succ"] == (srt[le_t] if le_t < lt_R else math.inf)
                    cases += 1
    assert cases > 1000


# ----------------------------------------------------------------------------- Algorithm 1
def test_appendix_A_kelley_step_is_interior_mean_exact_rationals():
    """with the tightest cuts, step 1.1 equals the arithmetic mean of
    the elements strictly inside the bracket — exact rationals, random tiny instances, all k.
    This is the identity the CUDA driver's iterate relies on (R4)."""
    rng = random.Random(7)
    checked = 0
    for _ in range(600):
        n = rng.randint(3, 9)
        xs = [Fraction(rng.randint(-20, 20), rng.choice([1, 2, 4])) for _ in range(n)]
        srt = sorted(xs)
        for k in range(1, n + 1):
            yL, yR = srt[0], srt[-1]
            for _step in range(n):
                inner = [a for a in xs if yL < a < yR]
                if not inner:
                    break
                fl = [float(a) for a in xs]
                fL, fR = frac_F(fl, yL, k), frac_F(fl, yR, k)
                c_le_L = sum(1 for a in xs if a <= yL)
                c_lt_R = sum(1 for a in xs if a < yR)
                gL = n * (c_le_L - k + Fraction(1, 2))
                gR = n * (c_lt_R - k + Fraction(1, 2))
                if gL >= 0 or gR <= 0:
                    break            # x_(k) is an end point: no interior step
                t = (fR - fL + yL * gL - yR * gR) / (gL - gR)
                assert t == sum(inner) / len(inner)
                checked += 1
                c_lt = sum(1 for a in xs if a < t)
                c_le = sum(1 for a in xs if a <= t)
                if c_lt < k <= c_le:
                    break
                if c_le < k:
                    yL = t
                else:
                    yR = t
    assert checked > 500


def test_cutting_plane_first_iterate_matches_interior_mean():
    for dist in ("uniform", "normal", "mix1"):
        x = datagen.make(dist, 10_001, "f64")
        k = O.median_rank(x.size)
        r = O.cutting_plane(x, k, maxit=1)
        rec = O.init_record(x)
        inner = x[(x > rec["min"]) & (x < rec["max"])]
        assert r["trace"][0][0] == pytest.approx(float(np.mean(inner.astype(O.LD))), rel=1e-9, abs=1e-12)


def test_cutting_plane_exact_all_permutations_and_ranks():
    rng = random.Random(8)
    for n in range(1, 7):
        base = [rng.choice([0.0, 1.0, 1.0, 2.0, -3.0, 1e9, 0.25]) for _ in range(n)]
        for perm in set(itertools.permutations(base)):
            x = np.array(perm, dtype=np.float64)
            for k in range(1, n + 1):
                r = O.cutting_plane(x, k)
                assert r["value"] == brute_kth(list(perm), k)
                assert r["reductions"] <= 64 + 1                       # P:L194 maxit+1


def test_cutting_plane_random_tiny_with_dups_and_signed_zero():
    rng = random.Random(9)
    for xs in tiny_samples(rng, 300):
        for dt in (np.float32, np.float64):
            x = np.array(xs, dtype=dt)
            for k in range(1, x.size + 1):
                for z_cap in (0, 2):
                    r = O.cutting_plane(x, k, z_cap=z_cap)
                    assert r["value"] == brute_kth([dt(a) for a in xs], k)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_cutting_plane_distributions_sizes_ranks(dtype):
    """SPEC acceptance 1, scaled: every distribution x n in {16, 1000, 1e5} x ranks."""
    for dist in datagen.ALL_DISTS:
        for n in (16, 1000, 100_000):
            x = datagen.make(dist, n, dtype)
            for k in sorted({1, 2, O.median_rank(n), n // 10 or 1, n - 1, n}):
                z_cap = max(n // 64, 16)
                r = O.cutting_plane(x, k, z_cap=z_cap)
                assert r["value"] == O.order_statistic(x, k)
                assert r["reductions"] <= 64 + 1


def test_claim_pivot_interval_after_7_iterations():
    """7 CP iterations leave < 2^19 of 2^25 elements (= n/64) in the pivot interval;
    P:L423: z is typically 1-5% of x.  Scaled to n=2^21, median, paper's 9 distributions."""
    n = 1 << 21
    for dist in datagen.PAPER_DISTS:
        x = datagen.make(dist, n, "f32")
        r = O.cutting_plane(x, O.median_rank(n), maxit=7)
        assert r["exit"] in ("maxit", "hit")
        if r["exit"] == "maxit":
            assert r["z_count"] < n / 64
            assert r["z_count"] <= 0.05 * n


def test_claim_outlier_insensitivity():
    """P:L410-416, Fig. 4: CP iteration count is insensitive to a huge outlier (10^3..10^9):
    iterations to reach the n/64 pivot interval vary by <= 2; ~1e20 breaks the
    double-precision sums (more iterations), yet the hybrid finish stays exact."""
    for dtype in ("f32", "f64"):
        x0 = datagen.make("normal", 1 << 16, dtype)
        k = O.median_rank(x0.size)
        its = []
        for M in (1e3, 1e6, 1e9):
            x = datagen.inject_outliers(x0.copy(), 1, M)
            r = O.cutting_plane(x, k, z_cap=x.size // 64)
            assert r["value"] == O.order_statistic(x, k)
            its.append(r["iterations"])
        assert max(its) - min(its) <= 2
        x = datagen.inject_outliers(x0.copy(), 1, 1e20)
        r = O.cutting_plane(x, k, z_cap=x.size // 64)
        assert r["value"] == O.order_statistic(x, k)
        assert r["iterations"] > max(its)


# ----------------------------------------------------------------------------- robust regression
def test_lms_exact_fit_is_zero_and_brute_force():
    """LMS breakdown: if more than half of the rows fit theta* exactly, Med(r^2)=0
    at theta*, and any other theta gives > 0."""
    rng = np.random.default_rng(3)
    n, p = 301, 3
    X = rng.standard_normal((n, p))
    X[:, -1] = 1.0
    th = np.array([2.0, -1.0, 0.5])
    y = X @ th
    bad = rng.random(n) < 0.4
    y[bad] += 50 + rng.standard_normal(bad.sum())
    thetas = np.stack([th, th + 0.1, np.zeros(p)])
    v = O.lms_objective(X, y, thetas)
    assert v[0] == 0.0 and v[1] > 0 and v[2] > 0
    # brute force per column (pure Python sort of a row-by-row residual loop)
    for j, t in enumerate(thetas):
        r2 = sorted((sum(X[i, c] * t[c] for c in range(p)) - y[i]) ** 2 for i in range(n))
        assert v[j] == pytest.approx(r2[O.median_rank(n) - 1], rel=1e-12, abs=1e-20)


def test_lms_median_of_squares_equals_square_of_median_abs_R19():
    rng = np.random.default_rng(4)
    for _ in range(50):
        r = rng.standard_normal(rng.integers(1, 40)).astype(np.float32)
        r2 = (r * r).astype(np.float32)
        k = O.median_rank(r.size)
        assert O.order_statistic(r2, k) == np.float32(O.order_statistic(np.abs(r), k)) ** 2


def test_lts_identity_h_smallest():
    """with a, b from the multiplicity of the threshold, F equals the sum of the h
    smallest squares exactly (engineered ties included)."""
    rng = random.Random(10)
    for _ in range(500):
        n = rng.randint(1, 30)
        rsq = [float(rng.choice([0, 1, 1, 4, 9, 2.25, 16])) if rng.random() < .5 else rng.random()
               for _ in range(n)]
        h = rng.randint(1, n)
        expect = sum(sorted(rsq)[:h])
        assert O.lts_objective(np.array(rsq), h) == pytest.approx(expect, rel=4 * 2.2e-16, abs=1e-300)


# ----------------------------------------------------------------------------- C++ baselines
def test_order_statistic_c_matches_definition():
    """oracle.order_statistic_c (std::nth_element / std::sort on a copy) pinned to the
    definition written out: every k of small random arrays with ties, +-0 and huge magnitudes
    against sorted(list) in Python, for both dtypes; the input is left untouched."""
    rng = np.random.default_rng(7)
    for dtype in (np.float32, np.float64):
        for n in (1, 2, 3, 7, 64, 257):
            x = rng.integers(-5, 6, n).astype(dtype) * rng.choice([1.0, 1e9, 1e-30], n).astype(dtype)
            x[rng.random(n) < 0.2] = -0.0
            before = x.copy()
            s = sorted(float(v) for v in x)
            for k in range(1, n + 1):
                want = s[k - 1] + 0.0
                for method in ("nth_element", "sort"):
                    got = float(O.order_statistic_c(x, k, method))
                    assert got == want and (got != 0 or math.copysign(1, got) == 1), (n, k, method)
            assert np.array_equal(before, x, equal_nan=True)
    with pytest.raises(ValueError):
        O.order_statistic_c(np.ones(3, np.float32), 4)


# ----------------------------------------------------------------------------- kNN via d_(k)
def test_knn_distances_exact_on_integer_grid():
    """float32 squared distances of small-integer points are exact: equal to the integer formula."""
    rng = np.random.default_rng(3)
    X = rng.integers(-20, 21, (50, 4)).astype(np.float32)
    Q = rng.integers(-20, 21, (7, 4)).astype(np.float32)
    D = O.knn_distances_sq(X, Q)
    for j in range(7):
        for i in range(50):
            assert D[j, i] == sum(int(Q[j, l] - X[i, l]) ** 2 for l in range(4))


def test_knn_without_ties_is_mean_of_k_nearest():
    """No ties at d_(k): the rho/a,b reduction = the mean of f over the k nearest points found by a
    full sort (the 'usual approach' of P:L485), uniform and inverse-distance weights."""
    rng = np.random.default_rng(4)
    X = rng.standard_normal((300, 3)).astype(np.float32)
    f = rng.standard_normal(300).astype(np.float32)
    Q = rng.standard_normal((5, 3)).astype(np.float32)
    for k in (1, 2, 17, 300):
        got, dk = O.knn_regress(X, f, Q, k)
        gw, _ = O.knn_regress(X, f, Q, k, weighting=1)
        for j in range(5):
            d = [float(sum((float(Q[j, l]) - float(X[i, l])) ** 2 for l in range(3))) for i in range(300)]
            idx = sorted(range(300), key=lambda i: d[i])[:k]
            assert got[j] == pytest.approx(sum(float(f[i]) for i in idx) / k, rel=1e-12)
            D = O.knn_distances_sq(X, Q)[j]
            w = [1.0 / (float(D[i]) + 1e-12) for i in idx]
            assert gw[j] == pytest.approx(sum(w[q] * float(f[i]) for q, i in enumerate(idx)) / sum(w), rel=1e-9)
            assert dk[j] == np.sort(D)[k - 1]


def test_knn_ties_share_weight_as_the_average_over_tie_choices():
    """Ties at d_(k): rho = a/b is exactly the average, over every way of picking the a missing
    neighbours among the b tied points, of the plain k-nearest mean (exact rationals)."""
    X = np.array([[0.0], [1.0], [-1.0], [2.0], [-2.0], [2.0], [3.0]], np.float32)  # distances 0,1,1,4,4,4,9
    f = np.array([10, 20, 30, 40, 50, 60, 70], np.float32)
    Q = np.zeros((1, 1), np.float32)
    for k in range(1, 8):
        got, _ = O.knn_regress(X, f, Q, k)
        d = [int(x[0]) ** 2 for x in X]
        dk = sorted(d)[k - 1]
        below = [i for i in range(7) if d[i] < dk]
        tied = [i for i in range(7) if d[i] == dk]
        a = k - len(below)
        means = [Fraction(sum(int(f[i]) for i in below + list(c)), k) for c in itertools.combinations(tied, a)]
        assert got[0] == pytest.approx(float(sum(means) / len(means)), rel=1e-15)


def test_bisection_result_and_outlier_sensitivity():
    """oracle.bisection (the paper's comparison driver): the exact element by the definition, and the
    paper's claim P:L413 — its iteration count grows with log2 of the data range (outliers 1e3 ->
    1e9 add ~log2(1e6) ~ 20 iterations) while Kelley's stays within 2 (Fig. 4)."""
    rng = np.random.default_rng(12)
    x = rng.random(20001)
    for k in (1, 7, 10001, 20000, 20001):
        assert O.bisection(x, k, z_cap=0)["value"] == np.sort(x)[k - 1]
    its, cps = [], []
    for mag in (1e3, 1e9):
        y = x.copy()
        y[rng.choice(y.size, 20, replace=False)] = mag
        its.append(O.bisection(y, O.median_rank(y.size), z_cap=64)["iterations"])
        cps.append(O.cutting_plane(y, O.median_rank(y.size), z_cap=64)["iterations"])
        assert O.bisection(y, O.median_rank(y.size), z_cap=64)["value"] == np.sort(y)[O.median_rank(y.size) - 1]
    assert its[1] - its[0] >= 15, its
    assert abs(cps[1] - cps[0]) <= 2, cps


def test_brent_root_result_and_outlier_sensitivity():
    """oracle.brent_root (zbrent on the count function): the exact element by the definition for
    every kind of rank, and the paper's claim (Brent's root finder 'degraded when data
    contained very large outliers', reverting to bisection steps): 1e9 outliers cost >= 10 more
    iterations than 1e3, the cutting plane none."""
    rng = np.random.default_rng(5)
    x = rng.random(20001)
    for k in (1, 2, 7, 10001, 19999, 20001):
        assert O.brent_root(x, k)["value"] == np.sort(x)[k - 1]
    xd = np.floor(256 * rng.random(5001)).astype(np.float32)   # many duplicates
    for k in (1, 100, 2501, 5001):
        assert O.brent_root(xd, k)["value"] == np.sort(xd)[k - 1]
    its, cps = [], []
    for mag in (1e3, 1e9):
        y = x.copy()
        y[rng.choice(y.size, 20, replace=False)] = mag
        its.append(O.brent_root(y, 10001, z_cap=64)["iterations"])
        cps.append(O.cutting_plane(y, 10001, z_cap=64)["iterations"])
    assert its[1] - its[0] >= 10, its
    assert abs(cps[1] - cps[0]) <= 2, cps


def test_knn_classify_is_the_majority_of_the_k_nearest():
    """No ties at d_(k): the vote equals the class counts among the k nearest by a full sort, the
    winner their majority (smallest class on a tie); with ties the votes sum to k exactly."""
    rng = np.random.default_rng(8)
    X = rng.standard_normal((400, 2)).astype(np.float32)
    lab = rng.integers(0, 5, 400).astype(np.int32)
    Q = rng.standard_normal((6, 2)).astype(np.float32)
    for k in (1, 5, 40):
        cls, votes = O.knn_classify(X, lab, Q, k, 5)
        D = O.knn_distances_sq(X, Q)
        for j in range(6):
            idx = np.argsort(D[j], kind="stable")[:k]
            cnt = np.bincount(lab[idx], minlength=5)
            assert np.array_equal(votes[j], cnt.astype(np.float64))
            assert cls[j] == int(np.argmax(cnt))
    Xg = np.array([[0.0], [1.0], [-1.0], [2.0], [-2.0]], np.float32)          # ties at distance 1, 4
    cls, votes = O.knn_classify(Xg, np.array([0, 1, 2, 1, 2], np.int32), np.zeros((1, 1), np.float32), 2, 3)
    assert votes[0].tolist() == [1.0, 0.5, 0.5] and cls[0] == 0


def test_brent_min_step_tracks_an_independent_brent():
    """oracle.BrentMinStep (NR `brent`, the paper's 'Brent's method of optimization', P:L136,
    P:L229) against scipy's fminbound — an independent implementation of Brent's method from the
    same golden-section starting point: the evaluation points agree through the golden and the
    parabolic phases (up to NR's 7-digit golden constant) until the steps reach the tolerance.
    A wrong sign or operand in the parabola, or a wrong bracket update, leaves that path."""
    from scipy.optimize import fminbound
    for f, a, b in ((lambda u: math.exp(u) - 2.0 * u + 0.1 * math.sin(5.0 * u), 0.0, 3.0),
                    (lambda u: abs(u - 0.3) ** 1.5 + 0.2 * u * u, -2.0, 1.0),
                    (lambda u: (u - 7.25) ** 2 * (1.0 + 0.01 * u), 0.0, 100.0)):
        pts = []

        def g(u):
            pts.append(float(u))
            return f(float(u))

        fminbound(g, a, b, xtol=1e-12, maxfun=60)
        br = O.BrentMinStep(a, b)
        mine = []
        for _ in range(8):
            u = br.propose()
            mine.append(u)
            br.accept(u, f(u), a, b)
        assert np.allclose(mine, pts[:8], rtol=0, atol=1e-6 * (b - a)), (mine, pts[:8])
    # a linear function: every parabola is rejected (collinear points) -> pure golden-section steps
    br = O.BrentMinStep(0.0, 1.0)
    pts = []
    for _ in range(6):
        u = br.propose()
        pts.append(u)
        br.accept(u, u, 0.0, 1.0)
    # golden section toward the minimum at 0: 0.381966, then the larger segment's golden point
    # 0.618034 (worse: b <- it), then x shrinks by 1 - CGOLD = 0.618034 per step
    assert pts[0] == pytest.approx(0.381966, abs=1e-12) and pts[1] == pytest.approx(0.618034, abs=1e-6)
    assert all(pts[i + 1] / pts[i] == pytest.approx(0.618034, abs=1e-6) for i in range(2, 5))


def test_brent_min_result_and_outlier_sensitivity():
    """oracle.brent_min: the exact element by the definition for every kind of rank (the hybrid
    finish after NR's convergence), and the paper's claim (Fig. 4 caption P:L514: with very
    large outliers F is linear over most of the range, the parabolic fits fail and Brent's method
    reverts to golden section): 1e9 outliers cost >= 10 more iterations than 1e3, the cutting plane
    none.  brent_min_replay driven by brent_min's own F values retraces it exactly."""
    rng = np.random.default_rng(5)
    x = rng.random(20001)
    for k in (1, 2, 7, 10001, 19999, 20001):
        r = O.brent_min(x, k)
        assert r["value"] == np.sort(x)[k - 1]
        assert r["iterations"] < 60
    xd = np.floor(256 * rng.random(5001)).astype(np.float32)   # many duplicates
    for k in (1, 100, 2501, 5001):
        assert O.brent_min(xd, k)["value"] == np.sort(xd)[k - 1]
    its, cps = [], []
    for mag in (1e3, 1e9):
        y = x.copy()
        y[rng.choice(y.size, 20, replace=False)] = mag
        its.append(O.brent_min(y, 10001, z_cap=64)["iterations"])
        cps.append(O.cutting_plane(y, 10001, z_cap=64)["iterations"])
    assert its[1] - its[0] >= 10, its
    assert abs(cps[1] - cps[0]) <= 2, cps
    r = O.brent_min(x, 10001)
    rp = O.brent_min_replay(x, 10001, [row[1] for row in r["trace"]])
    assert rp["trace"] == r["trace"] and rp["value"] == r["value"]
