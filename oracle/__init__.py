"""CPU oracle for the cutting-plane order-statistic path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  The product path (paper_1104_2732_b200, libcpsel.so)
never imports, links or executes anything here, and this package imports nothing
from the product path.  It shares no code with the CUDA kernels; the only common
dependency is the seeded input generator in datagen/ (which holds no method
arithmetic).

Plain, slow, obviously correct: numpy for whole-array steps (a library sort /
partition is used only as the "sort" step the paper itself names), Python
integers for counts, np.longdouble (80-bit on x86) for sums, fractions.Fraction
for exact subgradients.  Every function cites the PAPER.md line it follows
(P:Lnnn = /root/reference/PAPER.md line nnn).  Readings where the paper is silent
or inconsistent are numbered R1..R20 and listed in DESIGN.md §3.

Pins (tests/test_oracle_pins.py) tie every function to something other than
itself: brute-force rank definition on tiny inputs, exact-rational finite
differences, the paper's closed forms, SPEC worked examples under
tests/golden/, the Appendix-A identity in exact rationals, and the paper's
algorithmic claims.
parity unpinned: none of the functions below (the iteration-count claims are
only bounds, see DESIGN.md §3 "pins").
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

LD = np.longdouble


# ============================================================================ helpers
def _as_array(x) -> np.ndarray:
    x = np.asarray(x)
    if x.dtype not in (np.float32, np.float64):
        x = x.astype(np.float64)
    return x


def _f64(v):
    """Comparison value as a *strong* float64 scalar: numpy then promotes a float32 array to
    float64 before comparing (a bare Python float would be rounded to float32 under NEP 50)."""
    return np.float64(v)


def canonical(v):
    """-0.0 -> +0.0 (reading R13: ±0 compare equal; the returned bits are canonical)."""
    return v + type(v)(0) if v == 0 else v


def check_input(x, k: int) -> int:
    """Validation of the selection problem (SPEC S:L61-62 rank range, S:L85 NaN rejected).

    Returns n.  Raises ValueError on n==0, k out of [1,n] or a non-finite element (R12).
    """
    x = _as_array(x)
    n = x.size
    if n == 0:
        raise ValueError("empty sample")
    if not (1 <= k <= n):
        raise ValueError(f"rank k={k} out of [1,{n}]")
    if not np.all(np.isfinite(x)):
        raise ValueError("non-finite element")
    return n


def median_rank(n: int) -> int:
    """Med(x) = x_([(n+1)/2]), [t] the integer part — the lower median (R3)."""
    return (n + 1) // 2


# ============================================================================ plain definition
def order_statistic(x, k: int):
    """x_(k): the k-th smallest element (P:L19 abstract).

    Plain definition: sort (here: numpy's partition, a library selection primitive)
    and take position k-1.  Returned in the input dtype, canonical zero (R13).
    """
    x = _as_array(x)
    check_input(x, k)
    return canonical(np.partition(x, k - 1)[k - 1])


def order_statistic_sorted(x, k: int):
    """Second, independent path: full sort then index (P:L37 'sort the elements ... and select')."""
    x = _as_array(x)
    check_input(x, k)
    return canonical(np.sort(x, kind="stable")[k - 1])


def median(x):
    """Med(x)."""
    x = _as_array(x)
    return order_statistic(x, median_rank(x.size))


def rank_counts(x, v):
    """(#{x_i < v}, #{x_i = v}) with IEEE comparisons (P:L130 'count' terms)."""
    x = _as_array(x)
    v = _f64(v)
    return int(np.count_nonzero(x < v)), int(np.count_nonzero(x == v))


# ============================================================================ objectives (Eq. 1, Eq. 2)
def f_median(x, y) -> LD:
    """Eq. (1) objective f(y) = sum_i |x_i - y|, long-double sum."""
    xl = _as_array(x).astype(LD)
    return LD(np.sum(np.abs(xl - LD(y))))


def u_paper(t, n: int, kp: int):
    """Eq. (2) penalty exactly as printed:
    u(t) = (n-kp+1/2) t for t >= 0, -(kp-1/2) t for t < 0.
    """
    t = np.asarray(t, dtype=LD)
    return np.where(t >= 0, (LD(n) - LD(kp) + LD(0.5)) * t, -(LD(kp) - LD(0.5)) * t)


def paper_k(n: int, k: int) -> int:
    """Eq. (2)'s k selects the k-th LARGEST element (reading R2);
    the API's k-th smallest is Eq. (2) with paper-k = n-k+1."""
    return n - k + 1


def f_os(x, y, k: int) -> LD:
    """F_k(y) = sum_i u(x_i - y) (Eq. 2) for the k-th smallest (R2)."""
    x = _as_array(x)
    n = x.size
    t = x.astype(LD) - LD(y)
    return LD(np.sum(u_paper(t, n, paper_k(n, k))))


# ============================================================================ subdifferentials
def g_paper(x, y):
    """The set-valued g of P:L130 *as printed*:
    g(y) = count(x_i>y) + count(x_i<y)(-1) + count(x_i=y)[-1,1]   (Minkowski sum).
    Returned as the exact interval (lo, hi).  Reading R1: this is -df; see subdiff_median.
    """
    x = _as_array(x)
    c_lt, c_eq = rank_counts(x, y)
    c_gt = x.size - c_lt - c_eq
    return (c_gt - c_lt - c_eq, c_gt - c_lt + c_eq)


def subdiff_median(x, y):
    """Clarke subdifferential of Eq. (1) (with d|t| of P:L122-127):
    each |x_i - y| contributes -1 (x_i>y), +1 (x_i<y), [-1,1] (x_i=y); Minkowski sum.
    Exact integer interval (lo, hi)."""
    x = _as_array(x)
    c_lt, c_eq = rank_counts(x, y)
    c_gt = x.size - c_lt - c_eq
    return (c_lt - c_gt - c_eq, c_lt - c_gt + c_eq)


def subdiff_os(x, y, k: int):
    """Subdifferential of F_k(y) = sum_i u(x_i - y) (Eq. 2), term by term as in P:L128-132:
    d/dy u(x_i - y) = -u'(x_i - y); u' = (n-kp+1/2) on t>0, -(kp-1/2) on t<0,
    [-(kp-1/2), n-kp+1/2] at t=0.  Exact Fractions (lo, hi)."""
    x = _as_array(x)
    n = x.size
    kp = paper_k(n, k)
    wpos = Fraction(2 * (n - kp) + 1, 2)   # slope of u for t >= 0
    wneg = Fraction(2 * kp - 1, 2)         # -slope of u for t < 0
    c_lt, c_eq = rank_counts(x, y)
    c_gt = n - c_lt - c_eq
    # x_i > y : t>0, d/dy = -wpos ; x_i < y : t<0, d/dy = +wneg ; x_i = y : [-wpos, +wneg]
    lo = c_lt * wneg - c_gt * wpos - c_eq * wpos
    hi = c_lt * wneg - c_gt * wpos + c_eq * wneg
    return lo, hi


# ============================================================================ reductions used by Algorithm 1
def init_record(x):
    """The single init reduction of P:L155/P:L194: y_L = x_(1), y_R = x_(n), sum x_i
    (+ the multiplicities of min and max, reading R5)."""
    x = _as_array(x)
    mn, mx = x.min(), x.max()
    return {
        "min": canonical(mn), "cnt_min": int(np.count_nonzero(x == mn)),
        "max": canonical(mx), "cnt_max": int(np.count_nonzero(x == mx)),
        "sum": LD(np.sum(x.astype(LD))),
    }


def pass_stats(x, t, y_lo, y_hi):
    """Everything one objective pass at t can report (Fig. 1):
      c_lt = #{x<t}, c_eq = #{x=t}                           (subgradient counts)
      P = sum (x-t)^+, N = sum (t-x)^+                         (F's two halves, direct)
      L_lo = sum_{y_lo<x<t} (t-x), L_hi = sum_{t<x<y_hi} (x-t) (bracket-local sums)
      pred = max{x : y_lo<x<t} (-inf if none), succ = min{x : t<x<y_hi} (+inf if none)
      (P:L192 footnote 'largest x_i <= y~', restricted to the bracket)
    Sums in long double."""
    x = _as_array(x)
    xl = x.astype(LD)
    t_ = LD(t)
    t, y_lo, y_hi = _f64(t), _f64(y_lo), _f64(y_hi)
    lt, gt, eq = x < t, x > t, x == t
    lo_in = lt & (x > y_lo)
    hi_in = gt & (x < y_hi)
    return {
        "c_lt": int(np.count_nonzero(lt)), "c_eq": int(np.count_nonzero(eq)),
        "P": LD(np.sum(xl[gt] - t_)), "N": LD(np.sum(t_ - xl[lt])),
        "L_lo": LD(np.sum(t_ - xl[lo_in])), "L_hi": LD(np.sum(xl[hi_in] - t_)),
        "c_lo": int(np.count_nonzero(lo_in)), "c_hi": int(np.count_nonzero(hi_in)),
        "pred": float(x[lo_in].max()) if lo_in.any() else -math.inf,
        "succ": float(x[hi_in].min()) if hi_in.any() else math.inf,
    }


def F_from_PN(n: int, k: int, P, N) -> LD:
    """F_k = (k-1/2) P + (n-k+1/2) N (Eq. 2 with paper-k = n-k+1, R2)."""
    return (LD(k) - LD(0.5)) * LD(P) + (LD(n) - LD(k) + LD(0.5)) * LD(N)


# ============================================================================ Algorithm 1 (literal)
def hybrid_finish(x, k: int, y_L, y_R):
    """Second stage of the hybrid method (Fig. 1 SortZ P:L284-294):
    z = {x_i : y_L < x_i < y_R} (copy_if), sort z, return z_(k-m) with
    m = #{x_i <= y_L} (reading R3: 1-based rank k-m, i.e. 0-based index k-m-1)."""
    x = _as_array(x)
    y_L, y_R = _f64(y_L), _f64(y_R)
    m = int(np.count_nonzero(x <= y_L))
    z = np.sort(x[(x > y_L) & (x < y_R)])
    if not (1 <= k - m <= z.size):
        raise AssertionError("bracket does not contain the k-th order statistic")
    return canonical(z[k - m - 1]), int(z.size)


def cutting_plane(x, k: int, maxit: int = 64, z_cap: int = 0, tol_f: float | None = None):
    """Kelley's cutting plane method, Algorithm 1, for F_k (Eq. 2), followed by
    the hybrid finish.  Straightforward double precision:

    step 0: one reduction -> y_L=x_(1), y_R=x_(n), sum x; then the closed
        forms F(y_L) = (k-1/2)(sum x - n y_L), F(y_R) = (n-k+1/2)(n y_R - sum x)
        (Eq. 1's f(y_L)=sum x - n y_L, f(y_R)=n y_R - sum x, weighted per Eq. 2) and
        g_L = right end of dF(y_L), g_R = left end of dF(y_R) (R4 tightest cuts, R5 multiplicity).
        If k <= cnt_min -> x_(1); if k > n-cnt_max -> x_(n).
    step 1.1: t = (fR - fL + y_L gL - y_R gR)/(gL - gR) in double; if rounding puts t
        outside ]y_L, y_R[ the midpoint is used and counted as a fallback.
    step 1.2: ft = F(t) by a direct long-double reduction, gt = dF(t) (exact interval).
    step 1.3: stop if 0 in dF(t) (t is then x_(k)); or if the bracket interior
        #{y_L<x<y_R} <= z_cap (R7/R8: the count replaces tolerance_f); or, when tol_f is
        given, the paper's own y_R - y_L <= tolerance_f.
    step 1.4 (sign fixed per R1): dF(t) < 0 -> y_L <- t (gL = right end),
        else y_R <- t (gR = left end).
    step 2 / hybrid: the exact finish by copy_if + sort.

    Returns dict(value, iterations, reductions, fallbacks, trace, y_L, y_R, z_count, exit).
    trace rows: (t, F(t), c_lt, c_eq, interior count after the update).
    """
    x = _as_array(x)
    n = check_input(x, k)
    rec = init_record(x)
    reductions = 1
    yL, yR = float(rec["min"]), float(rec["max"])
    base = {"iterations": 0, "reductions": reductions, "fallbacks": 0, "trace": [],
            "y_L": yL, "y_R": yR, "z_count": 0}
    if k <= rec["cnt_min"]:
        return dict(base, value=rec["min"], exit="init_min")
    if k > n - rec["cnt_max"]:
        return dict(base, value=rec["max"], exit="init_max")
    S = rec["sum"]
    fL = float((LD(k) - LD(0.5)) * (S - LD(n) * LD(yL)))
    fR = float((LD(n) - LD(k) + LD(0.5)) * (LD(n) * LD(yR) - S))
    gL = float(Fraction(n * (2 * rec["cnt_min"] - 2 * k + 1), 2))            # dF+(y_L)
    gR = float(Fraction(n * (2 * (n - rec["cnt_max"]) - 2 * k + 1), 2))      # dF-(y_R)
    c_le_L = rec["cnt_min"]            # #{x <= y_L}
    c_lt_R = n - rec["cnt_max"]        # #{x <  y_R}
    trace, fallbacks, exit_reason, value = [], 0, "maxit", None
    it = 0
    for it in range(1, maxit + 1):
        t = (fR - fL + yL * gL - yR * gR) / (gL - gR)                       # step 1.1
        if not (yL < t < yR):
            t = 0.5 * (yL + yR)
            fallbacks += 1
        ft = float(f_os(x, t, k))                                             # step 1.2
        lo, hi = subdiff_os(x, t, k)
        reductions += 1
        c_lt, c_eq = rank_counts(x, t)
        if lo <= 0 <= hi:                                                     # step 1.3
            trace.append((t, ft, c_lt, c_eq, 0))
            value, exit_reason = canonical(x.dtype.type(t)), "hit"
            break
        if hi < 0:                                                            # step 1.4
            yL, fL, gL, c_le_L = t, ft, float(hi), c_lt + c_eq
        else:
            yR, fR, gR, c_lt_R = t, ft, float(lo), c_lt
        interior = c_lt_R - c_le_L
        trace.append((t, ft, c_lt, c_eq, interior))
        if interior <= z_cap:
            exit_reason = "z_cap"
            break
        if tol_f is not None and yR - yL <= tol_f:
            exit_reason = "tol_f"
            break
    z_count = 0
    if value is None:                                                         # step 2 + hybrid
        value, z_count = hybrid_finish(x, k, yL, yR)
    return {"value": value, "iterations": it, "reductions": reductions, "fallbacks": fallbacks,
            "trace": trace, "y_L": yL, "y_R": yR, "z_count": z_count, "exit": exit_reason}


def bisection(x, k: int, maxit: int = 400, z_cap: int = 0):
    """The paper's bisection comparison ("we adapted the classical bisection method", P:L204:
    "methods based on solving 0 in g(y)"): from [y_L, y_R] = [x_(1), x_(n)], t = (y_L + y_R)/2 in
    double, rounded to the data's dtype; 0 in dF_k(t) (c_lt < k <= c_le) -> t; dF_k(t) < 0 (c_le < k)
    -> y_L <- t, else y_R <- t; until the bracket interior holds <= z_cap elements, then the hybrid
    finish.  Its iteration count grows like log2 of the data range.
    Returns dict(value, iterations, trace=[(t, c_lt, c_eq, interior)])."""
    x = _as_array(x)
    n = check_input(x, k)
    rec = init_record(x)
    if k <= rec["cnt_min"]:
        return {"value": rec["min"], "iterations": 0, "trace": []}
    if k > n - rec["cnt_max"]:
        return {"value": rec["max"], "iterations": 0, "trace": []}
    yL, yR = float(rec["min"]), float(rec["max"])
    c_le_L, c_lt_R = rec["cnt_min"], n - rec["cnt_max"]
    trace = []
    for it in range(1, maxit + 1):
        t = float(x.dtype.type(0.5 * yL + 0.5 * yR))
        if not (yL < t < yR):  # adjacent floats: nothing strictly inside, the finish decides
            break
        c_lt, c_eq = rank_counts(x, t)
        if c_lt < k <= c_lt + c_eq:
            trace.append((t, c_lt, c_eq, 0))
            return {"value": canonical(x.dtype.type(t)), "iterations": it, "trace": trace}
        if c_lt + c_eq < k:
            yL, c_le_L = t, c_lt + c_eq
        else:
            yR, c_lt_R = t, c_lt
        trace.append((t, c_lt, c_eq, c_lt_R - c_le_L))
        if c_lt_R - c_le_L <= z_cap:
            break
    value, _ = hybrid_finish(x, k, yL, yR)
    return {"value": value, "iterations": it, "trace": trace}


def _snap(t: float, yL: float, yR: float, dt):
    """t rounded to the dtype and nudged strictly inside ]yL, yR[ (reading R9)."""
    f = dt(t) if math.isfinite(t) else dt(0.5 * yL + 0.5 * yR)
    if not f > dt(yL):
        f = np.nextafter(dt(yL), dt(math.inf))
    if not f < dt(yR):
        f = np.nextafter(dt(yR), dt(-math.inf))
    return float(f)


def brent_root(x, k: int, maxit: int = 400, z_cap: int = 0):
    """The paper's Brent root-finding comparison ("the method of parabolas combined with golden
    section, which is also known as Brent algorithm [NR]", "solving 0 in g(y)"): Numerical
    Recipes' zbrent, literally, on f(t) = c_lt(t) + c_le(t) - 2k + 1 (an integer: < 0 below x_(k),
    > 0 above, so its sign change is the target), each proposed point rounded into the open
    bracket (R9); 0 in dF_k(t) -> t; the exact bracket [y_L, y_R] from the counts as in
    `bisection`; stop when the interior holds <= z_cap elements, then the hybrid finish.
    Returns dict(value, iterations, trace=[(t, c_lt, c_eq, interior)])."""
    x = _as_array(x)
    n = check_input(x, k)
    dt = x.dtype.type
    rec = init_record(x)
    if k <= rec["cnt_min"]:
        return {"value": rec["min"], "iterations": 0, "trace": []}
    if k > n - rec["cnt_max"]:
        return {"value": rec["max"], "iterations": 0, "trace": []}
    yL, yR = float(rec["min"]), float(rec["max"])
    c_le_L, c_lt_R = rec["cnt_min"], n - rec["cnt_max"]
    eps = 2.220446049250313e-16
    a, fa = yL, 2.0 * c_le_L - 2.0 * k + 1.0
    b, fb = yR, 2.0 * c_lt_R - 2.0 * k + 1.0
    c, fc = b, fb
    d = e = b - a
    trace = []
    it = 0
    for it in range(1, maxit + 1):
        if (fb > 0 and fc > 0) or (fb < 0 and fc < 0):
            c, fc = a, fa
            e = d = b - a
        if abs(fc) < abs(fb):
            a, b, c = b, c, b
            fa, fb, fc = fb, fc, fb
        tol1 = 2.0 * eps * abs(b)
        xm = 0.5 * (c - b)
        if abs(e) >= tol1 and abs(fa) > abs(fb):
            s_ = fb / fa
            if a == c:
                p_ = 2.0 * xm * s_
                q_ = 1.0 - s_
            else:
                qq, r_ = fa / fc, fb / fc
                p_ = s_ * (2.0 * xm * qq * (qq - r_) - (b - a) * (r_ - 1.0))
                q_ = (qq - 1.0) * (r_ - 1.0) * (s_ - 1.0)
            if p_ > 0:
                q_ = -q_
            p_ = abs(p_)
            if 2.0 * p_ < min(3.0 * xm * q_ - abs(tol1 * q_), abs(e * q_)):
                e = d
                d = p_ / q_
            else:
                d = xm
                e = d
        else:
            d = xm
            e = d
        t = _snap(b + (d if abs(d) > tol1 else (tol1 if xm >= 0 else -tol1)), yL, yR, dt)
        if not (yL < t < yR):
            break
        c_lt, c_eq = rank_counts(x, t)
        a, fa = b, fb
        b, fb = t, float(c_lt + c_lt + c_eq) - 2.0 * k + 1.0
        if c_lt < k <= c_lt + c_eq:
            trace.append((t, c_lt, c_eq, 0))
            return {"value": canonical(dt(t)), "iterations": it, "trace": trace}
        if c_lt + c_eq < k:
            yL, c_le_L = t, c_lt + c_eq
        else:
            yR, c_lt_R = t, c_lt
        trace.append((t, c_lt, c_eq, c_lt_R - c_le_L))
        if c_lt_R - c_le_L <= z_cap:
            break
    value, _ = hybrid_finish(x, k, yL, yR)
    return {"value": value, "iterations": it, "trace": trace}


class BrentMinStep:
    """Numerical Recipes' `brent` (parabolic interpolation, golden section when the parabola is
    rejected), the paper's 'Brent's method of optimization' (P:L113, P:L136, P:L204, P:L226,
    P:L229), literally, one evaluation at a time so that a run can be driven by any F values
    (the oracle's own in `brent_min`, a GPU trace's in `brent_min_replay`).  Reading R37: Brent's
    own bracket [a, b] is kept as NR keeps it and then intersected with the exact bracket
    [y_L, y_R] that the counts give (convexity of F makes both valid; the counts are exact);
    the first point is NR's golden-section point of [y_L, y_R]."""
    CGOLD = 0.3819660
    TOL = 1.4901161193847656e-08   # sqrt(DBL_EPSILON) (NR: ~ the square root of the precision)
    ZEPS = 1.0e-10

    def __init__(self, yL: float, yR: float):
        self.a, self.b = yL, yR
        self.x = self.w = self.v = yL + self.CGOLD * (yR - yL)
        self.fx = self.fw = self.fv = math.nan
        self.d = self.e = 0.0
        self.started = False

    def propose(self):
        """The next point, or None once NR's convergence test holds (then the hybrid finish)."""
        if not self.started:
            return self.x
        a, b, x, w, v = self.a, self.b, self.x, self.w, self.v
        fx, fw, fv = self.fx, self.fw, self.fv
        xm = 0.5 * (a + b)
        tol1 = self.TOL * abs(x) + self.ZEPS
        tol2 = 2.0 * tol1
        if abs(x - xm) <= tol2 - 0.5 * (b - a):  # NR's convergence test: brent returns x
            return None
        if abs(self.e) > tol1:
            r = (x - w) * (fx - fv)
            q = (x - v) * (fx - fw)
            p = (x - v) * q - (x - w) * r
            q = 2.0 * (q - r)
            if q > 0.0:
                p = -p
            q = abs(q)
            etemp = self.e
            self.e = self.d
            if abs(p) >= abs(0.5 * q * etemp) or p <= q * (a - x) or p >= q * (b - x):
                self.e = (a - x) if x >= xm else (b - x)
                self.d = self.CGOLD * self.e
            else:
                self.d = p / q
                u = x + self.d
                if u - a < tol2 or b - u < tol2:
                    self.d = abs(tol1) if xm - x >= 0.0 else -abs(tol1)
        else:
            self.e = (a - x) if x >= xm else (b - x)
            self.d = self.CGOLD * self.e
        return x + self.d if abs(self.d) >= tol1 else x + (abs(tol1) if self.d >= 0.0 else -abs(tol1))

    def accept(self, u: float, fu: float, yL: float, yR: float):
        """F(u) = fu; [yL, yR] is the exact bracket after u's counts."""
        if not self.started:  # the first evaluation: x = w = v = u
            self.x = self.w = self.v = u
            self.fx = self.fw = self.fv = fu
            self.started = True
        elif fu <= self.fx:
            if u >= self.x:
                self.a = self.x
            else:
                self.b = self.x
            self.v, self.w, self.x = self.w, self.x, u
            self.fv, self.fw, self.fx = self.fw, self.fx, fu
        else:
            if u < self.x:
                self.a = u
            else:
                self.b = u
            if fu <= self.fw or self.w == self.x:
                self.v, self.w = self.w, u
                self.fv, self.fw = self.fw, fu
            elif fu <= self.fv or self.v == self.x or self.v == self.w:
                self.v, self.fv = u, fu
        self.a = max(self.a, yL)
        self.b = min(self.b, yR)


def _brent_min_run(x, k: int, maxit: int, z_cap: int, F_of):
    """Shared loop of brent_min / brent_min_replay: F_of(it, t) gives F_k(t) for iteration it."""
    x = _as_array(x)
    n = check_input(x, k)
    dt = x.dtype.type
    rec = init_record(x)
    if k <= rec["cnt_min"]:
        return {"value": rec["min"], "iterations": 0, "trace": []}
    if k > n - rec["cnt_max"]:
        return {"value": rec["max"], "iterations": 0, "trace": []}
    yL, yR = float(rec["min"]), float(rec["max"])
    c_le_L, c_lt_R = rec["cnt_min"], n - rec["cnt_max"]
    br = BrentMinStep(yL, yR)
    trace = []
    it = 0
    for it in range(1, maxit + 1):
        u = br.propose()
        if u is None:
            break
        t = _snap(u, yL, yR, dt)
        if not (yL < t < yR):
            break
        c_lt, c_eq = rank_counts(x, t)
        F = F_of(it, t)
        if c_lt < k <= c_lt + c_eq:
            trace.append((t, F, c_lt, c_eq, 0))
            return {"value": canonical(dt(t)), "iterations": it, "trace": trace}
        if c_lt + c_eq < k:
            yL, c_le_L = t, c_lt + c_eq
        else:
            yR, c_lt_R = t, c_lt
        br.accept(t, F, yL, yR)
        trace.append((t, F, c_lt, c_eq, c_lt_R - c_le_L))
        if c_lt_R - c_le_L <= z_cap:
            break
    value, _ = hybrid_finish(x, k, yL, yR)
    return {"value": value, "iterations": it, "trace": trace}


def brent_min(x, k: int, maxit: int = 400, z_cap: int = 0):
    """The paper's 'Brent's method of optimization' comparison: NR
    `brent` minimising F_k (Eq. 2, R2) with F from long-double direct sums (f_os), each proposed
    point rounded into the exact open bracket (R9); 0 in dF_k(t) -> t; the exact bracket
    [y_L, y_R] from the counts as in `bisection` (R37); stop when the interior holds <= z_cap
    elements or NR's convergence test holds, then the hybrid finish.  The paper (Fig. 4): with very large
    outliers F is linear over most of the range, the parabolic fits fail and Brent reverts to
    golden section — its iteration count grows with the range.
    Returns dict(value, iterations, trace=[(t, F, c_lt, c_eq, interior)])."""
    xa = _as_array(x)
    return _brent_min_run(xa, k, maxit, z_cap, lambda it, t: float(f_os(xa, t, k)))


def brent_min_replay(x, k: int, F_values, maxit: int = 400, z_cap: int = 0):
    """brent_min driven by given F values (F_values[i] = F at iteration i+1, e.g. a GPU trace's):
    the points it proposes are exactly what a correct implementation of the same steps proposes
    from those F values; the counts are the oracle's own."""
    xa = _as_array(x)
    return _brent_min_run(xa, k, min(maxit, len(F_values)), z_cap, lambda it, t: float(F_values[it - 1]))


def eval_at(x, k: int, t, y_lo, y_hi):
    """Replay hook: one pass at t (pass_stats) plus F_k(t) and dF_k(t) — compared against the
    GPU's cpsel_eval / trace at identical t."""
    s = pass_stats(x, t, y_lo, y_hi)
    n = _as_array(x).size
    s["F"] = F_from_PN(n, k, s["P"], s["N"])
    s["subdiff"] = subdiff_os(x, t, k)
    return s


# ============================================================================ robust regression (§6)
def lms_residuals_sq(X, y, thetas):
    """r_i(theta) = f_theta(x_i) - y_i (model P:L440) and r_i^2, in float64.
    X: n x p, y: n, thetas: C x p (theta_j as rows).  Returns S (n x C) float64."""
    X64 = np.asarray(X, dtype=np.float64)
    y64 = np.asarray(y, dtype=np.float64)
    T64 = np.asarray(thetas, dtype=np.float64)
    R = X64 @ T64.T - y64[:, None]
    return R * R


def lms_objective(X, y, thetas):
    """LMS objective F(theta_j) = Med(r_i(theta_j)^2) per candidate (reading R19: median of
    the squared residuals, lower median P:L32).  float64 result per column."""
    S = lms_residuals_sq(X, y, thetas)
    n = S.shape[0]
    k = median_rank(n)
    return np.array([np.partition(S[:, j], k - 1)[k - 1] for j in range(S.shape[1])])


def lts_objective(rsq, h: int):
    """LTS objective via the rho reformulation, reading R20:
    m = (r^2)_(h); b_L = #{r^2 < m}; b = #{r^2 = m}; a = h - b_L;
    F = sum_{r^2<m} r^2 + (a/b) sum_{r^2=m} r^2   (= sum of the h smallest squares)."""
    r = np.asarray(rsq, dtype=np.float64)
    m = np.partition(r, h - 1)[h - 1]
    bL = int(np.count_nonzero(r < m))
    b = int(np.count_nonzero(r == m))
    a = h - bL
    return float(np.sum(r[r < m].astype(LD)) + LD(a) / LD(b) * np.sum(r[r == m].astype(LD)))


# ============================================================================ C++ baselines
_CLIB = None


def _clib():
    """oracle/liboracle_c.so (built by __graft_entry__.build() from oracle/cselect.cpp)."""
    global _CLIB
    if _CLIB is None:
        import ctypes
        import os
        p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liboracle_c.so")
        if not os.path.exists(p):
            build_c()
        lib = ctypes.CDLL(p)
        for name, ct in (("f32", ctypes.c_float), ("f64", ctypes.c_double)):
            for fn in ("oracle_nth_element_", "oracle_sort_select_"):
                f = getattr(lib, fn + name)
                f.restype = ctypes.c_double
                f.argtypes = [ctypes.POINTER(ct), ctypes.c_uint64, ctypes.c_uint64]
        _CLIB = lib
    return _CLIB


def build_c() -> str:
    """Compile oracle/cselect.cpp (g++ -O2, single thread) into oracle/liboracle_c.so."""
    import os
    import subprocess
    d = os.path.dirname(os.path.abspath(__file__))
    out = os.path.join(d, "liboracle_c.so")
    subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", out + ".tmp",
                    os.path.join(d, "cselect.cpp")], check=True)
    os.replace(out + ".tmp", out)
    return out


def order_statistic_c(x, k: int, method: str = "nth_element"):
    """x_(k) by the C++ std::nth_element (the paper's CPU quickselect row) or
    std::sort on a copy — the single-core CPU baselines of SURVEY §8(d)."""
    import ctypes
    x = np.ascontiguousarray(_as_array(x))
    n = check_input(x, k)
    name = ("oracle_nth_element_" if method == "nth_element" else "oracle_sort_select_") + \
        ("f32" if x.dtype == np.float32 else "f64")
    ct = ctypes.c_float if x.dtype == np.float32 else ctypes.c_double
    v = getattr(_clib(), name)(x.ctypes.data_as(ctypes.POINTER(ct)), n, k)
    return canonical(x.dtype.type(v))


# ============================================================================ kNN via d_(k)
def knn_distances_sq(X, Q):
    """Squared Euclidean distances D[j, i] = sum_l (Q[j,l] - X[i,l])^2 (P:L483 'the array of
    distances d'), in float32 with every operation rounded (numpy float32 arithmetic), l in order
    0..p-1 — the definition written out in the precision the path computes in (north_star: the
    decision d < d_(k) is taken in the same precision on both sides)."""
    X = np.asarray(X, dtype=np.float32)
    Q = np.asarray(Q, dtype=np.float32)
    acc = np.zeros((Q.shape[0], X.shape[0]), dtype=np.float32)
    for l in range(X.shape[1]):
        e = Q[:, l:l + 1] - X[None, :, l]          # float32 - float32 -> float32 (rounded)
        acc = acc + e * e                           # float32 product, float32 sum (each rounded)
    return acc


def knn_weights(d2, weighting: int):
    """w_i: 1 (plain mean of the k nearest) or 1/(d2 + 1e-12), a decreasing function of the
    distance (P:L483 'w_i are the weights that are decreasing functions of the distances')."""
    d2 = np.asarray(d2, dtype=LD)
    return np.ones_like(d2) if weighting == 0 else LD(1) / (d2 + LD(1e-12))


def knn_regress(X, f, Q, k: int, weighting: int = 0):
    """kNN regression by the k-th order statistic: d_(k) = the k-th smallest distance,
    then the indicator rho (P:L469-476 with h = k): rho = 1 for d < d_(k), a/b for d = d_(k) (a =
    k - #{d < d_(k)}, b = #{d = d_(k)}), 0 otherwise, and f(q) = sum rho w f / sum rho w by
    reduction (long double).  Returns (predictions float64[nq], d2_(k) float32[nq])."""
    D = knn_distances_sq(X, Q)
    f = np.asarray(f, dtype=np.float32).astype(LD)
    out = np.empty(D.shape[0], dtype=np.float64)
    dk = np.empty(D.shape[0], dtype=np.float32)
    for j in range(D.shape[0]):
        row = D[j]
        t = order_statistic(row, k)
        lt, eq = row < t, row == t
        a, b = k - int(np.count_nonzero(lt)), int(np.count_nonzero(eq))
        rho = lt.astype(LD) + eq.astype(LD) * (LD(a) / LD(b))
        w = knn_weights(row, weighting) * rho
        out[j] = float(np.sum(w * f) / np.sum(w))
        dk[j] = t
    return out, dk


def knn_classify(X, labels, Q, k: int, n_classes: int, weighting: int = 0):
    """kNN classification ("the majority vote (among the k nearest neighbors) is applied"):
    the votes V_c = sum_i rho_i w_i [label_i = c] with the indicator rho of `knn_regress` (R33) and
    the winner = argmax V_c, the smallest class among equal votes.  Returns (classes int32[nq],
    votes float64[nq, n_classes])."""
    D = knn_distances_sq(X, Q)
    labels = np.asarray(labels)
    out = np.empty(D.shape[0], dtype=np.int32)
    votes = np.zeros((D.shape[0], n_classes), dtype=np.float64)
    for j in range(D.shape[0]):
        row = D[j]
        t = order_statistic(row, k)
        lt, eq = row < t, row == t
        a, b = k - int(np.count_nonzero(lt)), int(np.count_nonzero(eq))
        rho = lt.astype(LD) + eq.astype(LD) * (LD(a) / LD(b))
        w = knn_weights(row, weighting) * rho
        for c in range(n_classes):
            votes[j, c] = float(np.sum(w[labels == c]))
        out[j] = int(np.argmax(votes[j]))   # first maximum = smallest class among equal votes
    return out, votes
