"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Bar (north_star): the selected element bit-exact (after -0 -> +0), every count exact, F and the
pass sums within relative 1e-6 (float32) / 1e-12 (float64)."""
import math

import numpy as np
import pytest

import datagen
import oracle as O

pytestmark = pytest.mark.gpu

REL = {"f32": 1e-6, "f64": 1e-12}


@pytest.fixture(scope="module")
def cp():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1104_2732_b200 as cp
    cp.load()
    return cp


def tdev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def canon(v):
    return 0.0 if v == 0 else v


def host(t):
    return t.cpu().numpy()


# ----------------------------------------------------------------------------- a1: init
@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("n,off", [(1, 0), (2, 1), (7, 3), (1_000_003, 0), (1_000_003, 1), (4_194_305, 3)])
def test_init_reduction(cp, dtype, n, off):
    x = datagen.make("mix3", n + off, dtype)[off:]       # ragged tail + misaligned start
    cp.set_config(init_cut=0)                            # the shifted sum is computed without the cut
    s = cp.init_stats(tdev(datagen.make("mix3", n + off, dtype))[off:])
    cp.set_config(init_cut=1)
    rec = O.init_record(x)
    assert s["vmin"] == rec["min"] and s["vmax"] == rec["max"]
    assert s["cnt_min"] == rec["cnt_min"] and s["cnt_max"] == rec["cnt_max"] and s["nonfinite"] == 0
    assert s["x0"] == float(x[0])
    # S' = sum (x_i - x_0) cancels by design (R10): its error is bounded relative to the condition
    # scale sum |x_i - x_0| (fp64 accumulation of exact-or-rounded differences), at north_star's
    # relative bound: 1e-6 (f32) / 1e-12 (f64) of that scale
    xl = x.astype(O.LD)
    ref = float(np.sum(xl - xl[0]))
    scale = float(np.sum(np.abs(xl - xl[0])))
    assert abs(s["S"] - ref) <= REL[dtype] * max(scale, 1e-300), (s["S"], ref, scale)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("dist", ["uniform", "mix2", "dup256", "cauchy"])
def test_init_extra_cut(cp, dtype, dist):
    """R23: the init pass's two extra cuts — t_lo <= t_hi are elements of x bracketing the median
    rank, and the counts / sums at them match the oracle's direct evaluation."""
    n = 2_000_003
    x = datagen.make(dist, n, dtype)
    s = cp.init_stats(tdev(x))
    assert s["has_cut"] & 2 and s["has_cut"] & 4          # cuts, with the positive-part sums
    tl, th = s["t_lo"], s["t_hi"]
    assert tl <= th and np.isfinite(tl) and np.isfinite(th)   # any floats (R29: key-class bounds)
    rl = O.pass_stats(x, tl, -math.inf, math.inf)
    rh = O.pass_stats(x, th, tl, th)
    assert s["c_le_lo"] == rl["c_lt"] + rl["c_eq"]
    assert s["c_lt_hi"] == rh["c_lt"]
    assert s["N_lo"] == pytest.approx(float(rl["N"]), rel=REL[dtype], abs=1e-300)
    assert s["P_hi"] == pytest.approx(float(rh["P"]), rel=REL[dtype], abs=1e-300)
    # I = sum_{t_lo<x<t_hi} (x - t_lo) = L_hi of a pass at t_lo with bracket upper end t_hi
    ri = O.pass_stats(x, tl, -math.inf, th)
    assert s["I_in"] == pytest.approx(float(ri["L_hi"]), rel=REL[dtype], abs=1e-300)
    k = O.median_rank(n)
    assert rl["c_lt"] < k <= rh["c_lt"] + rh["c_eq"]        # the cuts bracket the target
    assert rh["c_lt"] - rl["c_lt"] < 0.2 * n                 # ... tightly (1024 samples, +-3.5 sd)


def test_init_counts_nonfinite(cp):
    for bad in (np.nan, np.inf, -np.inf):
        x = datagen.make("normal", 100_000, "f32")
        x[777] = bad
        assert cp.init_stats(tdev(x))["nonfinite"] == 1


# ----------------------------------------------------------------------------- a2: one pass
@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("dist", ["normal", "mix1", "dup256", "cauchy"])
def test_eval_pass_matches_oracle(cp, dtype, dist):
    n = 1_000_003
    x = datagen.make(dist, n, dtype)
    xd = tdev(x)
    rng = np.random.default_rng(1)
    npdt = np.float32 if dtype == "f32" else np.float64
    qs = np.quantile(x, [0.01, 0.2, 0.45, 0.5, 0.55, 0.8, 0.99]).astype(npdt)
    cases = [(x[5], -math.inf, math.inf), (x[n // 2], x[n // 3], x[2 * n // 3])]
    for _ in range(6):
        a, t, b = np.sort(rng.choice(qs, 3))
        cases.append((t, a, b))
    for t, lo, hi in cases:
        t, lo, hi = float(npdt(t)), float(lo), float(hi)
        g = cp.eval(xd, t, lo, hi)
        r = O.pass_stats(x, t, lo, hi)
        for key in ("c_lt", "c_eq", "c_lo", "c_hi"):
            assert g[key] == r[key], key
        assert g["pred"] == r["pred"] and g["succ"] == r["succ"]
        for key in ("L_lo", "L_hi", "P", "N"):
            assert g[key] == pytest.approx(float(r[key]), rel=REL[dtype], abs=1e-300), key


def test_eval_misaligned_and_tiny(cp):
    for n in (1, 2, 3, 5, 9, 33, 257, 4099):
        for off in (0, 1, 2, 3):
            x = datagen.make("normal", n + off, "f32")
            xd = tdev(x)[off:]
            xs = x[off:]
            t = float(xs[len(xs) // 2])
            g = cp.eval(xd, t, -math.inf, math.inf)
            r = O.pass_stats(xs, t, -math.inf, math.inf)
            assert (g["c_lt"], g["c_eq"], g["c_lo"], g["c_hi"]) == (r["c_lt"], r["c_eq"], r["c_lo"], r["c_hi"])
            assert g["N"] == pytest.approx(float(r["N"]), rel=1e-6, abs=1e-30)


# ----------------------------------------------------------------------------- a5: small select
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_small_select(cp, dtype):
    rng = np.random.default_rng(2)
    npdt = np.float32 if dtype == "f32" else np.float64
    for m in (1, 2, 3, 31, 1000, 65_537, 1_000_001):
        z = (rng.standard_normal(m) * 10 ** rng.uniform(-30, 30, m)).astype(npdt)
        z[rng.integers(0, m, m // 10 + 1)] = 0.0
        z[rng.integers(0, m, m // 10 + 1)] = -0.0
        z[rng.integers(0, m, m // 7 + 1)] = z[0]
        zd = tdev(z)
        for r in sorted({1, min(2, m), m // 3 or 1, (m + 1) // 2, m}):
            got = cp.small_select(zd, r)
            assert canon(got) == float(O.order_statistic(z, r))
            assert math.copysign(1, got) > 0 or got != 0


# ----------------------------------------------------------------------------- end to end
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_select_tiny_all_ranks(cp, dtype):
    rng = np.random.default_rng(3)
    npdt = np.float32 if dtype == "f32" else np.float64
    for force in (0, 1):
        cp.set_config(force_cp=force, z_cap=1 if force else 0, select_cap=1 if force else 0)
        for _ in range(60):
            n = int(rng.integers(1, 12))
            x = rng.choice(np.array([0.0, -0.0, 1.0, 1.0, -2.0, 3.5, 1e9, -1e9, 7.0]), n).astype(npdt)
            xd = tdev(x)
            for k in range(1, n + 1):
                assert canon(cp.select_kth(xd, k)) == float(O.order_statistic(x, k))
    cp.set_config(force_cp=0, z_cap=0, select_cap=0)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_select_distributions_forced_cp(cp, dtype):
    """Every distribution x ranks, through the cutting-plane passes (force_cp) with several
    compaction thresholds, n spanning many tiles plus a ragged tail."""
    n = 300_007
    for dist in datagen.ALL_DISTS:
        x = datagen.make(dist, n, dtype)
        xd = tdev(x)
        for k in sorted({1, 2, n // 10, O.median_rank(n), n - 1, n}):
            want = float(O.order_statistic(x, k))
            for zc, sc, cut in ((0, 0, 1), (0, 0, 0), (512, 0, 1), (50_000, 0, 0), (0, 64, 1), (10**9, 1000, 1)):
                cp.set_config(force_cp=1, z_cap=zc, select_cap=sc, init_cut=cut)
                v, info = cp.select_kth(xd, k, return_info=True)
                assert canon(v) == want, (dist, k, zc, sc, cut, info)
                assert info["passes"] == info["cp_iters"] + 1
    cp.set_config(force_cp=0, z_cap=0, select_cap=0, init_cut=1)


def test_select_adversarial_orders_and_sample_positions(cp):
    """The two extra cuts come from strided samples (R23): poison exactly those positions so the cuts
    miss the target, and feed sorted / reverse-sorted / two-valued / constant arrays — the result
    must stay exact (the cuts are exact either way; the compacted bracket is simply not used)."""
    n = 3_000_017
    base = datagen.make("normal", n, "f32")
    m = 1024
    pos = (np.arange(m, dtype=np.int64) * n) // m + (n // m) // 2
    cases = {}
    x = base.copy(); x[pos] = -7.0; cases["samples_low"] = x
    x = base.copy(); x[pos] = 9.0; cases["samples_high"] = x
    x = base.copy(); x[pos] = np.float32(np.median(base)); cases["samples_at_median"] = x
    cases["sorted"] = np.sort(base)
    cases["reversed"] = np.sort(base)[::-1].copy()
    x = np.where(base < 0, np.float32(-1.0), np.float32(2.0)); cases["two_valued"] = x
    cases["constant"] = np.full(n, 3.5, np.float32)
    for name, x in cases.items():
        xd = tdev(x)
        for k in (1, 17, n // 3, O.median_rank(n), n - 5, n):
            v, info = cp.select_kth(xd, k, return_info=True)
            assert canon(v) == float(O.order_statistic(x, k)), (name, k, info)


def test_select_direct_path_config0(cp):
    """BASELINE configs[0]: median of n=1e5 float32 uniform (n <= direct_threshold -> direct select)."""
    x = datagen.make("uniform", 100_000, "f32")
    v, info = cp.median(tdev(x), return_info=True)
    assert canon(v) == float(O.median(x))
    assert info["exit"] in ("direct_select", "init_min", "init_max")


@pytest.mark.parametrize("dtype,n", [("f32", 131_072), ("f32", 131_071), ("f32", 4097), ("f64", 65_536),
                                     ("f64", 65_537), ("f64", 3)])
def test_select_direct_one_launch_bounds(cp, dtype, n):
    """§8f-3 small arrays: n <= direct_threshold and within the 8-CTA cluster's register capacity
    (2^17 f32, 2^16 f64) is ONE exact_cluster_kernel launch; just above it the init + radix path.
    Duplicates, signed zeros and a huge dynamic range; every rank class bit-exact."""
    rng = np.random.default_rng(n)
    x = (rng.standard_normal(n) * np.exp(rng.uniform(-30, 30, n))).astype(np.float32 if dtype == "f32" else np.float64)
    x[::7] = x[n // 2]                                       # a value with many copies
    x[1::11] = -0.0
    x[2::13] = 0.0
    xd = tdev(x)
    for k in sorted({1, 2, n // 3, O.median_rank(n), n - 1, n}):
        v, info = cp.select_kth(xd, k, return_info=True)
        assert canon(v) == float(O.order_statistic(x, k)), (dtype, n, k, info)
    cap = 131_072 if dtype == "f32" else 65_536
    if n <= cap:
        assert info["launches"] == 1 and info["exit"] == "direct_select"


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_select_direct_one_launch_rejects_nonfinite(cp, bad):
    x = datagen.make("uniform", 100_000, "f32")
    x[99_999] = bad
    with pytest.raises(ValueError, match="NaN or Inf"):
        cp.median(tdev(x))
    x[99_999] = 0.5
    assert canon(cp.median(tdev(x))) == float(O.median(x))


@pytest.mark.parametrize("dist", datagen.BENCH_DISTS)
def test_select_config1_2pow24_f32(cp, dist):
    """BASELINE configs[1]: n=2^24 float32, k in {median, 1, n/10, n-1}."""
    n = 1 << 24
    xd = datagen.make(dist, n, "f32", device="cuda")
    x = host(xd)
    for k in (O.median_rank(n), 1, n // 10, n - 1):
        v, info = cp.select_kth(xd, k, return_info=True)
        assert canon(v) == float(O.order_statistic(x, k)), (dist, k, info)


@pytest.mark.parametrize("dist", ["uniform", "normal"])
def test_select_config2_2pow28_f64(cp, dist):
    """BASELINE configs[2]: k-th order statistic of n=2^28 float64 vs the sort-based oracle."""
    n = 1 << 28
    xd = datagen.make(dist, n, "f64", device="cuda")
    x = host(xd)
    for k in (O.median_rank(n), n // 10):
        v, info = cp.select_kth(xd, k, return_info=True)
        assert canon(v) == float(O.order_statistic(x, k)), (dist, k, info)
    del xd


def test_select_bench_size_2pow30_f32(cp):
    """The bench workload (n=2^30 float32) in the launch configuration bench.py times: the result
    is checked by the rank invariant #{x<v} <= k-1 < #{x<=v} computed by the oracle on the host copy."""
    import torch
    n = 1 << 30
    for dist in datagen.BENCH_DISTS:   # the four arrays bench.py times
        xd = datagen.make(dist, n, "f32", device="cuda")
        k = O.median_rank(n)
        v, info = cp.median(xd, return_info=True)
        # the same element from the paper's method as published (Kelley passes from [x_(1), x_(n)])
        cp.set_config(init_cut=0, pass_cuts=0, objective=1)
        v2 = cp.median(xd)
        cp.set_config(init_cut=1, pass_cuts=1, objective=0)
        assert v2 == v, (dist, v, v2)
        x = host(xd)
        del xd
        torch.cuda.empty_cache()
        c_lt, c_eq = O.rank_counts(x, v)
        assert c_lt <= k - 1 < c_lt + c_eq, (dist, info)
        del x


UNK = (1 << 64) - 1  # a count the trace row does not carry


def test_trace_replay_F_parity(cp):
    """Every cutting-plane pass of a real run: counts exact and F_k(t) within 1e-6 / 1e-12
    relative of the oracle's direct long-double evaluation at the same t."""
    for dtype in ("f32", "f64"):
        for dist in ("normal", "mix4", "cauchy"):
            x = datagen.make(dist, 2_000_003, dtype)
            xd = tdev(x)
            for k in (O.median_rank(x.size), 1000):
                cp.set_config(force_cp=1, z_cap=1000, objective=1)
                cp.select_kth(xd, k)
                tr = cp.get_trace()
                assert tr
                for row in tr:
                    ref = O.eval_at(x, k, row["t"], -math.inf, math.inf)
                    if row["kind"] == 2:                 # init cuts: #x<t_hi only (R24)
                        assert row["c_eq"] == UNK and row["c_lt"] in (UNK, ref["c_lt"])
                    else:
                        assert (row["c_lt"], row["c_eq"]) == (ref["c_lt"], ref["c_eq"])
                    assert row["F"] == pytest.approx(float(ref["F"]), rel=REL[dtype])
    cp.set_config(force_cp=0, z_cap=0, objective=0)


@pytest.mark.parametrize("objective", [0, 1])
def test_fused_init_trace(cp, objective):
    """The fused init pass (cuts + copy-out of ]t_lo, t_hi[, R23) at a size where the segmented
    buffers exist: value exact; with objective=1 every row's F_k(t) matches the oracle, with
    objective=0 the rows after the cuts carry F = NaN (R25) and the counts stay exact."""
    x = datagen.make("normal", (1 << 23) + 77, "f32")
    xd = tdev(x)
    k = O.median_rank(x.size)
    cp.set_config(objective=objective)
    v, info = cp.select_kth(xd, k, return_info=True)
    tr = cp.get_trace()
    cp.set_config(objective=0)
    assert v == O.order_statistic(x, k)
    assert info["init_written"] > 0 and tr[0]["kind"] == 2
    for row in tr:
        ref = O.eval_at(x, k, row["t"], -math.inf, math.inf)
        if row["kind"] not in (2, 3):                    # sample cuts carry one-sided counts
            assert (row["c_lt"], row["c_eq"]) == (ref["c_lt"], ref["c_eq"])
        if objective:
            assert row["F"] == pytest.approx(float(ref["F"]), rel=REL["f32"])
        else:
            assert math.isnan(row["F"])


@pytest.mark.parametrize("order", ["random", "sorted", "reversed"])
def test_pass_cuts_all_dists(cp, order):
    """R26 cut passes on the GPU (segmented sample kernel + cut pass): exact on every distribution,
    rank and input order (sorted input makes the warp runs value-ordered), and the cut passes do
    run at this size."""
    n = (1 << 23) + 77
    saw_cut = False
    cp.set_config(select_cap=1 << 16)                   # a deeper cascade: several cut passes
    for dist in datagen.ALL_DISTS:
        x = datagen.make(dist, n, "f32")
        if order == "sorted":
            x = np.sort(x)
        elif order == "reversed":
            x = np.sort(x)[::-1].copy()
        xd = tdev(x)
        srt = np.sort(x)
        for k in (3, n // 7, O.median_rank(n), n - n // 5, n - 2):
            v = cp.select_kth(xd, k)
            assert v == srt[k - 1], (dist, order, k)
            saw_cut |= any(r["kind"] == 3 for r in cp.get_trace())
        del xd
    cp.set_config(select_cap=0)
    assert saw_cut


@pytest.mark.parametrize("case", ["normal", "dup256", "flt_max"])
def test_fused_init_extreme_ranks(cp, case):
    """R27: the fused init pass does not count #min/#max — the bracket starts at their outer
    neighbours; ranks at the very ends still come out exact, and +-FLT_MAX (outer neighbour
    infinite) falls back to the checked init with counts."""
    n = (1 << 23) + 77
    x = datagen.make("dup256" if case == "dup256" else "normal", n, "f32")
    if case == "flt_max":
        x[[5, 77, 1000]] = np.float32(np.finfo(np.float32).max)
        x[[6, 78]] = -np.float32(np.finfo(np.float32).max)
    xd = tdev(x)
    srt = np.sort(x)
    for k in (1, 2, 3, n // 2, n - 2, n - 1, n):
        assert cp.select_kth(xd, k) == srt[k - 1], (case, k)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_fused_init_rejects_nonfinite(cp, dtype, bad):
    """The fused init pass at a size with segmented buffers: one NaN / +-Inf anywhere is rejected
    (ENONFINITE, R12) — NaNs are caught by the extremes' vote, +-Inf by the extremes themselves."""
    n = (1 << 22) + 3
    x = datagen.make("normal", n, dtype)
    x[n // 3] = bad
    with pytest.raises(ValueError):
        cp.median(tdev(x))
    x[n // 3] = 0.5
    assert cp.median(tdev(x)) == float(np.sort(x)[(n + 1) // 2 - 1])


def test_host_buffer_path(cp):
    import torch
    x = datagen.make("normal", 3_000_001, "f32")
    xt = torch.from_numpy(x).pin_memory()
    k = 1_234_567
    assert canon(cp.select_kth_host(xt, k)) == float(O.order_statistic(x, k))


def test_errors_fail_loudly(cp):
    import torch
    x = datagen.make("normal", 1000, "f32")
    xd = tdev(x)
    with pytest.raises(ValueError):
        cp.select_kth(xd, 0)
    with pytest.raises(ValueError):
        cp.select_kth(xd, 1001)
    x[3] = np.nan
    with pytest.raises(ValueError):
        cp.median(tdev(x))
    with pytest.raises(ValueError):
        cp.median(torch.from_numpy(x))          # CPU tensor: no CPU fallback
    with pytest.raises(ValueError):
        cp.median(torch.ones(10, device="cuda", dtype=torch.float16))


def test_sharded_world1_nccl(cp):
    """The NCCL sharded entry point with world size 1 equals the single-GPU result."""
    import torch
    uid = cp.nccl_unique_id()
    cp.comm_init(uid, 0, 1, torch.cuda.current_device())
    for dist, dtype in (("normal", "f32"), ("mix5", "f64"), ("dup256", "f32")):
        x = datagen.make(dist, 1_000_003, dtype)
        xd = tdev(x)
        for k in (1, 77, O.median_rank(x.size), x.size):
            assert canon(cp.select_kth_sharded(xd, k)) == float(O.order_statistic(x, k))
    # large enough for the fused init at pooled sample cuts and the cut passes (R26-R28): the
    # init's copy (~0.5% of n with R40's pooled sample, ~42k) exceeds the select cap
    cp.set_config(select_cap=1 << 14)
    try:
        for dist in ("uniform", "cauchy", "dup256"):
            x = datagen.make(dist, (1 << 23) + 77, "f32")
            xd = tdev(x)
            srt = np.sort(x)
            for k in (1, 3, x.size // 10, x.size - 1, O.median_rank(x.size)):
                v, info = cp.select_kth_sharded(xd, k, return_info=True)
                assert v == srt[k - 1], (dist, k)
            assert info["init_written"] > 0                  # (the median: the cuts bracket it)
            assert any(r["kind"] == 3 for r in cp.get_trace())
    finally:
        cp.set_config(select_cap=0)


def test_direct_chain_declined_then_reused(cp):
    """Direct device chain (n >= 2^27): when the init's sample cuts miss the target (here: x is huge
    exactly at the strided sample positions, so both cuts lie far above the median) the
    chained radix rounds must stand down — clearing the round-0 digit counts the init pass took —
    and the host continues with Kelley passes; the next selection through the chain is exact."""
    n = 1 << 27
    xd = datagen.make("normal", n, "f32", device="cuda")
    # the f32 init sample: 131072 strided values (the cluster's size, CPSEL_SAMPLE_X=1) or 4x that
    # (the grid kernel's default, R40) — both sets of positions poisoned
    pos = np.concatenate([np.arange(ms, dtype=np.int64) * (n // ms) + (n // ms) // 2 for ms in (131072, 524288)])
    import torch
    xd[torch.from_numpy(pos).cuda()] = 1e30
    k = O.median_rank(n)
    v, info = cp.select_kth(xd, k, return_info=True)
    x = host(xd)
    assert canon(v) == float(O.order_statistic(x, k)), info
    assert info["passes"] > 1                                   # not the chained finish
    y = datagen.make("uniform", n, "f32", device="cuda")
    for kk in (k, n // 10):
        v2, info2 = cp.select_kth(y, kk, return_info=True)
        assert canon(v2) == float(O.order_statistic(host(y), kk)), info2


@pytest.mark.parametrize("dist", ["uniform", "dup256"])
def test_direct_chain_extreme_ranks(cp, dist):
    """n = 2^27 + 3 takes the direct device chain; the extreme ranks (the cuts sit at the ends of the
    sample, or the chain stands down) and a ragged n stay bit-exact."""
    n = (1 << 27) + 3
    xd = datagen.make(dist, n, "f32", device="cuda")
    x = host(xd)
    xs = np.sort(x)
    for k in (1, 2, 1000, n - 1, n):
        v, info = cp.select_kth(xd, k, return_info=True)
        assert canon(v) == float(xs[k - 1]), (dist, k, info)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_extreme_ranks_open_cuts(cp, dtype):
    """Extreme ranks (k = 1, 2, n-1, n): the sample rank of the outer cut falls off the sample, the
    cut opens to -/+ the largest float and the init pass's copy holds the target — one pass, exact."""
    import torch
    n = (1 << 23) + 5
    x = datagen.make("normal", n, dtype)
    xd = torch.from_numpy(x).cuda()
    srt = np.sort(x)
    for k in (1, 2, 3, n - 2, n - 1, n):
        v, info = cp.select_kth(xd, k, return_info=True)
        assert v == canon(float(srt[k - 1])), (k, v)
        assert info["passes"] == 1, (k, info)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("dist", ["uniform", "cauchy", "mix1", "dup256"])
def test_device_loop_matches_host_loop(cp, dtype, dist):
    """§8f-3: the device-resident Kelley loop (one CUDA graph: WHILE {step kernel; pass kernel} + the
    exact select) takes exactly the host driver's steps — the same iterates, counts and interior
    sizes at every pass, the same element — and the element is the oracle's."""
    import torch
    n = 3_000_007
    x = datagen.make(dist, n, dtype)
    xd = torch.from_numpy(x).cuda()
    srt = np.sort(x)
    for cfg in (dict(init_cut=0, pass_cuts=0, objective=1), dict(init_cut=0, pass_cuts=0, objective=0, z_cap=1 << 20)):
        for k in (2, n // 10, O.median_rank(n), n - 1):
            out = {}
            for dl in (0, 1):
                cp.set_config(device_loop=dl, **cfg)
                v, info = cp.select_kth(xd, k, return_info=True)
                out[dl] = (v, info, cp.get_trace())
            cp.set_config(device_loop=0, init_cut=1, pass_cuts=1, objective=0, z_cap=0)
            (v0, i0, t0), (v1, i1, t1) = out[0], out[1]
            assert v0 == v1 == canon(float(srt[k - 1])), (k, v0, v1)
            assert i0["passes"] == i1["passes"] and i0["exit"] == i1["exit"], (i0, i1)
            assert len(t0) == len(t1)
            for a, b in zip(t0, t1):
                assert (a["t"], a["c_lt"], a["c_eq"], a["interior"], a["compacted"], a["kind"]) == \
                       (b["t"], b["c_lt"], b["c_eq"], b["interior"], b["compacted"], b["kind"])
                if cfg["objective"]:
                    assert b["F"] == pytest.approx(a["F"], rel=1e-12)
            assert i1["launches"] < i0["launches"] + 4      # one graph launch for the whole loop


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_bisection_driver_matches_oracle(cp, dtype):
    """driver=1 (bisection), driver=2 (Brent's root finder) and driver=3 (Brent's minimisation), the
    paper's comparisons: the same element as the oracle, their iterates
    exactly the oracle's (value midpoints / zbrent's points, rounded into the bracket; Brent's
    minimisation: the points oracle.BrentMinStep proposes from the trace's F values, which match the
    oracle's direct F within rel 1e-6 / 1e-12) with the same counts; and the paper's outlier claim
    (P:L313, P:L413-414 vs P:L416): with 1e9 outliers all three need many more passes than with 1e3,
    the cutting plane at most 2 more."""
    import torch
    n = 1_000_003
    base = datagen.make("uniform", n, dtype)
    passes = {}
    for mag in (1e3, 1e9):
        x = datagen.inject_outliers(base.copy(), 100, mag)
        xd = tdev(x)
        k = O.median_rank(n)
        refs = {1: O.bisection(x, k, z_cap=0), 2: O.brent_root(x, k, z_cap=0)}
        for drv in (1, 2, 3, 0):
            cp.set_config(driver=drv, init_cut=0, pass_cuts=0)
            v, info = cp.select_kth(xd, k, return_info=True)
            tr = cp.get_trace()
            cp.set_config(driver=0, init_cut=1, pass_cuts=1)
            assert v == canon(float(np.sort(x)[k - 1])), (mag, drv)
            passes[(mag, drv)] = info["passes"]
            if drv in refs:
                ref = refs[drv]
                assert len(tr) <= len(ref["trace"]) and all(r["kind"] == 3 + drv for r in tr)
                for r, (t, c_lt, c_eq, interior) in zip(tr, ref["trace"]):
                    assert r["t"] == t and (r["c_lt"], r["c_eq"]) == (c_lt, c_eq), (r, t, c_lt, c_eq)
            elif drv == 3:
                rows = [r for r in tr if r["kind"] == 6]
                assert rows and rows == tr[:len(rows)]
                ref = O.brent_min_replay(x, k, [r["F"] for r in rows])
                assert len(ref["trace"]) >= len(rows) - 1
                for r, (t, F, c_lt, c_eq, _) in zip(rows, ref["trace"]):
                    assert r["t"] == t and (r["c_lt"], r["c_eq"]) == (c_lt, c_eq), (r, t, c_lt, c_eq)
                for r in rows[:6]:
                    assert r["F"] == pytest.approx(float(O.f_os(x, r["t"], k)), rel=1e-6 if dtype == "f32" else 1e-12)
    assert passes[(1e9, 1)] - passes[(1e3, 1)] >= 15, passes
    assert passes[(1e9, 2)] - passes[(1e3, 2)] >= 10, passes
    assert passes[(1e9, 3)] - passes[(1e3, 3)] >= 10, passes
    assert passes[(1e9, 0)] - passes[(1e3, 0)] <= 2, passes


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_value_binned_finish_paths(cp, dtype):
    """The direct chain's value-binned finish (vbin_finish_kernel, §8f-3/a5): the init counts its copy
    per value bin of ]t_lo, t_hi[, the finish selects inside the target bin.  All three of its exits
    stay exact: a small bin (shared-memory select: every rank of smooth data), a bin of ONE value
    (many duplicates at the target: no select at all), and a bin holding more than its capacity of
    distinct values (a dense cluster at the target: the fallback to the key-digit radix select)."""
    import torch
    n = (1 << 23) + 11
    rng = np.random.default_rng(23)
    base = rng.random(n).astype(np.float64)
    # the init's sample cuts (8192 samples at this n) keep about +-2% of the ranks around the target:
    # a value bin is ~2e-5 wide here
    cases = {"smooth": base.copy()}
    cases["one_value"] = np.floor(base * 500.0) / 500.0      # 500 levels ~2e-3 apart: a bin holds one
    c = base.copy()
    idx = rng.choice(n, 40_000, replace=False)              # 0.5% of the ranks, inside the cuts:
    ulp = float(np.spacing(np.float32(0.5)))                 # 40k elements on 10 values ~6e-7 apart,
    c[idx] = 0.5 + ulp * rng.integers(0, 10, idx.size)       # one bin over its 16384-element capacity
    cases["dense_cluster"] = c
    launches = {}
    for name, xv in cases.items():
        x = xv.astype(np.float32 if dtype == "f32" else np.float64)
        xd = torch.from_numpy(x).cuda()
        xs = np.sort(x)
        for k in (O.median_rank(n), n // 2 + 777, n // 3):
            v, info = cp.select_kth(xd, k, return_info=True)
            assert v == canon(float(xs[k - 1])), (name, k, v, info)
            launches[(name, k)] = info["launches"]
    km = O.median_rank(n)
    # the cluster's bin overflows: the key-digit radix select runs after the finish (more launches)
    assert launches[("dense_cluster", km)] > launches[("smooth", km)] == launches[("one_value", km)], launches


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_value_binned_finish_infinite_span(cp, dtype):
    """The value-binned finish when t_hi - t_lo overflows (R38's open span: the copy's first digit
    is then the top 11 bits of the order-preserving key, and vb_bounds takes the values of that key
    class, whose ends may be NaN keys).  Two modes of opposite sign near the largest finite value,
    so the sample cuts around the median straddle the gap; also ranks inside either mode."""
    import torch
    n = (1 << 23) + 11
    rng = np.random.default_rng(29)
    big = float(np.finfo(np.float32 if dtype == "f32" else np.float64).max)
    u = rng.random(n)
    sign = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    x = (sign * big * (0.75 + 0.25 * u)).astype(np.float32 if dtype == "f32" else np.float64)  # span 1.5 big
    xd = torch.from_numpy(x).cuda()
    xs = np.sort(x)
    for k in (O.median_rank(n), O.median_rank(n) + 5, n // 3, 2 * n // 3, 17, n - 17):
        v, info = cp.select_kth(xd, k, return_info=True)
        assert v == canon(float(xs[k - 1])), (k, v, float(xs[k - 1]), info)


_SAMPLE_PROBE = r"""
import json, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import datagen
import oracle as O
import paper_1104_2732_b200 as cp
out = {}
for dtype, lg in (("f32", 27), ("f64", 27)):
    x = datagen.make("normal", (1 << lg) + 5, dtype)
    xd = torch.from_numpy(x).cuda()
    k = O.median_rank(x.size)
    v, info = cp.select_kth(xd, k, return_info=True)
    out[dtype] = {"v": float(v), "want": float(O.order_statistic(x, k)), "written": int(info["init_written"]),
                  "launches": int(info["launches"]), "exit": info["exit"]}
print(json.dumps(out))
"""


def _probe(env):
    import json
    import os
    import subprocess
    import sys
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", _SAMPLE_PROBE], env=e, capture_output=True, text=True, timeout=600,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_sample_grid_kernel_cuts():
    """R40: the one-GPU sample cuts from the cooperative grid kernel.  At the cluster's sample size
    (CPSEL_SAMPLE_X=1) its cuts are the cluster kernel's (R29: the same strided sample, the same
    three sample ranks, the same digits), so the init copies exactly as many elements; at the default
    524288 samples the rank window shrinks by sqrt(S'/S) (3.5 sigma of the larger sample), so the copy
    does too — and every selection stays exact (each call's value against the oracle)."""
    old = _probe({"CPSEL_SAMPLE_GRID": "0"})
    grid1 = _probe({"CPSEL_SAMPLE_GRID": "1", "CPSEL_SAMPLE_X": "1"})
    dflt = _probe({})
    for dtype, shrink in (("f32", 2.0), ("f64", 8 ** 0.5)):
        for r in (old[dtype], grid1[dtype], dflt[dtype]):
            assert r["v"] == r["want"], r
        assert grid1[dtype]["written"] == old[dtype]["written"], (old, grid1)
        assert old[dtype]["launches"] == grid1[dtype]["launches"] + 1, (old, grid1)  # gather + pick -> one
        ratio = dflt[dtype]["written"] / old[dtype]["written"]
        assert 0.7 / shrink < ratio < 1.3 / shrink, (dtype, ratio, old, dflt)


def test_concurrent_threads_own_contexts():
    """Python threads each get their own ctx and stream (threading.local): four threads running the
    default one-GPU path at once — the cooperative sample-grid kernel (R40), the fused init and the
    chained finish of several selections in flight on one device — all return the oracle's values."""
    import threading
    import torch
    import paper_1104_2732_b200 as cpm
    n = (1 << 27) + 7                    # > 2^26: the 128-CTA sample grid, the direct chain
    xs = [datagen.make(d, n, "f32") for d in ("uniform", "normal", "cauchy", "dup256")]
    want = [float(O.median(x)) for x in xs]
    xds = [tdev(x) for x in xs]
    torch.cuda.synchronize()
    got, errs = {}, []

    def worker(i):
        try:
            torch.cuda.set_device(0)
            vs = [cpm.median(xds[i]) for _ in range(6)]
            got[i] = vs
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    th = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
    [t.start() for t in th]
    [t.join(120) for t in th]
    assert not any(t.is_alive() for t in th), "a selection thread did not finish"
    assert not errs, errs
    for i in range(4):
        assert all(canon(v) == want[i] for v in got[i]), (i, got[i], want[i])
