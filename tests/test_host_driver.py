"""The C++ cutting-plane driver (libcpsel.so, cpsel_drive_host) on CPU with numpy data steps,
against the oracle; and the sharded (N>1) host logic with world-size-2 gloo process groups."""
import math
import os
import socket

import numpy as np
import pytest

import datagen
import oracle as O
from tests._hostbe import drive


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_1104_2732_b200 import build
    build.build()


def canon(v):
    return 0.0 if v == 0 else v


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_driver_matches_oracle_distributions(dtype):
    for dist in datagen.ALL_DISTS:
        x = datagen.make(dist, 20_011, dtype)
        n = x.size
        for k in sorted({1, 2, n // 10, O.median_rank(n), n - 1, n}):
            for cfg in ({"force_cp": 1, "z_cap": 64}, {"force_cp": 1, "z_cap": 4096}, {},
                        {"force_cp": 1, "select_cap": 16}, {"force_cp": 1, "select_cap": 1, "z_cap": 10_000}):
                for cut in (False, True):
                    v, info, trace = drive(x, k, dtype, config=cfg, cut=cut)
                    assert canon(v) == float(O.order_statistic(x, k)), (dist, k, cfg, cut, info)
                    assert info["passes"] == info["cp_iters"] + 1          # maxit+1 reductions


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("cut_shift", [0.0, 0.3, -0.3])
def test_driver_pass_cuts(dtype, cut_shift):
    """R26 cut passes (two sample cuts of the compacted bracket, copy of what lies between them):
    exact on every distribution and rank, also when the cuts are deliberately off target
    (cut_shift moves them by 30% of the sample: the far-side branches move the bracket to the
    adjacent float and continue on the uncompacted array)."""
    for dist in datagen.ALL_DISTS:
        x = datagen.make(dist, 20_011, dtype)
        n = x.size
        for k in sorted({1, 2, n // 10, O.median_rank(n), n - 1, n}):
            for cfg in ({"force_cp": 1, "z_cap": 15_000, "select_cap": 16},
                        {"force_cp": 1, "z_cap": 20_011, "select_cap": 300}):
                v, info, trace = drive(x, k, dtype, config=cfg, cut=True, pass_cuts=True, cut_shift=cut_shift)
                assert canon(v) == float(O.order_statistic(x, k)), (dist, k, cfg, info)
                assert info["passes"] == info["cp_iters"] + 1
    # the cut passes do run (uniform data, median)
    x = datagen.make("uniform", 20_011, dtype)
    _, _, trace = drive(x, O.median_rank(x.size), dtype, config={"force_cp": 1, "select_cap": 16},
                        cut=True, pass_cuts=True)
    assert any(r["kind"] == 3 for r in trace)


def test_pooled_cuts_bracket_the_pooled_rank():
    """R28: cuts pooled from uneven shards' samples (weights m_g / #samples_g) bracket the pooled
    order statistic, are sample values of the shards, and the estimate lies between them."""
    import paper_1104_2732_b200 as cp
    from tests._hostbe import sample_keys
    rng = np.random.default_rng(28)
    for dtype in ("f32", "f64"):
        npdt = np.float32 if dtype == "f32" else np.float64
        for sizes in ([300_000, 5_000, 0, 120_000], [1000, 1000], [7, 200_000], [3]):
            shards = [rng.standard_normal(m).astype(npdt) * (g + 1) + g for g, m in enumerate(sizes)]
            allx = np.concatenate(shards)
            srt = np.sort(allx)
            keys = np.stack([sample_keys(sh) for sh in shards])
            for r in sorted({1, max(allx.size // 10, 1), (allx.size + 1) // 2, allx.size}):
                ta, tb, te = cp.pooled_cuts(keys, sizes, r, dtype)
                assert ta <= te <= tb
                assert any(np.any(sh == ta) for sh in shards) and any(np.any(sh == tb) for sh in shards)
                if 10 < r < allx.size - 10 and allx.size > 1000:
                    assert ta <= srt[r - 1] <= tb, (sizes, r)


def test_driver_tiny_all_ranks_with_ties_and_signed_zero():
    rng = np.random.default_rng(5)
    for _ in range(300):
        n = int(rng.integers(1, 14))
        x = rng.choice(np.array([0.0, -0.0, 1.0, 1.0, -2.0, 3.5, 1e9, -1e9, 7.0]), n)
        for dtype in ("f32", "f64"):
            xd = x.astype(np.float32 if dtype == "f32" else np.float64)
            for k in range(1, n + 1):
                for cfg in ({"force_cp": 1, "z_cap": 1}, {"force_cp": 1, "z_cap": 3},
                            {"force_cp": 1, "select_cap": 1}):
                    for cut in (False, True):
                        v, info, _ = drive(xd, k, dtype, config=cfg, cut=cut)
                        assert canon(v) == float(O.order_statistic(xd, k))


def test_driver_trace_matches_oracle_replay():
    """Every traced pass (incl. the init pass's extra cut): counts exact, F within rel 1e-12 of the
    oracle's direct long-double F."""
    x = datagen.make("mix1", 50_000, "f64")
    k = O.median_rank(x.size)
    v, info, trace = drive(x, k, "f64", config={"force_cp": 1, "z_cap": 100}, cut=True)
    assert trace and trace[0]["kind"] == 2
    for row in trace:
        ref = O.eval_at(x, k, row["t"], -math.inf, math.inf)
        UNK = (1 << 64) - 1                        # a count the init cut does not evaluate (R24)
        if row["kind"] == 2:
            assert row["c_eq"] == UNK and row["c_lt"] in (UNK, ref["c_lt"])
        else:
            assert row["c_lt"] == ref["c_lt"] and row["c_eq"] == ref["c_eq"]
        assert row["F"] == pytest.approx(float(ref["F"]), rel=1e-12)


def test_driver_first_iterate_is_interior_mean_and_in_dtype():
    x = datagen.make("normal", 10_001, "f32")
    k = O.median_rank(x.size)
    _, _, trace = drive(x, k, "f32", config={"force_cp": 1, "z_cap": 10})
    rec = O.init_record(x)
    inner = x[(x > rec["min"]) & (x < rec["max"])].astype(np.float64)
    assert trace[0]["t"] == float(np.float32(inner.mean()))
    assert all(float(np.float32(r["t"])) == r["t"] for r in trace)


def test_driver_outlier_insensitive_and_1e20():
    """pass count flat in the outlier magnitude; the local-sum form also survives 1e20 (R11)."""
    base = datagen.make("normal", 1 << 16, "f32")
    k = O.median_rank(base.size)
    its = []
    for M in (1e3, 1e6, 1e9, 1e20):
        x = datagen.inject_outliers(base.copy(), 1, M)
        v, info, _ = drive(x, k, "f32", config={"force_cp": 1, "z_cap": (1 << 16) // 64})
        assert canon(v) == float(O.order_statistic(x, k))
        its.append(info["cp_iters"])
    assert max(its) - min(its) <= 2


def test_driver_pathological_geometric_uses_safeguard():
    """x_i = 2^i (interior mean hugs the top): the ordered-key safeguard bounds the pass count."""
    x = np.array([2.0 ** i for i in range(-120, 120)], dtype=np.float32)
    x = np.concatenate([x, x[::-1], x])
    for k in (1, 5, 300, x.size // 2, x.size - 3):
        v, info, _ = drive(x, k, "f32", config={"force_cp": 1, "z_cap": 1})
        assert canon(v) == float(O.order_statistic(x, k))
        assert info["passes"] <= 80


def test_driver_rejects_nonfinite():
    import paper_1104_2732_b200 as cp
    x = np.array([1.0, np.nan, 2.0], np.float32)
    with pytest.raises(cp.CpselError):
        drive(x, 1, "f32")


# ---------------------------------------------------------------------------- sharded, gloo
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sharded_worker(rank, world, port, cases, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def comm(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    results = []
    for dist_name, n, dtype, k, zc, split in cases:
        x = datagen.make(dist_name, n, dtype)
        bounds = [0] + split + [n]
        shard = x[bounds[rank]:bounds[rank + 1]]
        for cuts in (False, True):   # plain, and with the pooled sample cuts of R28 (init + cut passes)
            v, info, trace = drive(shard, k, dtype, comm=comm, config={"force_cp": 1, "z_cap": zc, "select_cap": 50},
                                   cut=cuts, pass_cuts=cuts)
            results.append((v, info["passes"], [(r["t"], r["c_lt"], r["c_eq"], r["kind"]) for r in trace]))
    q.put((rank, results))
    dist.destroy_process_group()


def test_sharded_host_logic_gloo_world2():
    """World-size-2 gloo: the sharded combine (rank-order sums, min/max merge, shifted-sum
    re-basing, all-gather of the kept halves) gives every rank the same decisions and the
    unsharded answer — including an empty shard and uneven shards."""
    import torch.multiprocessing as mp
    n = 30_000
    cases = [("normal", n, "f32", O.median_rank(n), 256, [n // 2]),
             ("mix2", n, "f64", n // 10, 64, [7]),
             ("dup256", n, "f32", n - 1, 512, [n // 3]),
             ("cauchy", n, "f32", 12345, 1000, [0]),          # rank 0 holds nothing
             ("uniform", n, "f64", 1, 128, [n - 1])]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, cases, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for i, (dist_name, n_, dtype, k, zc, split) in enumerate(cases):
        x = datagen.make(dist_name, n_, dtype)
        expect = float(O.order_statistic(x, k))
        for j in (2 * i, 2 * i + 1):
            assert canon(got[0][j][0]) == expect and canon(got[1][j][0]) == expect
            assert got[0][j][1:] == got[1][j][1:]             # identical driver decisions
    # the pooled cuts ran (kind-2 init cuts and kind-3 cut passes) in the median case
    assert any(row[3] == 2 for row in got[0][1][2]) and any(row[3] == 3 for row in got[0][1][2])


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_driver_brent_min_replays_the_oracle(dtype):
    """driver=3 (Brent's minimisation): the exact element, and every point it
    proposed is the point oracle.BrentMinStep proposes from the same F values (the trace's, which
    match the oracle's direct long-double F within the north_star tolerance); the counts exact."""
    tol = 1e-6 if dtype == "f32" else 1e-12
    for dist in ("uniform", "normal", "cauchy", "dup256"):
        x = datagen.make(dist, 20_011, dtype)
        n = x.size
        for k in (2, n // 10, O.median_rank(n), n - 1):
            v, info, trace = drive(x, k, dtype, config={"driver": 3, "force_cp": 1, "z_cap": n, "select_cap": 8})
            assert canon(v) == float(O.order_statistic(x, k)), (dist, k, info)
            rows = [r for r in trace if r["kind"] == 6]
            assert rows == trace[:len(rows)] and (rows or info["exit"] in ("init_min", "init_max"))
            ref = O.brent_min_replay(x, k, [r["F"] for r in rows])
            assert len(ref["trace"]) >= len(rows) - 1
            for r, (t, F, c_lt, c_eq, _) in zip(rows, ref["trace"]):
                assert r["t"] == t and (r["c_lt"], r["c_eq"]) == (c_lt, c_eq), (dist, k, r, t)
                assert r["F"] == pytest.approx(float(O.f_os(x, t, k)), rel=tol)
