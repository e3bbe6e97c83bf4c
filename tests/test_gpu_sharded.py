"""The sharded path (§8 a6/e) executed for real at G >= 2 on ONE GPU: G virtual ranks, each a host
thread with its own ctx and stream, attached to a loopback group (SURVEY §4 "G virtual shards on
one GPU").  The C++ ShardedBackend runs unchanged — pooled sample cuts (R28), fused init per rank,
tuple all-gathers and rank-order combine, cut passes, Kelley passes, the packed all-gather-v of the
bracket and the exact select — only the transport is a device-to-device copy instead of NCCL.

Every rank must return the same element, bit-exact with the oracle's sort-based selection of the
concatenated shards ('partial sums from several GPUs are added')."""
import threading

import numpy as np
import pytest

import datagen
import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cp():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1104_2732_b200 as cp
    cp.load()
    return cp


def canon(v):
    return 0.0 if v == 0 else v


def run_virtual(cp, xd, bounds, ks, config=None, timeout=600):
    """Select every k in ks over the concatenation of xd[bounds[g]:bounds[g+1]] with G =
    len(bounds)-1 virtual ranks.  Returns per rank the list of (value, info)."""
    import torch
    G = len(bounds) - 1
    grp = cp.LoopbackGroup(G)
    out = [None] * G
    errs = []
    torch.cuda.synchronize()

    def worker(g):
        try:
            torch.cuda.set_device(xd.device)
            s = torch.cuda.Stream(xd.device)
            with torch.cuda.stream(s):
                dev = xd.device.index
                if config:
                    cp.set_config(dev, **config)
                cp.comm_init_loopback(grp, g, dev)
                shard = xd[bounds[g]:bounds[g + 1]]
                out[g] = [cp.select_kth_sharded(shard, k, return_info=True) for k in ks]
            s.synchronize()
        except Exception as e:  # surfaced below
            errs.append((g, e))

    th = [threading.Thread(target=worker, args=(g,)) for g in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
    assert not any(t.is_alive() for t in th), "a virtual rank hung"
    assert not errs, errs
    return out


def bounds_for(n, G, kind):
    if kind == "even":
        return [n * g // G for g in range(G + 1)]
    if kind == "uneven":          # ragged, one rank ~half of everything
        w = np.array([1, 7, 3, 13, 2, 5, 11, 4][:G], dtype=np.float64)
        c = np.concatenate([[0], np.cumsum(w)]) / w.sum()
        b = [int(round(v * n)) for v in c]
        b[-1] = n
        return b
    if kind == "empty":           # 8 ranks: empty shards first, in the middle and last
        assert G == 8
        return [0, 0, n // 5, n // 5, 2 * n // 5, 3 * n // 5, 4 * n // 5, n, n]
    raise ValueError(kind)


def check(x, res, ks):
    srt = np.sort(x)
    for j, k in enumerate(ks):
        want = canon(float(srt[k - 1]))
        got = {canon(r[j][0]) for r in res}
        assert got == {want}, (k, got, want)


@pytest.mark.parametrize("G,kind", [(2, "even"), (4, "uneven"), (8, "empty"), (8, "uneven")])
@pytest.mark.parametrize("dist,dtype", [("uniform", "f32"), ("cauchy", "f32"), ("dup256", "f32"), ("normal", "f64")])
def test_virtual_shards_fused_path(cp, G, kind, dist, dtype):
    """n large enough for the fused init at the pooled cuts, the cut passes and the all-gather-v
    of a packed segmented bracket (the default config, select_cap 2^22)."""
    n = 12_000_007
    x = datagen.make(dist, n, dtype)
    import torch
    xd = torch.from_numpy(x).cuda()
    ks = [1, 3, n // 10, O.median_rank(n), n - 1, n]
    res = run_virtual(cp, xd, bounds_for(n, G, kind), ks)
    check(x, res, ks)
    med = [r[3][1] for r in res]
    if dist != "dup256":  # (dup256: the median's value fills the whole bracket, nothing strictly inside)
        assert all(i["init_written"] > 0 for i in med)       # the pooled cuts ran in the init pass


@pytest.mark.parametrize("G", [2, 4, 8])
def test_virtual_shards_default_config_mid_size(cp, G):
    """n ~ 2^23 with the default caps — the init's copy is below the select cap
    right away, so the first step is the all-gather-v of the SEGMENTED init copy (packed per rank)."""
    import torch
    n = (1 << 23) + 77
    for dist in ("uniform", "mix2"):
        x = datagen.make(dist, n, "f32")
        xd = torch.from_numpy(x).cuda()
        ks = [n // 10, O.median_rank(n), n - n // 7]
        res = run_virtual(cp, xd, bounds_for(n, G, "uneven"), ks)
        check(x, res, ks)
        assert all(r[1][1]["exit"] == "compact_select" for r in res)


@pytest.mark.parametrize("cfg", [dict(init_cut=0), dict(init_cut=0, pass_cuts=0, objective=1),
                                 dict(select_cap=1 << 12, z_cap=1 << 20)])
def test_virtual_shards_kelley_passes(cp, cfg):
    """The plain init (all-gathered records, rank-order combine) and the Kelley passes with their
    all-gathered tuples (compacting, segmented and dense halves), at G = 4 uneven + empty shards."""
    import torch
    n = 9_000_011
    for dist in ("normal", "mix1", "dup256"):
        x = datagen.make(dist, n, "f32")
        xd = torch.from_numpy(x).cuda()
        ks = [2, n // 10, O.median_rank(n), n - 2]
        b = bounds_for(n, 4, "uneven")
        b = b[:2] + [b[1]] + b[2:]      # 5 ranks, rank 1 empty
        res = run_virtual(cp, xd, b, ks, config=cfg)
        check(x, res, ks)
        assert all(r[2][1]["cp_iters"] >= 1 for r in res)


def test_virtual_shards_small_and_degenerate(cp):
    """Tiny global arrays (direct selection after the all-gathered init), all-equal data, ±0,
    one non-empty rank."""
    import torch
    cases = [np.array([3.0, 1.0, 2.0], np.float32), np.zeros(1000, np.float32),
             np.array([-0.0, 0.0] * 500 + [1.0], np.float32), datagen.make("mix3", 100_003, "f64")]
    for x in cases:
        xd = torch.from_numpy(x).cuda()
        n = x.size
        ks = sorted({1, O.median_rank(n), n})
        for b in ([0, n // 2, n], [0, 0, n, n], [0, 1, 2, 3, n]):
            res = run_virtual(cp, xd, b, ks)
            check(x, res, ks)


def test_virtual_shards_reject_nonfinite(cp):
    import torch
    x = datagen.make("normal", 9_000_000, "f32")
    x[7_777_777] = np.nan
    xd = torch.from_numpy(x).cuda()
    grp = cp.LoopbackGroup(2)
    errs = []

    def worker(g):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                cp.comm_init_loopback(grp, g, 0)
                cp.select_kth_sharded(xd[g * 4_500_000:(g + 1) * 4_500_000], 100)
        except ValueError as e:
            errs.append(str(e))

    th = [threading.Thread(target=worker, args=(g,)) for g in range(2)]
    [t.start() for t in th]
    [t.join(300) for t in th]
    assert len(errs) == 2 and all("NaN" in e or "status 3" in e for e in errs), errs


def test_sharded_2pow32_on_one_gpu(cp):
    """configs[3] size on one B200: the median of 2^32 + 3 float32 (64-bit counts past 2^32), by
    the one-GPU path and by 8 virtual ranks over the same array (the scaling base and the G = 8
    split), checked by the rank invariant #{x < v} < k <= #{x <= v} (north_star) — both identical."""
    import torch
    n = (1 << 32) + 3
    g = torch.Generator(device="cuda")
    g.manual_seed(datagen.SEED)
    xd = torch.rand(n, device="cuda", generator=g, dtype=torch.float32)
    k = (n + 1) // 2
    v1, info = cp.select_kth(xd, k, return_info=True)
    lt = int((xd < v1).sum())
    le = int((xd <= v1).sum())
    assert lt < k <= le, (v1, lt, le, k)
    res = run_virtual(cp, xd, [n * q // 8 for q in range(9)], [k])
    assert {r[0][0] for r in res} == {v1}
    for kk in (1, n):
        v = cp.select_kth(xd, kk)
        assert v == (float(xd.min()) if kk == 1 else float(xd.max()))
    del xd
    torch.cuda.empty_cache()


def test_loopback_missing_peer_fails_instead_of_hanging(cp, monkeypatch):
    """Failure detection: a rank whose peer never reaches the collective gets ENCCL after
    CPSEL_COMM_TIMEOUT_S, not a hang; a later, complete group on fresh threads still works."""
    import time
    import torch
    monkeypatch.setenv("CPSEL_COMM_TIMEOUT_S", "2")
    x = datagen.make("normal", 1 << 20, "f32")
    xd = torch.from_numpy(x).cuda()
    grp = cp.LoopbackGroup(2)
    res = {}

    def lone_rank():
        with torch.cuda.stream(torch.cuda.Stream()):
            cp.comm_init_loopback(grp, 0, 0)
            try:
                res["value"] = cp.select_kth_sharded(xd, 1000)
            except Exception as e:  # expected
                res["err"] = str(e)

    t0 = time.time()
    t = threading.Thread(target=lone_rank)
    t.start()
    t.join(120)
    assert not t.is_alive(), "the lone rank hung"
    assert "err" in res and "did not arrive" in res["err"], res
    assert time.time() - t0 < 60
    monkeypatch.delenv("CPSEL_COMM_TIMEOUT_S")
    out = run_virtual(cp, xd, [0, 400_000, 1 << 20], [1000])
    assert out[0][0][0] == out[1][0][0] == float(O.order_statistic(x, 1000))
