"""kNN regression via d_(k) (§8f-4) on the GPU against the oracle: the distances are
float32 with the same rounded operations on both sides, so every d2_(k) is bit-exact; the rho/a,b
reduction (fp64 on both sides, different order) agrees to 1e-9 relative."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cp():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1104_2732_b200 as cp
    cp.load()
    return cp


def problem(n, p, nq, seed, ties=False):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, p)).astype(np.float32)
    if ties:  # integer grid: many equal distances, exact in float32
        X = rng.integers(-3, 4, (n, p)).astype(np.float32)
    f = (np.sin(X[:, 0]) + 0.1 * rng.standard_normal(n)).astype(np.float32)
    Q = rng.standard_normal((nq, p)).astype(np.float32)
    if ties:
        Q = rng.integers(-2, 3, (nq, p)).astype(np.float32)
    return X, f, Q


@pytest.mark.parametrize("n,p,nq,ties", [(1000, 3, 5, False), (200_003, 10, 33, False), (50_000, 2, 17, True),
                                         (300_007, 1, 40, True)])
@pytest.mark.parametrize("weighting", [0, 1])
def test_knn_matches_oracle(cp, n, p, nq, ties, weighting):
    import torch
    X, f, Q = problem(n, p, nq, 11 + n + p, ties)
    Xd, fd, Qd = (torch.from_numpy(v).cuda() for v in (X, f, Q))
    for k in (1, 7, 64, n // 3, n):
        out, dk = cp.knn_regress(Xd, fd, Qd, k, weighting, return_dk=True)
        ref, rdk = O.knn_regress(X, f, Q, k, weighting)
        assert np.array_equal(dk.cpu().numpy(), rdk), k                       # d2_(k) bit-exact
        np.testing.assert_allclose(out.cpu().numpy(), ref.astype(np.float32), rtol=2e-6, atol=1e-6)


def test_knn_errors(cp):
    import torch
    X, f, Q = problem(100, 2, 3, 1)
    Xd, fd, Qd = (torch.from_numpy(v).cuda() for v in (X, f, Q))
    with pytest.raises(ValueError):
        cp.knn_regress(Xd, fd, Qd, 0)
    with pytest.raises(ValueError):
        cp.knn_regress(Xd, fd, Qd, 101)
    fb = fd.clone()
    fb[5] = float("nan")
    with pytest.raises(ValueError):
        cp.knn_regress(Xd, fb, Qd, 3)
    Qb = Qd.clone()
    Qb[1, 1] = float("inf")
    with pytest.raises(ValueError):
        cp.knn_regress(Xd, fd, Qb, 3)


@pytest.mark.parametrize("ties", [False, True])
@pytest.mark.parametrize("weighting", [0, 1])
def test_knn_classify_matches_oracle(cp, ties, weighting):
    import torch
    n, p, nq, C = 100_003, 4, 29, 7
    X, _, Q = problem(n, p, nq, 5 + int(ties), ties)
    lab = np.random.default_rng(9).integers(0, C, n).astype(np.int32)
    Xd, ld, Qd = torch.from_numpy(X).cuda(), torch.from_numpy(lab).cuda(), torch.from_numpy(Q).cuda()
    for k in (1, 9, 200):
        got, votes = cp.knn_classify(Xd, ld, Qd, k, C, weighting, return_votes=True)
        ref, rvotes = O.knn_classify(X, lab, Q, k, C, weighting)
        np.testing.assert_allclose(votes.cpu().numpy(), rvotes, rtol=1e-12, atol=1e-12 * k)
        gap = np.sort(rvotes, axis=1)[:, -1] - np.sort(rvotes, axis=1)[:, -2]
        sure = gap > 1e-9 * np.max(rvotes, axis=1)   # the winner is decided beyond rounding
        assert np.array_equal(got.cpu().numpy()[sure], ref[sure]), k
    with pytest.raises(ValueError):
        cp.knn_classify(Xd, torch.full_like(ld, C), Qd, 3, C)
