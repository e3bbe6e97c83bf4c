"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the selection method: it only draws random
samples with the shapes and distributions of the paper's workloads.  Both the
CUDA path and the oracle receive the *same* array produced here (a GPU tensor is
copied to the host for the oracle), so neither side depends on the other.

Distributions follow PAPER.md §5.1:
  uniform    U(0,1)
  normal     N(0,1)
  halfnormal |N(0,1)|
  beta25     Beta(2,5)
  mix1       2/3 N(0,1) + 1/3 N(100,1)
  mix2       1/2 N(0,1)+1 + 1/2 N(100,1)         (reading DESIGN.md R15)
  mix3       9/10 halfnormal + 1/10 constant 10
  mix4       2/3 halfnormal + 1/3 N(100,1)
  mix5       1/2 halfnormal+1 + 1/2 N(100,1)     (reading R15)
plus the BASELINE.json extras
  cauchy     standard Cauchy (heavy tailed)
  dup256     floor(256*U(0,1)): 256 distinct values, ~n/256 copies each
Mixture membership is a per-element Bernoulli draw with the stated proportion.
Outliers ("very large values ~1e9", "~1e20") are injected by
`inject_outliers` at seeded positions.

Generation back ends:
  device="cpu"  -> numpy Philox (np.random.Generator(np.random.Philox)), returns np.ndarray
  device="cuda" -> torch.Generator(device="cuda"), returns a CUDA torch.Tensor
Each is deterministic for a fixed (dist, n, dtype, seed); the two back ends draw
different streams (tests always give both sides the same array).
"""
from __future__ import annotations

import numpy as np

SEED = 11042732  # arXiv id, the default seed of every synthetic input

PAPER_DISTS = ["uniform", "normal", "halfnormal", "beta25",
               "mix1", "mix2", "mix3", "mix4", "mix5"]
EXTRA_DISTS = ["cauchy", "dup256"]
ALL_DISTS = PAPER_DISTS + EXTRA_DISTS
BENCH_DISTS = ["uniform", "normal", "cauchy", "dup256"]  # BASELINE.json configs[1]

_STREAM = {d: i + 1 for i, d in enumerate(ALL_DISTS)}


def _np_dtype(dtype: str):
    return {"f32": np.float32, "f64": np.float64}[dtype]


# ----------------------------------------------------------------------------- numpy
def _np_rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(np.random.SeedSequence([seed, stream])))


def _np_draw(dist: str, n: int, rng: np.random.Generator) -> np.ndarray:
    """float64 draws for one distribution (cast by the caller)."""
    if dist == "uniform":
        return rng.random(n)
    if dist == "normal":
        return rng.standard_normal(n)
    if dist == "halfnormal":
        return np.abs(rng.standard_normal(n))
    if dist == "beta25":
        return rng.beta(2.0, 5.0, n)
    if dist == "cauchy":
        return rng.standard_cauchy(n)
    if dist == "dup256":
        return np.floor(256.0 * rng.random(n))
    if dist in ("mix1", "mix2", "mix3", "mix4", "mix5"):
        u = rng.random(n)
        a = rng.standard_normal(n)
        b = rng.standard_normal(n) + 100.0
        if dist == "mix1":
            return np.where(u < 2.0 / 3.0, a, b)
        if dist == "mix2":
            return np.where(u < 0.5, a + 1.0, b)
        if dist == "mix3":
            return np.where(u < 0.9, np.abs(a), 10.0)
        if dist == "mix4":
            return np.where(u < 2.0 / 3.0, np.abs(a), b)
        return np.where(u < 0.5, np.abs(a) + 1.0, b)  # mix5
    raise ValueError(f"unknown distribution {dist!r}")


# ----------------------------------------------------------------------------- torch (device)
def _torch_draw(dist: str, n: int, dtype: str, seed: int, device):
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed * 64 + _STREAM[dist])
    tdt = {"f32": torch.float32, "f64": torch.float64}[dtype]

    def U():
        return torch.rand(n, generator=g, device=device, dtype=tdt)

    def N():
        return torch.randn(n, generator=g, device=device, dtype=tdt)

    if dist == "uniform":
        return U()
    if dist == "normal":
        return N()
    if dist == "halfnormal":
        return N().abs_()
    if dist == "cauchy":
        return torch.empty(n, device=device, dtype=tdt).cauchy_(generator=g)
    if dist == "dup256":
        return U().mul_(256.0).floor_()
    if dist == "beta25":
        # Beta(2,5) = G2/(G2+G5), G_a = -sum_{i<a} log U_i (integer-shape gamma)
        g2 = -(U().log_() + U().log_())
        g5 = -(U().log_() + U().log_() + U().log_() + U().log_() + U().log_())
        return g2.div_(g2 + g5)
    if dist in ("mix1", "mix2", "mix3", "mix4", "mix5"):
        u = U()
        a = N()
        b = N().add_(100.0)
        if dist == "mix1":
            return torch.where(u < 2.0 / 3.0, a, b)
        if dist == "mix2":
            return torch.where(u < 0.5, a + 1.0, b)
        if dist == "mix3":
            return torch.where(u < 0.9, a.abs(), torch.full_like(a, 10.0))
        if dist == "mix4":
            return torch.where(u < 2.0 / 3.0, a.abs(), b)
        return torch.where(u < 0.5, a.abs() + 1.0, b)
    raise ValueError(f"unknown distribution {dist!r}")


def make(dist: str, n: int, dtype: str = "f32", seed: int = SEED, device: str = "cpu"):
    """Draw n values of `dist` in `dtype` ("f32"|"f64").

    device="cpu" returns a numpy array; any other device returns a torch tensor there.
    """
    if n < 0:
        raise ValueError("n must be >= 0")
    if str(device) == "cpu":
        if dist not in _STREAM:
            raise ValueError(f"unknown distribution {dist!r}")
        x = _np_draw(dist, n, _np_rng(seed, _STREAM[dist]))
        return np.ascontiguousarray(x.astype(_np_dtype(dtype)))
    return _torch_draw(dist, n, dtype, seed, device)


def inject_outliers(x, count: int, magnitude: float, seed: int = SEED, sign: int = +1):
    """Overwrite `count` seeded positions of x (in place) with sign*magnitude."""
    n = len(x)
    pos = _np_rng(seed, 1000 + count).choice(n, size=min(count, n), replace=False)
    if isinstance(x, np.ndarray):
        x[pos] = sign * magnitude
    else:
        import torch
        x[torch.as_tensor(pos, device=x.device)] = sign * magnitude
    return x


def lms_problem(n: int = 1_000_000, p: int = 10, C: int = 4096, seed: int = SEED,
                outlier_frac: float = 0.3):
    """Synthetic LMS workload of BASELINE.json configs[4] (P:L438-449 model (model)).

    X: n x p float32 row-major, columns 0..p-2 ~ N(0,1), column p-1 = 1 (intercept).
    y = X theta* + eps, eps ~ N(0,1); a fraction `outlier_frac` of rows gets y += 100 + 10 N(0,1).
    thetas: p x C float32 column-major (i.e. array of shape (C, p) row-major):
            theta_j = theta* + sigma_j N(0, I), sigma_j log-spaced in [1e-3, 1].
    Returns numpy arrays (X[n,p], y[n], thetas_cp[C,p], theta_star[p]).
    """
    rng = _np_rng(seed, 4242)
    X = rng.standard_normal((n, p))
    X[:, p - 1] = 1.0
    theta_star = rng.standard_normal(p)
    y = X @ theta_star + rng.standard_normal(n)
    out = rng.random(n) < outlier_frac
    y[out] += 100.0 + 10.0 * rng.standard_normal(int(out.sum()))
    sig = np.logspace(-3.0, 0.0, C)
    thetas = theta_star[None, :] + sig[:, None] * rng.standard_normal((C, p))
    return (np.ascontiguousarray(X.astype(np.float32)), y.astype(np.float32),
            np.ascontiguousarray(thetas.astype(np.float32)), theta_star)


# ----------------------------------------------------------------------------- shard-invariant
# "generated on device; shard-invariant" — element i of the global array is a pure
# function of (seed, distribution, i), so rank g of G can draw exactly its block [lo, hi) and the
# concatenation over ranks is the same array for every G (the strong-scaling runs of configs[3]
# select from identical data at G = 1, 2, 4, 8).  Counter-based: splitmix64 of the global index,
# in int64 torch ops (wrapping multiply; logical shifts by masking), on any torch device.
_M64 = (1 << 64) - 1


def _s64(c: int) -> int:
    return c - (1 << 64) if c >= (1 << 63) else c


_SM_GAMMA, _SM_M1, _SM_M2 = _s64(0x9E3779B97F4A7C15), _s64(0xBF58476D1CE4E5B9), _s64(0x94D049BB133111EB)


def _shr(z, s: int):
    """logical right shift of int64 (torch's >> is arithmetic)"""
    return (z >> s) & ((1 << (64 - s)) - 1)


def _splitmix(idx, key: int):
    z = idx * _SM_GAMMA + _s64((key * 0xD1B54A32D192ED03) & _M64)
    z = (z ^ _shr(z, 30)) * _SM_M1
    z = (z ^ _shr(z, 27)) * _SM_M2
    return z ^ _shr(z, 31)


GLOBAL_DISTS = ["uniform", "normal"]  # configs[3]


def make_global(dist: str, n_global: int, lo: int, hi: int, dtype: str = "f32", seed: int = SEED,
                device="cpu", chunk: int = 1 << 26):
    """Elements [lo, hi) of the shard-invariant global array of n_global values of `dist`
    (uniform: 24 (f32) / 53 (f64) random bits; normal: Box-Muller of two such uniforms, in f64).
    Returns a torch tensor on `device`."""
    import torch
    if not (0 <= lo <= hi <= n_global):
        raise ValueError("need 0 <= lo <= hi <= n_global")
    if dist not in GLOBAL_DISTS:
        raise ValueError(f"make_global supports {GLOBAL_DISTS}")
    tdt = {"f32": torch.float32, "f64": torch.float64}[dtype]
    out = torch.empty(hi - lo, dtype=tdt, device=device)
    key = (seed * 64 + _STREAM[dist]) & _M64
    for a in range(lo, hi, chunk):
        b = min(a + chunk, hi)
        idx = torch.arange(a, b, dtype=torch.int64, device=device)
        if dist == "uniform":
            z = _splitmix(idx, key)
            if dtype == "f32":
                v = _shr(z, 40).to(torch.float32) * (2.0 ** -24)
            else:
                v = _shr(z, 11).to(torch.float64) * (2.0 ** -53)
        else:
            u1 = (_shr(_splitmix(idx, key), 11).to(torch.float64) + 1.0) * (2.0 ** -53)   # (0, 1]
            u2 = _shr(_splitmix(idx, key ^ 0x5DEECE66D), 11).to(torch.float64) * (2.0 ** -53)
            v = torch.sqrt(-2.0 * torch.log(u1)) * torch.cos((2.0 * np.pi) * u2)
        out[a - lo:b - lo] = v.to(tdt)
        del idx
    return out
