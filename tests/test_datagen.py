"""The seeded input generators (no method arithmetic): the shard-invariant global generator used
by the strong-scaling runs of configs[3] gives every rank exactly its block of one global array."""
import numpy as np

import datagen


def test_make_global_is_shard_invariant():
    n = 10_007
    for dist in datagen.GLOBAL_DISTS:
        for dtype in ("f32", "f64"):
            full = datagen.make_global(dist, n, 0, n, dtype)
            for G in (2, 3, 8):
                b = [n * g // G for g in range(G + 1)]
                parts = [datagen.make_global(dist, n, b[g], b[g + 1], dtype, chunk=999) for g in range(G)]
                import torch
                assert torch.equal(torch.cat(parts), full)


def test_make_global_moments():
    import torch
    n = 1 << 20
    u = datagen.make_global("uniform", n, 0, n, "f32").double()
    assert u.min() >= 0 and u.max() < 1 and abs(float(u.mean()) - 0.5) < 3e-3
    assert len(torch.unique(u)) > n * 0.95
    z = datagen.make_global("normal", n, 0, n, "f64")
    assert abs(float(z.mean())) < 5e-3 and abs(float(z.std()) - 1.0) < 5e-3
    assert np.isfinite(z.numpy()).all()
