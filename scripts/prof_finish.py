"""Four 2^30 f32 medians and two 2^28 f64 medians after a warm-up, for an ncu launch list of the
direct chain's kernels (compare CPSEL_VBIN=0/1)."""
import sys

import torch

sys.path.insert(0, ".")
import datagen  # noqa: E402
import paper_1104_2732_b200 as cp  # noqa: E402

for lg, dtype, dists in ((30, "f32", ("uniform", "normal", "cauchy", "dup256")), (28, "f64", ("uniform", "normal"))):
    for dist in dists:
        x = datagen.make(dist, 1 << lg, dtype, device="cuda")
        cp.median(x)
        torch.cuda.synchronize()
        cp.median(x)
        torch.cuda.synchronize()
        del x
        torch.cuda.empty_cache()
print("ok")
