"""Two 2^28 f64 uniform medians (the direct chain) — for an ncu capture of init_seg_kernel<double>."""
import sys

import torch

sys.path.insert(0, ".")
import datagen  # noqa: E402
import paper_1104_2732_b200 as cp  # noqa: E402

x = datagen.make("uniform", 1 << 28, "f64", device="cuda")
for _ in range(2):
    cp.median(x)
torch.cuda.synchronize()
print("ok")
