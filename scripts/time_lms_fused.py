"""Time the fused LMS objective (configs[4]) and its fused stage with CUDA events; one line.
Usage: python scripts/time_lms_fused.py [label]"""
import sys

import torch

sys.path.insert(0, ".")
import datagen  # noqa: E402
import paper_1104_2732_b200 as cp  # noqa: E402

X, y, th, _ = datagen.lms_problem(n=1_000_000, p=10, C=4096)
Xd, yd, thd = (torch.from_numpy(a).cuda() for a in (X, y, th))
best = None
for _ in range(6):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out, info = cp.lms_objective(Xd, yd, thd, return_info=True)
    e1.record()
    torch.cuda.synchronize()
    t = (e0.elapsed_time(e1), info["kernel_ms_init"], info["kernel_ms_passes"])
    best = t if best is None or t[0] < best[0] else best
print(sys.argv[1] if len(sys.argv) > 1 else "", "objective %.3f ms, fused stage %.3f ms, continuation %.3f ms" % best)
