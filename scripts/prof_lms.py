"""One fused LMS objective at configs[4] (n=1e6, p=10, C=4096) after one warm-up — the target of
`ncu -k regex:fused_tc_kernel` captures (profiles/r02_ncu_lms_fused*.md)."""
import sys

import torch

sys.path.insert(0, ".")
import datagen  # noqa: E402
import paper_1104_2732_b200 as cp  # noqa: E402

X, y, th, _ = datagen.lms_problem(n=1_000_000, p=10, C=4096)
Xd, yd, thd = (torch.from_numpy(a).cuda() for a in (X, y, th))
for _ in range(2):
    out = cp.lms_objective(Xd, yd, thd)
torch.cuda.synchronize()
print("ok", float(out[:8].sum()))
