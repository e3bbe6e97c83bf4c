"""Drive single kernels for ncu: a compacting full pass, bracket passes, the LMS residual GEMM and
the batched selection.  Usage under ncu (one GPU):  python scripts/prof_kernels.py {select,lms,lms_fused}"""
import sys

import torch

sys.path.insert(0, ".")
import datagen  # noqa: E402
import paper_1104_2732_b200 as cp  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "select"
if what == "select":
    x = datagen.make("uniform", 1 << 30, "f32", device="cuda")
    torch.cuda.synchronize()
    for _ in range(2):
        v, info = cp.median(x, return_info=True)
    print(v, info)
elif what == "lms":
    X, y, th, _ = datagen.lms_problem()
    Xd, yd, thd = (torch.from_numpy(a).cuda() for a in (X, y, th))
    for _ in range(2):
        S = cp.lms_residuals(Xd, yd, thd)
        torch.cuda.synchronize()
        out, info = cp.select_kth_batched(S, (X.shape[0] + 1) // 2, return_info=True)
        torch.cuda.synchronize()
    print(info)
elif what == "lms_fused":
    X, y, th, _ = datagen.lms_problem()
    Xd, yd, thd = (torch.from_numpy(a).cuda() for a in (X, y, th))
    cp.set_config(lms_fused=1)
    for _ in range(2):
        out, info = cp.lms_objective(Xd, yd, thd, return_info=True)
        torch.cuda.synchronize()
    print(info)
