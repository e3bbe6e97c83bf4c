"""LMS configuration (BASELINE configs[4]): n=1e6, p=10, C=4096.  Times the tcgen05 residual GEMM
(a7), the batched selection (a8) and the whole cpsel_lms_objective with CUDA events; one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import datagen  # noqa: E402
import paper_1104_2732_b200 as cp  # noqa: E402


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        r = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, r


n, p, C = 1_000_000, 10, 4096
X, y, th, _ = datagen.lms_problem(n=n, p=p, C=C)
Xd, yd, thd = (torch.from_numpy(a).cuda() for a in (X, y, th))
S = torch.empty((C, n), device="cuda", dtype=torch.float32)
ms_gemm, _ = timed(lambda: cp.lms_residuals(Xd, yd, thd, out=S))
k = (n + 1) // 2
ms_sel, (out, info) = timed(lambda: cp.select_kth_batched(S, k, return_info=True))
ms_all, (obj, info2) = timed(lambda: cp.lms_objective(Xd, yd, thd, return_info=True))
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
gemm_bytes = 4 * n * C
print(json.dumps({
    "config": {"workload": "LMS objective n=1e6 p=10 C=4096 (BASELINE configs[4])"},
    "gemm_ms": ms_gemm, "gemm_write_GBps": gemm_bytes / ms_gemm / 1e6,
    "gemm_frac_of_hbm": gemm_bytes / ms_gemm / 1e6 / peak,
    "gemm_tflops_3xtf32": 3 * 2 * n * 16 * C / ms_gemm / 1e9,
    "select_ms": ms_sel, "select_elements_per_s": n * C / (ms_sel / 1e3),
    "select_bytes": info["bytes_moved"], "select_GBps": info["bytes_moved"] / ms_sel / 1e6,
    "select_passes_per_column": info["passes"] / C,
    "objective_ms": ms_all, "objective_candidates_per_s": C / (ms_all / 1e3),
}))
