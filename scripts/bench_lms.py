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
k = (n + 1) // 2
h = (n + p) // 2
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
gemm_bytes = 4 * n * C
res = {"config": {"workload": "LMS objective n=1e6 p=10 C=4096 (BASELINE configs[4])"}}
# unfused: S stored by the row-major residual kernel, then the batched selection reads it
cp.set_config(lms_fused=0)
ms_gemm, _ = timed(lambda: cp.lms_residuals(Xd, yd, thd, out=S))
S0 = S.clone() if "--cmp" in sys.argv else None
ms_sel, (out, info) = timed(lambda: cp.select_kth_batched(S, k, return_info=True))
ms_all0, (obj0, _) = timed(lambda: cp.lms_objective(Xd, yd, thd, return_info=True))
ms_lts0, _ = timed(lambda: cp.lts_objective(Xd, yd, thd, h), reps=3, warm=1)
res["unfused"] = {
    "gemm_ms": ms_gemm, "gemm_write_GBps": gemm_bytes / ms_gemm / 1e6,
    "gemm_frac_of_hbm": gemm_bytes / ms_gemm / 1e6 / peak,
    "gemm_tflops_3xtf32": 3 * 2 * n * 16 * C / ms_gemm / 1e9,
    "select_ms": ms_sel, "select_elements_per_s": n * C / (ms_sel / 1e3),
    "select_bytes": info["bytes_moved"], "select_GBps": info["bytes_moved"] / ms_sel / 1e6,
    "select_passes_per_column": info["passes"] / C,
    "objective_ms": ms_all0, "objective_candidates_per_s": C / (ms_all0 / 1e3), "lts_ms": ms_lts0,
}
# fused: no S; residuals recomputed in the tcgen05 epilogue of one pass per objective
cp.set_config(lms_fused=1)
ms_all1, (obj1, info1) = timed(lambda: cp.lms_objective(Xd, yd, thd, return_info=True))
ms_lts1, _ = timed(lambda: cp.lts_objective(Xd, yd, thd, h), reps=3, warm=1)
res["fused"] = {
    "objective_ms": ms_all1, "objective_candidates_per_s": C / (ms_all1 / 1e3),
    "elements_per_s": n * C / (ms_all1 / 1e3),
    "fused_pass_ms": info1["kernel_ms_init"], "continuation_ms": info1["kernel_ms_passes"],
    "fallback_columns": info1["fallback_steps"], "passes_per_column": info1["passes"] / C,
    "tensor_tflops_3xtf32_in_fused_pass": 3 * 2 * n * 16 * C / info1["kernel_ms_init"] / 1e9,
    "lts_ms": ms_lts1,
}
if S0 is not None:
    cp.lms_residuals(Xd, yd, thd, out=S)
    res["fused_vs_unfused_S_bit_identical_frac"] = float((S == S0).float().mean())
    res["objective_equal_frac"] = float((obj0 == obj1).float().mean())
print(json.dumps(res))
