"""A/B helper for the direct chain's exact finish: ms per selection (CUDA events, best of 5) for the
bench's four 2^30 f32 medians, configs[1]'s 2^24 f32 ranks and configs[2]'s 2^28 f64 ranks; run once
per setting of CPSEL_VBIN (read at first use).  Usage: CPSEL_VBIN=0|1 python scripts/time_finish.py"""
import os
import sys

import torch

sys.path.insert(0, ".")
import datagen  # noqa: E402
import oracle as O  # noqa: E402
import paper_1104_2732_b200 as cp  # noqa: E402

tag = "vbin=" + os.environ.get("CPSEL_VBIN", "1")


def best(x, k, reps=5):
    cp.select_kth(x, k)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        v = cp.select_kth(x, k)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts), v


rows = []
for lg, dtype, ks in ((30, "f32", ("med",)), (24, "f32", ("med", 1, "n10", "nm1")), (28, "f64", ("med", "n10"))):
    for dist in ("uniform", "normal", "cauchy", "dup256"):
        if dtype == "f64" and dist in ("cauchy", "dup256"):
            continue
        x = datagen.make(dist, 1 << lg, dtype, device="cuda")
        n = x.numel()
        for kk in ks:
            k = {"med": (n + 1) // 2, "n10": n // 10, "nm1": n - 1}.get(kk, kk)
            ms, v = best(x, k)
            xs = x[:: max(1, n // (1 << 20))].cpu().numpy()
            ok = (x < v).sum().item() < k <= (x <= v).sum().item()
            rows.append(f"{tag} 2^{lg} {dtype} {dist:8s} k={kk!s:4s} {ms * 1e3:8.1f} us  rank_ok={ok}")
        del x
        torch.cuda.empty_cache()
print("\n".join(rows))
