"""Debug: how many columns of configs[4] should the fused path's R23 cuts miss?  Replays the cut
rule (16384 strided sample rows, ranks q -/+ (3.5 sd + 2), 22-bit key bin edges) on the GPU's S."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import datagen  # noqa: E402
import paper_1104_2732_b200 as cp  # noqa: E402

n, p, C = 1_000_000, 10, 4096
X, y, th, _ = datagen.lms_problem(n=n, p=p, C=C)
Xd, yd, thd = (torch.from_numpy(a).cuda() for a in (X, y, th))
out, info = cp.lms_objective(Xd, yd, thd, return_info=True)
print("fallback", info["fallback_steps"])
S = cp.lms_residuals(Xd, yd, thd)
ms = 16384
rows = torch.from_numpy((np.arange(ms, dtype=np.int64) * n) // ms + (n // ms) // 2).cuda()
k = (n + 1) // 2
q = (k - 0.5) / n * ms
w = 3.5 * np.sqrt(max(q * (ms - q) / ms, 0.0)) + 2.0
il, ih = int(np.floor(q - w)), int(np.ceil(q + w))
Ss = S[:, rows]
srt = torch.sort(Ss, dim=1).values
lo, hi = srt[:, il], srt[:, ih]
le = (S <= lo[:, None]).sum(1)
lt = (S < hi[:, None]).sum(1)
miss = ~((le < k) & (k <= lt))
print("exact-quantile misses", int(miss.sum()), "interior mean frac", float((lt - le).float().mean() / n))
kth = torch.kthvalue(S, k, dim=1).values
print("objective equal to kthvalue:", bool((kth == out).all()))
bad = torch.nonzero(miss).flatten()[:10].tolist()
for j in bad:
    print(j, float(lo[j]), float(hi[j]), float(kth[j]), int(le[j]), int(lt[j]))
