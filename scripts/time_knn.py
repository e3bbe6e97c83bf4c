"""kNN regression via d_(k) (§8f-4): time one configuration.  python scripts/time_knn.py [n] [p] [nq] [k]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1104_2732_b200 as cp  # noqa: E402

n, p, nq, k = (int(v) for v in (sys.argv[1:] + ["1000000", "10", "1024", "32"][len(sys.argv) - 1:])[:4])
rng = np.random.default_rng(11042732)
X = rng.standard_normal((n, p)).astype(np.float32)
f = (np.sin(X[:, 0]) + 0.1 * rng.standard_normal(n)).astype(np.float32)
Q = rng.standard_normal((nq, p)).astype(np.float32)
Xd, fd, Qd = (torch.from_numpy(v).cuda() for v in (X, f, Q))
cp.knn_regress(Xd, fd, Qd, k)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    out, info = cp.knn_regress(Xd, fd, Qd, k, return_info=True)
e1.record()
torch.cuda.synchronize()
print(f"n={n} p={p} nq={nq} k={k}: {e0.elapsed_time(e1) / 3:.3f} ms, passes/query {info['passes'] / nq:.2f}")
