"""Small workload touching every kernel, for compute-sanitizer (memcheck / racecheck / synccheck):
fused init+cuts+compaction, segmented passes (both variants), dense compaction, radix select,
direct eval, batched selection, tcgen05 residuals, sharded (world 1) path."""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import datagen  # noqa: E402
import oracle as O  # noqa: E402
import paper_1104_2732_b200 as cp  # noqa: E402

n = (1 << 21) + 3
for dist, dtype in (("normal", "f32"), ("cauchy", "f64")):
    x = datagen.make(dist, n, dtype)
    xd = torch.from_numpy(x).cuda()[1:]          # misaligned start
    xs = x[1:]
    for k in (1, 1000, O.median_rank(xs.size), xs.size - 7):
        v = cp.select_kth(xd, k)
        assert (0.0 if v == 0 else v) == float(O.order_statistic(xs, k)), (dist, dtype, k)
    s = cp.eval(xd, float(xs[77]), -math.inf, math.inf)
    assert s["c_lt"] == int((xs < xs[77]).sum())
cp.set_config(init_cut=0)
x = datagen.make("uniform", n, "f32")
assert cp.median(torch.from_numpy(x).cuda()) == float(O.median(x))
cp.set_config(init_cut=1)
S = torch.from_numpy(datagen.make("halfnormal", 3000 * 40, "f32").reshape(40, 3000)).cuda()
out = cp.select_kth_batched(S, 1500).cpu().numpy()
Sh = S.cpu().numpy()
assert all(out[j] == O.order_statistic(Sh[j], 1500) for j in range(40))
X, y, th, _ = datagen.lms_problem(n=3001, p=10, C=300)
R = cp.lms_residuals(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), torch.from_numpy(th).cuda())
torch.cuda.synchronize()
uid = cp.nccl_unique_id()
cp.comm_init(uid, 0, 1, 0)
x = datagen.make("mix1", n, "f32")
assert cp.select_kth_sharded(torch.from_numpy(x).cuda(), 12345) == float(O.order_statistic(x, 12345))
# round-1 additions: the direct device chain (init-counted radix round 0, n >= 2^27), the one-launch
# small-array path, the fused LMS / LTS tensor-core passes and their stored-S fallback
for dtype in ("f32", "f64"):
    xb = datagen.make("normal", (1 << 27) + 5, dtype, device="cuda")
    kb = O.median_rank(xb.numel())
    vb = cp.select_kth(xb, kb)
    assert (0.0 if vb == 0 else vb) == float(torch.kthvalue(xb.cpu(), kb).values), dtype
    del xb
for dtype, m in (("f32", 100_000), ("f64", 5_000)):
    xs = datagen.make("cauchy", m, dtype)
    assert cp.median(torch.from_numpy(xs).cuda()) == float(O.median(xs))
X, y, th, _ = datagen.lms_problem(n=20_011, p=10, C=140)
Xd, yd, thd = (torch.from_numpy(a).cuda() for a in (X, y, th))
got = cp.lms_objective(Xd, yd, thd).cpu().numpy()
S = cp.lms_residuals(Xd, yd, thd).cpu().numpy()
assert all(got[j] == O.order_statistic(S[j], O.median_rank(X.shape[0])) for j in range(140))
F, mth = cp.lts_objective(Xd, yd, thd, (X.shape[0] + 10) // 2)
torch.cuda.synchronize()
# round-2 additions: the cooperative radix select (every path above), the device-resident Kelley
# loop (CUDA graph), the bisection driver, kNN, and the loopback-sharded path at G = 2
x = datagen.make("mix2", n, "f32")
xd = torch.from_numpy(x).cuda()
for cfg in (dict(init_cut=0, pass_cuts=0, objective=1, device_loop=1), dict(init_cut=0, pass_cuts=0, driver=1),
            dict(init_cut=0, pass_cuts=0, driver=3)):
    cp.set_config(**cfg)
    assert cp.select_kth(xd, 777) == float(O.order_statistic(x, 777)), cfg
    cp.set_config(init_cut=1, pass_cuts=1, objective=0, device_loop=0, driver=0)
rng = np.random.default_rng(1)
Xk = rng.standard_normal((5000, 3)).astype(np.float32)
fk = rng.standard_normal(5000).astype(np.float32)
Qk = rng.standard_normal((20, 3)).astype(np.float32)
out, dk = cp.knn_regress(*(torch.from_numpy(a).cuda() for a in (Xk, fk, Qk)), 9, return_dk=True)
assert np.array_equal(dk.cpu().numpy(), O.knn_regress(Xk, fk, Qk, 9)[1])
import threading
grp = cp.LoopbackGroup(2)
res = [None, None]
xs = datagen.make("uniform", 9_000_001, "f32")
xsd = torch.from_numpy(xs).cuda()
torch.cuda.synchronize()


def rank(g):
    with torch.cuda.stream(torch.cuda.Stream()):
        cp.comm_init_loopback(grp, g, 0)
        res[g] = cp.select_kth_sharded(xsd[g * 4_000_000:(g + 1) * 4_000_000] if g == 0 else xsd[4_000_000:], 4_500_001)


th_ = [threading.Thread(target=rank, args=(g,)) for g in range(2)]
[t.start() for t in th_]
[t.join() for t in th_]
assert res[0] == res[1] == float(O.order_statistic(xs, 4_500_001)), res
torch.cuda.synchronize()
print("sanitize workload ok")
# round-2 (late) additions: the value-binned finish's overflow fallback (a dense cluster at the
# target), f64 through the value bins, Brent's minimisation driver (above)
nb = (1 << 23) + 11
rng = np.random.default_rng(23)
xc = rng.random(nb).astype(np.float32)
idc = rng.choice(nb, 40_000, replace=False)
xc[idc] = np.float32(0.5) + np.float32(np.spacing(np.float32(0.5))) * rng.integers(0, 10, idc.size).astype(np.float32)
assert cp.median(torch.from_numpy(xc).cuda()) == float(O.median(xc))
xf = rng.random(nb)
assert cp.median(torch.from_numpy(xf).cuda()) == float(O.median(xf))
torch.cuda.synchronize()
print("sanitize workload ok")
