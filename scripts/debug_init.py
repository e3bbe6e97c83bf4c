import sys, numpy as np, torch
sys.path.insert(0, '.')
import datagen, paper_1104_2732_b200 as cp
for lg in (24, 26, 28, 30):
    for dist in ("uniform", "dup256"):
        xd = datagen.make(dist, 1 << lg, "f32", device="cuda")
        s = cp.init_stats(xd)
        mn = xd.min().item(); mx = xd.max().item()
        cmin = int((xd == mn).sum().item()); cmax = int((xd == mx).sum().item())
        v, info = cp.median(xd, return_info=True)
        print(lg, dist, s, "torch:", mn, cmin, mx, cmax, "median", v, info["exit"], info["cp_iters"], flush=True)
        del xd; torch.cuda.empty_cache()
