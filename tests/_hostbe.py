"""Numpy data steps for libcpsel's host-only driver (cpsel_drive_host).

The driver (C++) decides every query point; these callbacks only evaluate one pass over a
(possibly sharded) numpy array, exactly as the CUDA kernels would, and combine shards through
an optional `comm` (gloo all-gather).  Test infrastructure, not the product path."""
import math

import numpy as np


def sample_keys(x, smax=1024):
    """Sorted order-preserving keys of min(len(x), smax) evenly strided samples of x, padded to 1024
    with ~0 (the layout the R28 pooled pick takes)."""
    m = x.size
    ms = min(m, smax)
    pos = np.arange(ms) if m == ms else (np.arange(ms, dtype=np.int64) * m) // ms + (m // ms) // 2
    v = x[pos]
    if v.dtype == np.float32:
        u = v.view(np.uint32).astype(np.uint64)
        k = np.where(u >> 31, (~u) & 0xFFFFFFFF, u | 0x80000000)
    else:
        u = v.view(np.uint64)
        k = np.where(u >> 63, ~u, u | np.uint64(1 << 63))
    out = np.full(1024, np.iinfo(np.uint64).max, dtype=np.uint64)
    out[:ms] = np.sort(k.astype(np.uint64))
    return out


class NumpyShard:
    def __init__(self, x, comm=None, cut_k=None, cut_shift=0.0):
        self.x = np.ascontiguousarray(x)
        self.cut_shift = cut_shift  # R26 cut pass: move the sample cuts by this fraction of the sample
        self.cut_k = cut_k  # evaluate the init pass's extra cut at a sample quantile of rank cut_k
        self.comm = comm  # callable: obj -> list of objs from every rank (rank order)
        self.kept = None
        self.cur = self.x

    def _gather(self, obj):
        return [obj] if self.comm is None else self.comm(obj)

    def init(self):
        x = self.x
        if x.size:
            mn, mx = x.min(), x.max()
            rec = {"vmin": float(mn), "vmax": float(mx), "cnt_min": int((x == mn).sum()),
                   "cnt_max": int((x == mx).sum()), "nonfinite": int((~np.isfinite(x)).sum()),
                   "x0": float(x[0]), "S": float(np.sum(x.astype(np.float64) - np.float64(x[0]))), "n": x.size}
        else:
            rec = {"vmin": math.inf, "vmax": -math.inf, "cnt_min": 0, "cnt_max": 0, "nonfinite": 0,
                   "x0": 0.0, "S": 0.0, "n": 0}
        out = None
        S = 0.0
        for r in self._gather(rec):
            if r["n"] == 0:
                continue
            if out is None:
                out = dict(r)
                S = r["S"]
                continue
            if r["vmin"] < out["vmin"]:
                out["vmin"], out["cnt_min"] = r["vmin"], r["cnt_min"]
            elif r["vmin"] == out["vmin"]:
                out["cnt_min"] += r["cnt_min"]
            if r["vmax"] > out["vmax"]:
                out["vmax"], out["cnt_max"] = r["vmax"], r["cnt_max"]
            elif r["vmax"] == out["vmax"]:
                out["cnt_max"] += r["cnt_max"]
            out["nonfinite"] += r["nonfinite"]
            S += r["S"] + r["n"] * (r["x0"] - out["x0"])
        out["S"] = S
        if self.cut_k is not None and self.comm is not None and sum(self._gather(x.size)) > 2:
            # R28: cuts common to all ranks from the pooled samples, statistics summed over ranks
            import paper_1104_2732_b200 as cp
            sizes = self._gather(x.size)
            keys = np.stack(self._gather(sample_keys(x)))
            dt = "f32" if x.dtype == np.float32 else "f64"
            tl, th, te = cp.pooled_cuts(keys, sizes, self.cut_k, dt)
            xd = x.astype(np.float64)
            inner = (x > tl) & (x < th)
            mine = {"c_le_lo": int((x <= tl).sum()), "c_lt_hi": int((x < th).sum()),
                    "N_lo": float(np.sum(tl - xd[x < tl])), "P_hi": float(np.sum(xd[x > th] - th)),
                    "I_in": float(np.sum(xd[inner] - tl))}
            tot = {key: sum(r[key] for r in self._gather(mine)) for key in mine}
            out.update(has_cut=6, t_lo=float(tl), t_hi=float(th), t_est=float(te), **tot)
        if self.cut_k is not None and self.comm is None and x.size > 2:
            # R23: two cuts at the sample quantiles bracketing rank k (1024 strided samples)
            n = x.size
            m = min(n, 1024)
            pos = np.arange(m) if n == m else (np.arange(m, dtype=np.int64) * n) // m + (n // m) // 2
            smp = np.sort(x[pos])
            q = (self.cut_k - 0.5) / n * m
            w = 3.5 * math.sqrt(max(q * (m - q) / m, 0.0)) + 2.0
            il, ih = max(int(math.floor(q - w)), 0), min(int(math.ceil(q + w)), m - 1)
            tl, th = np.float64(smp[il]), np.float64(smp[ih])
            xd = x.astype(np.float64)
            inner = (x > tl) & (x < th)
            out.update(has_cut=6, t_lo=float(tl), t_hi=float(th),
                       c_le_lo=int((x <= tl).sum()), c_lt_hi=int((x < th).sum()),
                       N_lo=float(np.sum(tl - xd[x < tl])), P_hi=float(np.sum(xd[x > th] - th)),
                       I_in=float(np.sum(xd[inner] - tl)))
        return out

    def pass_(self, t, lo, hi, compact):
        x = self.cur
        t64, lo64, hi64 = np.float64(t), np.float64(lo), np.float64(hi)
        lt, gt = x < t64, x > t64
        mlo, mhi = lt & (x > lo64), gt & (x < hi64)
        xd = x.astype(np.float64)
        mine = {"c_lt": int(lt.sum()), "c_eq": int((x == t64).sum()), "c_lo": int(mlo.sum()),
                "c_hi": int(mhi.sum()), "L_lo": float(np.sum(t64 - xd[mlo])), "L_hi": float(np.sum(xd[mhi] - t64)),
                "P": 0.0, "N": 0.0,
                "pred": float(x[mlo].max()) if mlo.any() else -math.inf,
                "succ": float(x[mhi].min()) if mhi.any() else math.inf}
        if compact:
            self.kept = (x[mlo].copy(), x[mhi].copy())
        out = {k: 0 for k in mine}
        out["pred"], out["succ"] = -math.inf, math.inf
        for r in self._gather(mine):
            for k in ("c_lt", "c_eq", "c_lo", "c_hi", "L_lo", "L_hi"):
                out[k] += r[k]
            out["pred"] = max(out["pred"], r["pred"])
            out["succ"] = min(out["succ"], r["succ"])
        return out

    def adopt(self, side):
        self.cur = self.kept[side]

    def cut(self, r):
        """R26 cut pass over the current array (exactly the bracket interior): 1024 evenly strided
        samples, cuts at sample ranks q -/+ (3.5 sd + 2) around local rank r (or, with
        cut_shift, deliberately off target to drive the far-side branches), the sample estimate of
        the target, #x<=t_a and the copy of ]t_a, t_b[."""
        x = self.cur
        if self.comm is not None:  # R28: pooled across ranks (the current arrays' sizes as weights)
            import paper_1104_2732_b200 as cp
            sizes = self._gather(x.size)
            keys = np.stack(self._gather(sample_keys(x)))
            ta, tb, te = cp.pooled_cuts(keys, sizes, r, "f32" if x.dtype == np.float32 else "f64")
            inner = (x > ta) & (x < tb)
            self.kept = (x[inner].copy(), None)
            both = self._gather((int((x <= ta).sum()), int(inner.sum())))
            return {"t_a": ta, "t_b": tb, "t_est": te, "le_a": sum(a for a, _ in both),
                    "inner": sum(b for _, b in both)}
        m = x.size
        ms = min(m, 1024)
        pos = np.arange(ms) if m == ms else (np.arange(ms, dtype=np.int64) * m) // ms + (m // ms) // 2
        smp = np.sort(x[pos])
        q = (r - 0.5) / m * ms + self.cut_shift * ms
        w = 3.5 * math.sqrt(max(q * (ms - q) / ms, 0.0)) + 2.0
        il = min(max(int(math.floor(q - w)), 0), ms - 1)
        ih = min(max(int(math.ceil(q + w)), il), ms - 1)
        ta, tb = smp[il], smp[ih]
        te = smp[min(max(int(math.floor(q)), 0), ms - 1)]
        inner = (x > ta) & (x < tb)
        self.kept = (x[inner].copy(), None)
        return {"t_a": float(ta), "t_b": float(tb), "t_est": float(te), "le_a": int((x <= ta).sum()),
                "inner": int(inner.sum())}

    def select(self, side, r):
        part = self.cur if side == 2 else self.kept[side]
        allz = np.concatenate(self._gather(part))
        return float(np.partition(allz, r - 1)[r - 1])


def drive(x, k, dtype, comm=None, config=None, cut=False, pass_cuts=False, cut_shift=0.0):
    import paper_1104_2732_b200 as cp
    be = NumpyShard(x, comm, cut_k=k if cut else None, cut_shift=cut_shift)
    n = x.size if comm is None else sum(comm(x.size))
    return cp.drive_host(n, k, dtype, be.init, be.pass_, be.adopt, be.select, config,
                         cut_fn=be.cut if pass_cuts else None)
