#!/usr/bin/env python
"""Benchmark: exact k-th order statistic by the cutting-plane path (BASELINE.json metric:
"elements/s and HBM-roofline fraction for k-th select at n=2^30, 1/2/4/8 B200").

N = 1 (the headline, BASELINE's metric configuration): one step = one median selection over each
of four resident synthetic arrays of 2^30 float32 (uniform, normal, Cauchy, many-duplicate;
configs[1]'s distributions at the metric size) = 4 x 2^30 elements.  The default path: the init
pass evaluates two cuts at sample quantiles of the target rank (R23/R29) and the exact radix
select finishes on the ~1% between them; Kelley passes run only when the cuts miss.  Side blocks
(rank 0, N = 1): "kelley" — the paper's method as published (Kelley passes from [x_(1), x_(n)],
init_cut=0 pass_cuts=0 objective=1) at the same size with its per-pass rooflines;
"configs" — BASELINE configs[0] (1e5), [1] (2^24 x 4 dists x 4 ranks), [2] (2^28 float64),
[3] (2^32 float32 on one GPU: the scaling base) and [4] (LMS); "cpu_baseline" — the oracle on the
host cores (np.partition, C++ nth_element / sort, the literal double-precision cutting plane).

N > 1 (torchrun, one process per GPU): configs[3] — the median of ONE global array of 2^32 float32
(uniform and normal, the shard-invariant generator: identical data for every N) sharded in
contiguous blocks over the N GPUs (strong scaling), one sharded selection per array per step: per
pass one NCCL all-gather of the 96-byte tuple, an all-gather-v of the bracket at the end.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Prints ONE JSON line (rank 0).  Timing: CUDA events on the launching stream bracketed by a barrier
and torch.cuda.synchronize(), max over ranks; inputs are larger than L2 (4 GiB per array; the
configs[0]/[1] side blocks flush L2 between calls).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "elements/s and HBM-roofline fraction for k-th select at n=2^30, 1/2/4/8 B200"
UNIT = "elements/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cpsel", choices=["cpsel", "reference"])
    ap.add_argument("--log2n", type=int, default=30)
    ap.add_argument("--dists", default="uniform,normal,cauchy,dup256")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=24.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--z-cap", type=int, default=0)
    ap.add_argument("--no-lms", action="store_true", help="skip the configs[4] LMS side measurement")
    ap.add_argument("--no-side", action="store_true", help="skip the kelley / configs side blocks")
    ap.add_argument("--global-log2n", type=int, default=32, help="N>1: log2 of the global array (configs[3])")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        time.sleep(0.25)

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [s.strip() for s in line.split(",")]
                if len(parts) >= 8:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------------------ reference arm
def run_reference(a, rank: int, world: int):
    """--impl reference: the oracle (sort-based selection, numpy partition) timed as it stands on the
    host cores, each step a bounded sample (2^24 elements of each distribution) of the workload."""
    if rank != 0:
        return
    import numpy as np

    import datagen
    import oracle
    dists = a.dists.split(",")
    m = 1 << 24
    xs = [datagen.make(d, m, "f32") for d in dists]
    k = oracle.median_rank(m)
    for _ in range(a.warmup):
        for x in xs:
            oracle.order_statistic(x, k)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        for x in xs:
            oracle.order_statistic(x, k)
    dt = time.perf_counter() - t0
    value = a.steps * len(xs) * m / dt
    sample = f"oracle.order_statistic (np.partition, 1 thread) median of 2^24-element samples of {dists} per step"
    n = 1 << a.log2n
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1e3 * dt / a.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"median of n=2^{a.log2n} float32 x {dists}", "n": n, "k": "median (n+1)//2"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ------------------------------------------------------------------------------ configs[4]
def lms_side(cp, torch, datagen, dev, reps=5):
    """LMS objective (n=1e6, p=10, C=4096): median of squared residuals per candidate on the fused
    path (residuals recomputed in the tcgen05 epilogue, no S in HBM), CUDA events over `reps` calls
    after 2 warm-up calls.  The fused pass is issue-bound: its roofline is the SM issue rate
    (148 SMs x 4 schedulers x 1 warp-instruction/clk x sm clock) over the 6 thread-instructions per
    residual of its element step."""
    n, p, C = 1_000_000, 10, 4096
    X, y, th, _ = datagen.lms_problem(n=n, p=p, C=C)
    Xd, yd, thd = (torch.from_numpy(v).to(dev) for v in (X, y, th))
    for _ in range(2):
        cp.lms_objective(Xd, yd, thd)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out, info = cp.lms_objective(Xd, yd, thd, return_info=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fused_ms = info["kernel_ms_init"]          # sample cuts + the fused tensor-core pass
    sm_mhz = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("sm_max_mhz", 1965.0) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1965.0
    peak_el = 148 * 4 * sm_mhz * 1e6 * 32 / 5.5  # residual-steps/s at full issue, 5.5 instr each
    return {"workload": "LMS objective n=1e6 p=10 C=4096 (BASELINE configs[4]), fused path",
            "ms": ms, "candidates_per_s": C / (ms / 1e3), "residuals_per_s": n * C / (ms / 1e3),
            "fused_stage_ms": fused_ms, "continuation_ms": info["kernel_ms_passes"],
            "fallback_columns": info["fallback_steps"], "passes_per_column": info["passes"] / C,
            "roofline_fused_stage": {"bound": "alu", "unit": "residuals/s", "achieved": n * C / (fused_ms / 1e3),
                                     "peak": peak_el, "frac": n * C / (fused_ms / 1e3) / peak_el,
                                     "peak_note": "issue rate 148x4x1 warp-instr/clk at sm_max_mhz, "
                                                  "5.5 thread-instructions per residual (one FMUL2 per two "
                                                  "residuals — y is folded into the tensor-core product, "
                                                  "R39 — + the 5-instruction cut step); the stage also "
                                                  "includes the sample-cut kernels"}}


# ------------------------------------------------------------------------------ side blocks (N=1)
def _ev(torch):
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def trace_classes(rows, n, es, peak):
    """per-pass roofline classes of a traced selection: algorithmic bytes = es x (elements read +
    elements written) per launch, over that launch's CUDA-event time"""
    cls = {}
    for r in rows:
        if r["kind"] == 2:          # the init's cut rows (evaluated inside the init pass)
            continue
        key = ("full_pass" if r["scanned"] == n else "bracket_pass") + ("_compacting" if r["compacted"] else "_hot")
        c = cls.setdefault(key, {"launches": 0, "bytes": 0, "ms": 0.0})
        c["launches"] += 1
        c["bytes"] += es * (r["scanned"] + r["written"])
        c["ms"] += r["kernel_ms"]
    for c in cls.values():
        c["GBps"] = c["bytes"] / (c["ms"] / 1e3) / 1e9 if c["ms"] > 0 else None
        c["frac"] = c["GBps"] / peak if c["GBps"] else None
    return cls


def kelley_side(cp, torch, datagen, dev, dists, log2n, peak, reps=3):
    """The paper's method as published (Algorithm 1 from the bracket [x_(1), x_(n)], one cut per
    pass, the interior-mean iterate = step 1.1 with the tightest cuts (App. A), F_k at every iterate,
    P:L155-198): init_cut=0, pass_cuts=0, objective=1.  Per distribution: ms per selection (CUDA
    events over `reps` calls), passes (the paper: 7 iterations at 2^25), the F trace, and
    the per-pass roofline of the traced call."""
    n = 1 << log2n
    k = (n + 1) // 2
    out = {"workload": f"median of n=2^{log2n} float32, Kelley passes from [x_(1), x_(n)] "
                       f"(init_cut=0, pass_cuts=0, objective=1)", "per_dist": {}}
    cfg = dict(init_cut=0, pass_cuts=0, objective=1)
    tot_ms, tot_bytes, all_rows = 0.0, 0, []
    for d in dists:
        x = datagen.make(d, n, "f32", device=dev)
        cp.set_config(dev.index, record_timing=0, **cfg)
        for _ in range(2):
            cp.select_kth(x, k)
        e0, e1 = _ev(torch)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            v, info = cp.select_kth(x, k, return_info=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        cp.set_config(dev.index, record_timing=1, **cfg)
        v2, info2 = cp.select_kth(x, k, return_info=True)
        rows = cp.get_trace(dev.index)
        all_rows += rows
        tot_ms += ms
        tot_bytes += info["bytes_moved"]
        out["per_dist"][d] = {
            "ms": ms, "elements_per_s": n / (ms / 1e3), "passes": info["passes"], "cp_iters": info["cp_iters"],
            "exit": info["exit"], "same_value_traced": v == v2,
            "F_trace": [r["F"] for r in rows], "interior_trace": [r["interior"] for r in rows],
            "whole_call_frac": info["bytes_moved"] / (ms / 1e3) / 1e9 / peak,
            "kernel_ms": {"init": info2["kernel_ms_init"], "passes": info2["kernel_ms_passes"],
                          "select": info2["kernel_ms_select"]},
            "classes": trace_classes(rows, n, 4, peak)}
        del x
    # the paper's outlier claim (P:L413-414 vs P:L416, Fig. 4): 100 values of 1e3 / 1e9 among uniform
    # data, the cutting plane against the comparison drivers: bisection (driver=1), Brent's
    # root finder (2) and Brent's minimisation (3)
    import datagen as dg
    x = dg.make("uniform", n, "f32", device=dev)
    pos = torch.randperm(n, generator=torch.Generator().manual_seed(dg.SEED))[:100].to(dev)
    out["outliers"] = {}
    for mag in (1e3, 1e9):
        x[pos] = mag
        for name, drv in (("kelley", 0), ("bisection", 1), ("brent_root", 2), ("brent_min", 3)):
            cp.set_config(dev.index, record_timing=0, driver=drv, **cfg)
            cp.select_kth(x, k)
            e0, e1 = _ev(torch)
            e0.record()
            v, info = cp.select_kth(x, k, return_info=True)
            e1.record()
            torch.cuda.synchronize()
            out["outliers"][f"{name}/{mag:g}"] = {"passes": info["passes"], "ms": e0.elapsed_time(e1)}
    del x
    cp.set_config(dev.index, record_timing=0, init_cut=1, pass_cuts=1, objective=0, driver=0)
    torch.cuda.empty_cache()
    out["elements_per_s"] = len(dists) * n / (tot_ms / 1e3)
    out["ms_per_selection"] = tot_ms / len(dists)
    out["whole_call_frac"] = tot_bytes / (tot_ms / 1e3) / 1e9 / peak
    out["classes"] = trace_classes(all_rows, n, 4, peak)
    out["paper_reference"] = "P:L198: 7 iterations at n=2^25 leave < 2^19 elements (then copy_if + sort)"
    return out


def knn_side(cp, torch, dev, peak, reps=3):
    """kNN regression via d_(k) (§8f-4): n=1e6 reference points in p=10, nq=1024
    queries, k=32 — distances (float32, written once), the batched k-th select per query and the
    rho/a,b reduction.  Bound: HBM (the nq x n distance matrix: written, then read by the select's
    passes and the reduction)."""
    import numpy as np
    n, p, nq, k = 1_000_000, 10, 1024, 32
    rng = np.random.default_rng(11042732)
    X = rng.standard_normal((n, p)).astype(np.float32)
    f = (np.sin(X[:, 0]) + 0.1 * rng.standard_normal(n)).astype(np.float32)
    Q = rng.standard_normal((nq, p)).astype(np.float32)
    Xd, fd, Qd = (torch.from_numpy(v).to(dev) for v in (X, f, Q))
    cp.knn_regress(Xd, fd, Qd, k)
    torch.cuda.synchronize()
    e0, e1 = _ev(torch)
    e0.record()
    for _ in range(reps):
        out, info = cp.knn_regress(Xd, fd, Qd, k, return_info=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return {"workload": "kNN regression n=1e6 p=10 nq=1024 k=32 (uniform weights)", "ms": ms,
            "queries_per_s": nq / (ms / 1e3), "distances_per_s": n * nq / (ms / 1e3),
            "bytes_moved": info["bytes_moved"], "GBps": info["bytes_moved"] / (ms / 1e3) / 1e9,
            "frac": info["bytes_moved"] / (ms / 1e3) / 1e9 / peak, "select_passes_per_query": info["passes"] / nq}


def _flush_l2(torch, buf):
    buf.add_(1.0)  # 256 MiB > 126 MB L2


def configs_side(cp, torch, datagen, dev, peak, reps=5):
    """BASELINE configs[0..3] at their stated sizes on one GPU (the metric config is the headline;
    configs[4] is the "lms" block).  Each call is timed alone with CUDA events after an L2 flush."""
    import numpy as np
    out = {}
    flush = torch.empty(1 << 26, device=dev, dtype=torch.float32)

    def timed(x, k, reps_=reps):
        cp.select_kth(x, k)
        ts = []
        for _ in range(reps_):
            _flush_l2(torch, flush)
            e0, e1 = _ev(torch)
            e0.record()
            v, info = cp.select_kth(x, k, return_info=True)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return v, info, statistics.median(ts)

    # configs[0]: median of 1e5 float32 uniform (the one-launch cluster select)
    x = datagen.make("uniform", 100_000, "f32", device=dev)
    v, info, ms = timed(x, 50_000, 50)
    out["configs0"] = {"workload": "median of n=1e5 float32 uniform", "us_per_call": ms * 1e3,
                       "elements_per_s": 1e5 / (ms / 1e3), "launches": info["launches"], "exit": info["exit"],
                       "bound": "latency (one 8-CTA cluster launch, L2-resident)"}
    # configs[1]: 2^24 float32 x 4 dists x k in {1, n/10, median, n-1}
    n = 1 << 24
    cells, tot_ms = {}, 0.0
    for d in ("uniform", "normal", "cauchy", "dup256"):
        x = datagen.make(d, n, "f32", device=dev)
        for kk, name in ((1, "1"), (n // 10, "n/10"), ((n + 1) // 2, "median"), (n - 1, "n-1")):
            v, info, ms = timed(x, kk)
            cells[f"{d}/{name}"] = {"ms": ms, "passes": info["passes"], "exit": info["exit"]}
            tot_ms += ms
    out["configs1"] = {"workload": "k in {1, n/10, median, n-1} of n=2^24 float32 x {uniform, normal, cauchy, dup256}",
                       "elements_per_s": 16 * n / (tot_ms / 1e3), "ms_per_selection": tot_ms / 16,
                       "roofline_frac_one_read": (n * 4) / (tot_ms / 16 / 1e3) / 1e9 / peak,
                       "note": "64 MiB input: L2 flushed before each call; latency-dominated (~4 launches)",
                       "cells": cells}
    del x
    # configs[2]: 2^28 float64, k in {median, 1, n/10, n-1}
    n = 1 << 28
    per, tot_ms, tot_b = {}, 0.0, 0
    for d in ("uniform", "normal"):
        x = datagen.make(d, n, "f64", device=dev)
        for kk, name in (((n + 1) // 2, "median"), (1, "1"), (n // 10, "n/10"), (n - 1, "n-1")):
            v, info, ms = timed(x, kk)
            per[f"{d}/{name}"] = {"ms": ms, "passes": info["passes"], "exit": info["exit"]}
            tot_ms += ms
            tot_b += info["bytes_moved"]
        del x
    out["configs2"] = {"workload": "k in {median, 1, n/10, n-1} of n=2^28 float64 x {uniform, normal}",
                       "elements_per_s": 8 * n / (tot_ms / 1e3), "ms_per_selection": tot_ms / 8,
                       "whole_call_frac": tot_b / (tot_ms / 1e3) / 1e9 / peak, "cells": per}
    torch.cuda.empty_cache()
    # configs[3] at G = 1: the median of 2^32 float32 on one B200 (the scaling base of the sharded runs)
    n = 1 << 32
    per, tot_ms, tot_b = {}, 0.0, 0
    for d in datagen.GLOBAL_DISTS:
        x = datagen.make_global(d, n, 0, n, "f32", device=dev)
        v, info, ms = timed(x, (n + 1) // 2, 3)
        per[d] = {"ms": ms, "passes": info["passes"], "exit": info["exit"], "value": v}
        tot_ms += ms
        tot_b += info["bytes_moved"]
        del x
        torch.cuda.empty_cache()
    out["configs3_g1"] = {"workload": "median of n=2^32 float32 (uniform, normal; shard-invariant generator) on ONE B200",
                          "elements_per_s": 2 * n / (tot_ms / 1e3), "ms_per_selection": tot_ms / 2,
                          "whole_call_frac": tot_b / (tot_ms / 1e3) / 1e9 / peak, "cells": per}
    del flush
    torch.cuda.empty_cache()
    return out


def cpu_side(xs_host, dists, seconds):
    """The oracle as it stands on the host cores (rank 0, N = 1), on bounded samples of the workload:
    np.partition (oracle.order_statistic), C++ std::nth_element and std::sort (oracle.order_statistic_c,
    single thread; the paper's CPU quickselect row) on 2^24-element prefixes, and the
    literal double-precision cutting plane (oracle.cutting_plane, Algorithm 1) on 2^22-element prefixes."""
    import platform

    import oracle
    model = platform.processor() or "?"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    rows = {}

    def run(name, fn, samples, budget):
        done, t0 = 0, time.perf_counter()
        while True:
            for smp in samples:
                fn(smp)
                done += smp.size
            if time.perf_counter() - t0 > budget:
                break
        dt = time.perf_counter() - t0
        rows[name] = {"value": done / dt, "unit": UNIT, "cores": 1, "elements": done, "seconds": dt}

    s24 = [x[:1 << 24] for x in xs_host]
    k24 = oracle.median_rank(1 << 24)
    run("np.partition", lambda z: oracle.order_statistic(z, k24), s24, seconds / 4)
    run("nth_element", lambda z: oracle.order_statistic_c(z, k24, "nth_element"), s24, seconds / 4)
    run("sort", lambda z: oracle.order_statistic_c(z, k24, "sort"), s24[:1], seconds / 4)
    s22 = [x[:1 << 22] for x in xs_host]
    k22 = oracle.median_rank(1 << 22)
    run("cutting_plane", lambda z: oracle.cutting_plane(z, k22, z_cap=1 << 16), s22[:2], seconds / 4)
    best_name = max(rows, key=lambda r: rows[r]["value"])
    return {"value": rows[best_name]["value"], "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"the fastest oracle row ({best_name}, 1 thread) on medians of the first 2^24 elements "
                      f"of {dists}; rows: np.partition (oracle.order_statistic), C++ std::nth_element and "
                      f"std::sort (oracle.order_statistic_c, 2^24), the literal long-double cutting plane "
                      f"(oracle.cutting_plane, 2^22)",
            "cpu_model": model, "nproc": os.cpu_count(), "rows": rows}


# ------------------------------------------------------------------------------ our arm
def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        return run_reference(a, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist

    import datagen
    import paper_1104_2732_b200 as cp

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cp.load()
    if world == 1:
        # the metric configuration: 2^30 float32 per array, the four distributions of configs[1]
        dists = a.dists.split(",")
        n = 1 << a.log2n
        xs = [datagen.make(d, n, "f32", device=dev) for d in dists]
        n_global = n
    else:
        # configs[3]: ONE global array of 2^32 float32 per distribution, rank r holding the contiguous
        # block [r*N/G, (r+1)*N/G) drawn by the shard-invariant generator (same data for every G)
        dists = list(datagen.GLOBAL_DISTS)
        n_global = 1 << a.global_log2n
        lo, hi = n_global * rank // world, n_global * (rank + 1) // world
        xs = [datagen.make_global(d, n_global, lo, hi, "f32", device=dev) for d in dists]
        n = hi - lo
    torch.cuda.synchronize()
    k = (n_global + 1) // 2
    cp.set_config(local, z_cap=a.z_cap)
    if world > 1:
        obj = [cp.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        cp.comm_init(obj[0], rank, world, local)

    def select(x):
        if world > 1:
            return cp.select_kth_sharded(x, k, return_info=True)
        v, raw = cp.select_kth(x, k, return_info="raw")  # the report's dict is built after timing
        return v, raw

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    for _ in range(a.warmup):
        for x in xs:
            select(x)
    # light timing in the timed region: only each selection's init kernel (the dominant kernel) is
    # bracketed by CUDA events, resolved after the loop; the per-kernel timing of every step
    # (record_timing=1) reads events back inside each call and would slow the step it measures
    cp.set_config(local, z_cap=a.z_cap, record_timing=2)
    cp.init_timings(local)  # empty the ring
    stream = torch.cuda.current_stream(dev)
    clocks = Clocks(local)
    infos = []
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.steps):
        for x in xs:
            infos.append(select(x)[1])
    e1.record(stream)
    infos = [i if isinstance(i, dict) else i.as_dict() for i in infos]
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / a.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = len(xs) * n_global / (ms / 1e3)
    init_ring = cp.init_timings(local)  # the timed region's init-kernel durations
    # per-pass trace rows (bytes and CUDA-event time of every kernel) from one more step after the
    # timed region with full timing; the dominant kernel's numbers come from the timed region itself
    cp.set_config(local, z_cap=a.z_cap, record_timing=1)
    traces, tinfos = [], []
    for x in xs:
        r = select(x)[1]
        tinfos.append(r if isinstance(r, dict) else r.as_dict())
        traces.append(cp.get_trace(local))

    # Dominant kernel: the class with the largest share of kernel time in the timed region (the init
    # pass).  Algorithmic bytes of one launch = 4 x (elements read + elements written); achieved =
    # sum of those bytes / sum of the CUDA-event durations of the launches.
    rows = [r for tr in traces for r in tr]
    init_ms = init_ring if len(init_ring) == len(infos) else [i["kernel_ms_init"] for i in tinfos] * a.steps
    sel_ms = [i["kernel_ms_select"] for i in tinfos]
    iters = [i["cp_iters"] for i in infos]
    peak, peak_src = peaks()

    def cls(sel):
        rr = [r for r in rows if sel(r)]
        by = sum(4 * (r["scanned"] + r["written"]) for r in rr)
        ms = sum(r["kernel_ms"] for r in rr)
        return {"launches": len(rr), "bytes": by, "ms": ms,
                "GBps": (by / (ms / 1e3) / 1e9) if ms > 0 else None}

    all_pass = cls(lambda r: r["kind"] != 2)
    hot_x = cls(lambda r: r["kind"] != 2 and not r["compacted"] and r["scanned"] == n)
    comp_x = cls(lambda r: r["kind"] != 2 and r["compacted"] and r["scanned"] == n)
    z_pass = cls(lambda r: r["kind"] != 2 and r["scanned"] < n)
    # the init pass (init_seg_kernel alone: the init reduction with the two cuts and the fused copy_if,
    # R23; its sample kernels are timed separately, R29)
    init_bytes = sum(4 * (n + i["init_written"]) for i in infos)
    init_ms_tot = sum(init_ms)
    init_cls = {"launches": len(infos), "bytes": init_bytes, "ms": init_ms_tot,
                "GBps": init_bytes / (init_ms_tot / 1e3) / 1e9 if init_ms_tot > 0 else None}
    init_GBps = init_cls["GBps"]
    # dominant kernel = the class with the largest share of kernel time in the timed region
    if init_ms_tot >= sum(i["kernel_ms_passes"] for i in infos):
        dom_name, dom = "init_seg_kernel<float> (a1 + the R23 cuts + fused a4 copy_if)", init_cls
    else:
        dom_name, dom = "seg_pass_kernel<float> / pass_kernel<float> (a2 + fused a4)", all_pass
    achieved = dom["GBps"]
    avg_pass_ms = dom["ms"] / max(dom["launches"], 1)
    bytes_per_pass = dom["bytes"] / max(dom["launches"], 1)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_pass_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        traffic = tj.get(dom_name.split("<")[0], {}).get("dram_bytes_per_launch")
    step_kernel_ms = sum(init_ms) / a.steps + sum(i["kernel_ms_passes"] + i["kernel_ms_select"] + i["kernel_ms_sample"]
                                                  for i in tinfos)
    launches = sum(i["launches"] for i in infos)
    # whole-call fraction: all algorithmic bytes of the timed selections (every pass's
    # reads + writes, the exact stage's reads of the copy) over the step time
    bytes_step = sum(i["bytes_moved"] for i in infos) / a.steps
    whole_call = {"bytes_per_step": bytes_step, "GBps": bytes_step / (ms / 1e3) / 1e9,
                  "frac": bytes_step / (ms / 1e3) / 1e9 / peak}
    cp.set_config(local, z_cap=a.z_cap, record_timing=0)

    # end to end through the C ABI with HOST buffers (H2D inside the timed region)
    e2e = None
    if not a.no_e2e and a.e2e_steps > 0:
        pinned = torch.empty(n, dtype=torch.float32, pin_memory=True)
        tot_s, tot_el, d2h = 0.0, 0, 0
        for s in range(a.e2e_steps):
            for x in xs:
                pinned.copy_(x)                         # untimed: stage this step's input on the host
                torch.cuda.synchronize()
                barrier()
                t0 = time.perf_counter()
                if world > 1:
                    xd = pinned.to(dev, non_blocking=True)
                    _, info = cp.select_kth_sharded(xd, k, return_info=True)
                    torch.cuda.synchronize()
                else:
                    _, info = cp.select_kth_host(pinned, k, device=local, return_info=True)
                dt = time.perf_counter() - t0
                if world > 1:
                    tt = torch.tensor([dt], device=dev)
                    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                    dt = float(tt.item())
                tot_s += dt
                tot_el += n_global
                d2h += 4 + 96 * info["passes"]
        del pinned
        e2e = {"value": tot_el / tot_s, "unit": UNIT, "h2d_bytes_per_step": len(xs) * n * 4,
               "d2h_bytes_per_step": d2h // a.e2e_steps,
               "note": "select_kth_host: pinned host array -> device staging copy inside the timed call"}

    # BASELINE configs[4] side measurement (rank 0, N=1): the LMS objective on the fused
    # tensor-core path — not the headline metric, reported under "lms"
    lms = None
    if rank == 0 and world == 1 and not a.no_lms:
        try:
            lms = lms_side(cp, torch, datagen, dev)
        except Exception as ex:  # the headline line must not depend on the side measurement
            lms = {"error": f"{type(ex).__name__}: {ex}"}

    # side blocks (rank 0, N=1): the paper's method as published, BASELINE configs[0..3]
    kelley = side = None
    if rank == 0 and world == 1 and not a.no_side:
        try:
            kelley = kelley_side(cp, torch, datagen, dev, dists, a.log2n, peak)
        except Exception as ex:
            kelley = {"error": f"{type(ex).__name__}: {ex}"}
        try:
            side = configs_side(cp, torch, datagen, dev, peak)
        except Exception as ex:
            side = {"error": f"{type(ex).__name__}: {ex}"}
        try:
            side["knn"] = knn_side(cp, torch, dev, peak)
        except Exception as ex:
            side["knn"] = {"error": f"{type(ex).__name__}: {ex}"}

    # CPU baseline: the oracle as it stands, on bounded host samples (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        cpu = cpu_side([x[:1 << 24].cpu().numpy() for x in xs], dists, a.cpu_seconds)

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak" if world == 1 else "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded; torch.Generator at N=1, the shard-invariant counter generator at N>1)",
            "config": {"workload": (f"median of n=2^{a.log2n} float32 x {dists} (4 selections per step; "
                                    f"path: sample-cut init pass + exact radix finish, Kelley passes if the "
                                    f"cuts miss)") if world == 1 else
                                   (f"configs[3]: median of ONE n=2^{a.global_log2n} float32 array per "
                                    f"distribution {dists}, contiguous shards of 2^{a.global_log2n}/{world} "
                                    f"per GPU ({len(dists)} sharded selections per step)"),
                       "n_per_gpu": n, "n_global": n_global, "k": "lower median (n+1)//2",
                       "parallelism": "single GPU" if world == 1 else f"sharded x{world} (NCCL tuple all-gather)",
                       "l2": "inputs larger than L2 (>= 2 GiB per array per GPU vs 126 MB L2); no flush needed",
                       "z_cap": a.z_cap or "auto"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": dom_name,
                         "bytes_per_launch": bytes_per_pass, "avg_launch_ms": avg_pass_ms,
                         "peak_source": peak_src,
                         "classes_note": "init_pass from the timed region; pass classes from one traced step after it",
                         "classes": {"init_pass": init_cls, "hot_full_pass": hot_x, "compacting_full_pass": comp_x,
                                     "bracket_passes": z_pass, "all_cp_passes": all_pass}},
            "whole_call_roofline": whole_call,
            "cp_iters": {"mean": statistics.fmean(iters), "min": min(iters), "max": max(iters)},
            "kernel_ms_per_step": {"init": sum(init_ms) / a.steps, "passes": sum(i["kernel_ms_passes"] for i in tinfos),
                                   "select": sum(sel_ms), "sample": sum(i["kernel_ms_sample"] for i in tinfos),
                                   "all": step_kernel_ms,
                                   "note": "init from the timed region (light timing); the others from one "
                                           "fully timed step after it"},
            "gpu_launches": launches,
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "kelley": kelley,
            "configs": side,
            "lms": lms,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
