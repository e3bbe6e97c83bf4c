"""The paper's method as a measured configuration: Kelley passes from [x_(1), x_(n)] (init_cut=0,
pass_cuts=0, objective=1 — P:L155-198), per-pass CUDA-event time and bytes from the trace.

python scripts/time_kelley.py [log2n] [dists] [--f64] [--zcap N] [--reps R] [--device-loop]
Prints one line per distribution (ms per selection, passes, achieved GB/s per pass class) and the
trace of the last call.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_1104_2732_b200 as cp  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
lg = int(args[0]) if args else 30
dists = (args[1] if len(args) > 1 else "uniform,normal,cauchy,dup256").split(",")
dtype = "f64" if "--f64" in sys.argv else "f32"
es = 8 if dtype == "f64" else 4
zcap = 0
reps = 5
for i, a in enumerate(sys.argv):
    if a == "--zcap":
        zcap = int(sys.argv[i + 1])
    if a == "--reps":
        reps = int(sys.argv[i + 1])
peak = 6549.8
if os.path.exists("MEASURED_PEAKS.json"):
    peak = float(json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"])
dev = torch.cuda.current_device()
n = 1 << lg
out = []
for d in dists:
    x = datagen.make(d, n, dtype, device="cuda")
    torch.cuda.synchronize()
    k = (n + 1) // 2
    cfg = dict(init_cut=0, pass_cuts=0, objective=1, z_cap=zcap,
               device_loop=1 if "--device-loop" in sys.argv else 0)
    cp.set_config(dev, record_timing=0, **cfg)
    for _ in range(2):
        cp.select_kth(x, k)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        v, info = cp.select_kth(x, k, return_info=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    cp.set_config(dev, record_timing=1, **cfg)
    v2, info2 = cp.select_kth(x, k, return_info=True)
    tr = cp.get_trace(dev)
    cls = {}
    for r in tr:
        key = ("full" if r["scanned"] == n else "bracket") + ("+compact" if r["compacted"] else "")
        c = cls.setdefault(key, {"launches": 0, "bytes": 0, "ms": 0.0})
        c["launches"] += 1
        c["bytes"] += es * (r["scanned"] + r["written"])
        c["ms"] += r["kernel_ms"]
    for c in cls.values():
        c["GBps"] = c["bytes"] / (c["ms"] / 1e3) / 1e9 if c["ms"] > 0 else None
        c["frac"] = c["GBps"] / peak if c["GBps"] else None
    line = {"dist": d, "n": n, "dtype": dtype, "ms": ms, "passes": info["passes"], "cp_iters": info["cp_iters"],
            "el_per_s": n / (ms / 1e3), "init_ms": info2["kernel_ms_init"], "passes_ms": info2["kernel_ms_passes"],
            "select_ms": info2["kernel_ms_select"], "driver_ms": info2["ms_total"], "classes": cls,
            "value_ok": v == v2, "exit": info["exit"]}
    out.append(line)
    print(json.dumps(line), flush=True)
    if "--trace" in sys.argv:
        for r in tr:
            print(f"  kind {r['kind']} t {r['t']:.9g} F {r['F']:.6g} scanned {r['scanned']:>11} written {r['written']:>10} "
                  f"interior {r['interior']:>11} compacted {r['compacted']} kernel_ms {r['kernel_ms']:.4f}", flush=True)
    del x
    torch.cuda.empty_cache()
cp.set_config(dev, record_timing=0, init_cut=1, pass_cuts=1, objective=0, z_cap=0, device_loop=0)
