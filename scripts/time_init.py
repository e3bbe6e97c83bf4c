"""Time one selection's parts with CUDA events (record_timing) and the host overhead around them:
python scripts/time_init.py [dist] [log2n] — mean kernel ms (init / passes / select), the driver's
own wall time (info.ms_total) and the Python call's wall time."""
import sys
import time

import torch

sys.path.insert(0, ".")
import datagen  # noqa: E402
import paper_1104_2732_b200 as cp  # noqa: E402

dist = sys.argv[1] if len(sys.argv) > 1 else "uniform"
lg = int(sys.argv[2]) if len(sys.argv) > 2 else 30
sharded = len(sys.argv) > 3 and sys.argv[3] == "sharded"  # the NCCL path at world size 1
dtype = "f64" if "f64" in sys.argv else "f32"
x = datagen.make(dist, 1 << lg, dtype, device="cuda")
torch.cuda.synchronize()
import os
cp.set_config(record_timing=1, select_cap=int(os.environ.get("SELECT_CAP", "0")))
if sharded:
    cp.comm_init(cp.nccl_unique_id(), 0, 1, torch.cuda.current_device())


def run():
    if sharded:
        return cp.select_kth_sharded(x, (x.numel() + 1) // 2, return_info=True)
    return cp.median(x, return_info=True)


for _ in range(3):
    run()
ini, pas, sel, tot, wall, passes, smp = [], [], [], [], [], [], []
for _ in range(20):
    t0 = time.perf_counter()
    v, info = run()
    wall.append(1e3 * (time.perf_counter() - t0))
    ini.append(info["kernel_ms_init"]); pas.append(info["kernel_ms_passes"]); sel.append(info["kernel_ms_select"])
    tot.append(info["ms_total"]); passes.append(info["passes"]); smp.append(info["kernel_ms_sample"])
m = lambda a: sum(a) / len(a)  # noqa: E731
k = m(ini) + m(pas) + m(sel) + m(smp)
print(f"{dist} 2^{lg} {dtype}{' sharded' if sharded else ''}: init {m(ini):.4f}  passes {m(pas):.4f}  select {m(sel):.4f}  "
      f"sample {m(smp):.4f}  kernels {k:.4f}  "
      f"driver wall {m(tot):.4f}  python wall {m(wall):.4f} ms  passes/call {m(passes):.1f}")
if "--trace" in sys.argv:
    for r in cp.get_trace(torch.cuda.current_device()):
        print(f"  kind {r['kind']} scanned {r['scanned']:>11} written {r['written']:>10} interior {r['interior']:>11} "
              f"compacted {r['compacted']} kernel_ms {r['kernel_ms']:.4f}")
