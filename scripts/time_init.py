"""Time the init pass (and the rest of one selection) of a 2^30 f32 median with CUDA events:
python scripts/time_init.py [dist] — prints mean kernel ms per selection part."""
import sys

import torch

sys.path.insert(0, ".")
import datagen  # noqa: E402
import paper_1104_2732_b200 as cp  # noqa: E402

dist = sys.argv[1] if len(sys.argv) > 1 else "uniform"
x = datagen.make(dist, 1 << 30, "f32", device="cuda")
torch.cuda.synchronize()
cp.set_config(record_timing=1)
for _ in range(3):
    cp.median(x)
ini, pas, sel = [], [], []
for _ in range(10):
    v, info = cp.median(x, return_info=True)
    ini.append(info["kernel_ms_init"]); pas.append(info["kernel_ms_passes"]); sel.append(info["kernel_ms_select"])
print(f"{dist}: init {sum(ini)/len(ini):.4f} ms  passes {sum(pas)/len(pas):.4f} ms  select {sum(sel)/len(sel):.4f} ms")
