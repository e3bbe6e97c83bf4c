"""Latency of small selections (BASELINE configs[0]: median of n=1e5 float32): the Python call's
wall time per median, CUDA-event kernel time, over 200 calls.  python scripts/time_small.py [n]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import datagen  # noqa: E402
import paper_1104_2732_b200 as cp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
x = datagen.make("uniform", n, "f32", device="cuda")
for _ in range(10):
    cp.median(x)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    cp.median(x)
wall = (time.perf_counter() - t0) / 200 * 1e3
cp.set_config(record_timing=1)
v, info = cp.median(x, return_info=True)
cp.set_config(record_timing=0)
print(f"n={n}: {wall * 1e3:.1f} us per median (python wall), kernel {info['kernel_ms_select'] * 1e3:.1f} us, "
      f"launches {info['launches']}, exit {info['exit']}, {n / (wall / 1e3):.3e} elements/s")
