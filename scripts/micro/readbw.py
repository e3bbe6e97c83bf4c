"""Read-bandwidth ceiling of the init pass's access pattern (micro-benchmark, not product code):
python scripts/micro/readbw.py — builds readbw.cu with nvcc, reads 4 GiB of float32 per launch."""
import ctypes
import os
import subprocess
import sys

import torch

d = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(d, "readbw.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                       os.path.join(d, "readbw.cu"), "-o", so])
lib = ctypes.CDLL(so)
n = 1 << 30
x = torch.rand(n, device="cuda")
out = torch.zeros(1, device="cuda")
for grid, u, pd in ((592, 4, 0), (592, 4, 1), (592, 4, 2), (592, 4, 4), (592, 8, 0), (1184, 4, 0), (1184, 4, 1)):
    ms = ctypes.c_float()
    r = lib.run_read(ctypes.c_void_p(x.data_ptr()), ctypes.c_uint64(n), ctypes.c_void_p(out.data_ptr()), grid, u, pd,
                     ctypes.byref(ms), 10)
    print(f"grid {grid} U {u} L2-prefetch distance {pd}: {ms.value * 1e3:.1f} us, {4 * n / ms.value / 1e6:.0f} GB/s (err {r})")
