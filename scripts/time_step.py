"""The bench step (4 medians of 2^30 float32) timed with CUDA events, with and without the per-kernel
event timing (record_timing) — how much the timing itself costs.  python scripts/time_step.py"""
import sys

import torch

sys.path.insert(0, ".")
import datagen  # noqa: E402
import paper_1104_2732_b200 as cp  # noqa: E402

xs = [datagen.make(d, 1 << 30, "f32", device="cuda") for d in datagen.BENCH_DISTS]
torch.cuda.synchronize()
for rt in (0, 1, 0, 1):
    cp.set_config(record_timing=rt)
    for _ in range(3):
        for x in xs:
            cp.select_kth(x, (x.numel() + 1) // 2, return_info="raw")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        for x in xs:
            cp.select_kth(x, (x.numel() + 1) // 2, return_info="raw")
    e1.record()
    torch.cuda.synchronize()
    print(f"record_timing={rt}: {e0.elapsed_time(e1) / 10:.4f} ms per step of 4 medians")
