"""Achievable HBM read bandwidth for a pure streaming read of 4 GiB (torch.sum / torch.amax over
2^30 float32), CUDA events, best of 10 — what a one-read-of-x pass can hope for."""
import torch
x = torch.rand(1 << 30, device="cuda")
for name, fn in (("sum", torch.sum), ("amax", torch.amax)):
    for _ in range(3):
        fn(x)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(x); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name}: {best:.4f} ms, {4 * 2**30 / best / 1e6:.0f} GB/s")
