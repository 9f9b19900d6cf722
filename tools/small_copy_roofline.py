"""Practical HBM roofline for a small (config-1 sized) working set: time torch copy / sum kernels over
4 x 10M f32 tensors (160 MB) with L2 flushed before every launch, next to the fusion step kernels."""
import torch

dev = torch.device("cuda", 0)
n = 9966592
xs = [torch.randn(n, device=dev) for _ in range(4)]
out = torch.empty(n, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def t(fn, reps=20):
    ms = []
    for _ in range(3):
        flush.zero_(); fn()
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    ms.sort()
    return ms[len(ms) // 2] * 1e3


big = torch.empty(4 * n, device=dev)
big2 = torch.empty(4 * n, device=dev)
for name, fn, nbytes in [
    ("copy 160 MB -> 160 MB (one launch)", lambda: big2.copy_(big), 2 * 16 * n),
    ("sum of 4 tensors (reads 160 MB, writes 40 MB)", lambda: torch.add(torch.add(xs[0], xs[1]), torch.add(xs[2], xs[3]), out=out), 0),
    ("4 x copy_ 40 MB", lambda: [out.copy_(x) for x in xs], 8 * 4 * n),
    ("read 160 MB (big.sum)", lambda: big.sum(), 16 * n),
]:
    us = t(fn)
    print(f"{name:55s} {us:8.1f} us" + (f"  {nbytes / us / 1e3:7.0f} GB/s" if nbytes else ""))
