"""PCIe copy bandwidth from pinned memory: 1 vs 2 H2D streams, with and without concurrent D2H."""
import torch

dev = torch.device("cuda", 0)
N = 8 << 30
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
ho = torch.empty(N // 4, dtype=torch.uint8, pin_memory=True)
d = torch.empty(N, dtype=torch.uint8, device=dev)
do = torch.empty(N // 4, dtype=torch.uint8, device=dev)
ss = [torch.cuda.Stream(dev) for _ in range(4)]


def run(n_h2d, chunk_mb, with_d2h):
    ch = chunk_mb << 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for s in ss:
        s.wait_event(e0)
    k = 0
    for off in range(0, N, ch):
        with torch.cuda.stream(ss[k % n_h2d]):
            d[off:off + ch].copy_(h[off:off + ch], non_blocking=True)
        k += 1
    if with_d2h:
        with torch.cuda.stream(ss[3]):
            for off in range(0, N // 4, ch):
                ho[off:off + ch].copy_(do[off:off + ch], non_blocking=True)
    for s in ss:
        e1.wait_stream(s) if hasattr(e1, "wait_stream") else None
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return N / ms / 1e6


for with_d2h in (False, True):
    for n in (1, 2, 3):
        for chunk in (64, 512):
            bw = [run(n, chunk, with_d2h) for _ in range(3)]
            print(f"h2d streams {n} chunk {chunk} MB d2h {with_d2h}: H2D {max(bw):.1f} GB/s")
