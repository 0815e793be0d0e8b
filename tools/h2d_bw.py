"""Pinned host->device copy bandwidth (one and two concurrent streams)."""
import torch

n = 418 * 2**20 // 8
h = [torch.empty(n, dtype=torch.int64, pin_memory=True) for _ in range(2)]
d = [torch.empty(n, dtype=torch.int64, device="cuda") for _ in range(2)]
st = [torch.cuda.Stream() for _ in range(2)]
for ns in (1, 2):
    for rep in range(3):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for s in range(ns):
            st[s].wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st[s]):
                for _ in range(4):
                    d[s].copy_(h[s], non_blocking=True)
        for s in range(ns):
            torch.cuda.current_stream().wait_stream(st[s])
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        print(f"streams {ns}: {ns * 4 * n * 8 / ms / 1e6:.1f} GB/s")
