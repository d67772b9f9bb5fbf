"""H2D bandwidth probe (development aid): 64 x 20.4 MB pinned -> device copies on 1, 2 or 4 streams."""
import torch

n, sz = 64, 1600 * 1064 * 3
host = [torch.rand(sz).pin_memory() for _ in range(8)]
dev = [torch.empty(sz, device="cuda") for _ in range(8)]
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in streams:
            s.wait_stream(torch.cuda.current_stream())
        for i in range(n):
            with torch.cuda.stream(streams[i % ns]):
                dev[i % 8].copy_(host[i % 8], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    print(f"streams={ns}: {n * sz * 4 / 1e9:.2f} GB in {ms:.2f} ms = {n * sz * 4 / ms / 1e6:.1f} GB/s")
