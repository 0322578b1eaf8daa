"""Pinned host -> device copy bandwidth: one stream vs split across 2/4 streams."""
import torch

n = 1 << 27  # 1 GiB of fp64
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cur = torch.cuda.current_stream()
        chunk = n // ns
        for i, st in enumerate(streams):
            st.wait_stream(cur)
            with torch.cuda.stream(st):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        for st in streams:
            cur.wait_stream(st)
        e1.record()
        torch.cuda.synchronize()
    print(f"{ns} stream(s): {n * 8 / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s", flush=True)
