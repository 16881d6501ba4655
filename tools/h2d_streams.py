"""Pinned host -> device bandwidth with 1, 2 or 4 copy streams (is one copy engine
the limit of the staged training pipeline?).  Usage: python tools/h2d_streams.py"""
import torch

n = 116 * 2 ** 20 // 4
srcs = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in range(8)]
dsts = [torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(8)]
for k in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    for _ in range(2):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for i in range(8):
            st = streams[i % k]
            st.wait_event(s)
            with torch.cuda.stream(st):
                dsts[i].copy_(srcs[i], non_blocking=True)
        for st in streams:
            e.wait_stream(st) if hasattr(e, "wait_stream") else None
            torch.cuda.current_stream().wait_stream(st)
        e.record()
        e.synchronize()
    print(f"{k} stream(s): {8 * n * 4 / (s.elapsed_time(e) * 1e-3) / 1e9:.1f} GB/s")
