"""Pinned H2D throughput of back-to-back 16 MiB copies (the onload transfer size)
on one stream vs alternating over two streams (is per-copy overhead hidden?)."""
import json
import torch

n, size = 48, 16 << 20
h = torch.empty(n * size, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n * size, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
out = {}
for ns in (1, 2, 1, 2):
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for st in streams[:ns]:
        st.wait_event(s0)
    for i in range(n):
        with torch.cuda.stream(streams[i % ns]):
            d[i * size:(i + 1) * size].copy_(h[i * size:(i + 1) * size], non_blocking=True)
    for st in streams[:ns]:
        s1.wait(st) if False else torch.cuda.current_stream().wait_stream(st)
    s1.record()
    torch.cuda.synchronize()
    out.setdefault(f"{ns}_stream_GBs", []).append(n * size / (s0.elapsed_time(s1) / 1e3) / 1e9)
print(json.dumps(out))
