"""One-off probe of a GPU box: host RAM/cores, PCIe H2D/D2H bandwidth from pinned memory."""
import os, time, subprocess, json
import torch
out = {}
out["nproc"] = os.cpu_count()
out["meminfo"] = open("/proc/meminfo").read().splitlines()[:3]
out["smi"] = subprocess.run(["nvidia-smi", "--query-gpu=name,memory.total,clocks.max.sm,pcie.link.gen.max,pcie.link.width.max", "--format=csv"], capture_output=True, text=True).stdout
dev = torch.device("cuda:0")
for gb in [1, 4]:
    n = gb << 30
    t0 = time.time(); h = torch.empty(n, dtype=torch.uint8, pin_memory=True); t1 = time.time()
    out[f"pin_alloc_{gb}GB_s"] = t1 - t0
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))]:
        fn(); torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); [fn() for _ in range(3)]; e.record(); torch.cuda.synchronize()
        out[f"{name}_{gb}GB_GBs"] = 3 * n / (s.elapsed_time(e) / 1e3) / 1e9
    # chunked 1 MiB copies (page-chunk transfer granularity)
    chunk = 1 << 20
    s.record()
    for i in range(0, n, chunk):
        d[i:i+chunk].copy_(h[i:i+chunk], non_blocking=True)
    e.record(); torch.cuda.synchronize()
    out[f"h2d_1MiB_chunks_{gb}GB_GBs"] = n / (s.elapsed_time(e) / 1e3) / 1e9
    del h, d
print(json.dumps(out, indent=1))
