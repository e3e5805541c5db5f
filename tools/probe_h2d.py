"""Probe the host link: H2D copy-engine bandwidth vs copy size (pinned), with and
without a concurrent D2H stream, plus the GPU's NUMA node and this process's
CPU affinity (pinned memory placement decides whether H2D crosses sockets)."""
import glob
import json
import os
import subprocess

import torch

out = {"nproc": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}
try:
    bus = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader"], capture_output=True,
                         text=True).stdout.strip().splitlines()[0].lower()
    dom = bus.split(":", 1)[1] if bus.count(":") > 2 else bus
    for p in glob.glob("/sys/bus/pci/devices/*"):
        if p.endswith(dom[-12:]):
            out["gpu_numa_node"] = open(p + "/numa_node").read().strip()
    out["numa_nodes"] = sorted(os.path.basename(p) for p in glob.glob("/sys/devices/system/node/node*"))
    out["lscpu"] = [l for l in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines()
                    if "NUMA" in l or "Model name" in l or "Socket" in l]
except Exception as e:  # noqa: BLE001
    out["numa_err"] = str(e)

dev = torch.device("cuda:0")
N = 2 << 30
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(N, dtype=torch.uint8, device=dev)
hd = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=True)
dd = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
s_h2d = torch.cuda.Stream()
s_d2h = torch.cuda.Stream()


def h2d(size, concurrent=False):
    n = N // size
    torch.cuda.synchronize()
    with torch.cuda.stream(s_h2d):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        if concurrent:
            with torch.cuda.stream(s_d2h):
                for _ in range(8):
                    hd.copy_(dd, non_blocking=True)
        for i in range(n):
            d[i * size:(i + 1) * size].copy_(h[i * size:(i + 1) * size], non_blocking=True)
        b.record()
    torch.cuda.synchronize()
    return N / (a.elapsed_time(b) / 1e3) / 1e9


for size in [512 << 10, 2 << 20, 8 << 20, 16 << 20, 64 << 20, 256 << 20]:
    h2d(size)
    out[f"h2d_{size >> 10}KiB_GBs"] = round(h2d(size), 2)
    out[f"h2d_{size >> 10}KiB_with_d2h_GBs"] = round(h2d(size, True), 2)
print(json.dumps(out, indent=1))
