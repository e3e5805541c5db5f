"""Summarise one `ncu --set full` report: speed-of-light, memory, occupancy,
scheduler sections + DRAM bytes and tensor-pipe activity (for profiles/)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
NCU = "/usr/local/cuda/bin/ncu"
det = subprocess.run([NCU, "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(det)))
h = rows[0]
si, mi, vi, ui = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
keep = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Occupancy", "Warp State Statistics",
        "Launch Statistics", "Scheduler Statistics", "Compute Workload Analysis")
kn = h.index("Kernel Name") if "Kernel Name" in h else None
if kn is not None and len(rows) > 1:
    print(f"kernel: {rows[1][kn]}")
for r in rows[1:]:
    if r[si] in keep and r[mi]:
        print(f"{r[si][:28]:28s} | {r[mi]} = {r[vi]} {r[ui]}")
raw = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hh, uu, vv = rr[0], rr[1], rr[2]
for w in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
          "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
          "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]:
    if w in hh:
        i = hh.index(w)
        print(f"raw | {w} = {vv[i]} {uu[i]}")
