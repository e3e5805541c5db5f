"""Copy-engine idle time of a serving run, from a chrome trace written by
`tools/kernel_times.py --trace <file>` (gzip allowed).

Prints how busy the host->device copy stream was over its active span and the
idle gaps between consecutive onload copies (> 20 us) — the measure used to
find the false ring-event dependencies and the metadata-copy stall
(profiles/r01g_h2d_idle.txt).

  python tools/h2d_idle.py trace.json[.gz]
"""
import collections
import gzip
import json
import sys


def main():
    path = sys.argv[1]
    with (gzip.open(path) if path.endswith(".gz") else open(path)) as f:
        t = json.load(f)
    ev = [e for e in t["traceEvents"] if e.get("ph") == "X" and e.get("cat") == "gpu_memcpy" and "HtoD" in e["name"]]
    # the onload stream is the one carrying most of the H2D time (batch metadata is small)
    busy_by_stream = collections.Counter()
    for e in ev:
        busy_by_stream[e["args"].get("stream")] += e["dur"]
    s = busy_by_stream.most_common(1)[0][0]
    h = sorted((e for e in ev if e["args"].get("stream") == s), key=lambda e: e["ts"])
    span = h[-1]["ts"] + h[-1]["dur"] - h[0]["ts"]
    busy = sum(e["dur"] for e in h)
    gaps = [b["ts"] - (a["ts"] + a["dur"]) for a, b in zip(h, h[1:])]
    big = [g for g in gaps if g > 20]
    gbs = sum(e["args"].get("bytes", 0) for e in h) / busy / 1e3
    print(f"h2d busy {busy / 1e3:.1f} ms of span {span / 1e3:.1f} ms ({100 * busy / span:.1f}%); "
          f"gaps>20us: {len(big)} totalling {sum(big) / 1e3:.2f} ms; max {max(gaps):.0f} us; "
          f"{gbs:.1f} GB/s while copying")


if __name__ == "__main__":
    main()
