"""Per-source-line hotspots of one kernel in an ncu report (needs -lineinfo builds).

    python tools/ncu_lines.py gpurun_out/x.ncu-rep raster_kernel [--top 25]

Prints, per CUDA source line, warp-stall samples, instructions executed (warp level) and the
dominant stall reasons, sorted by samples.
"""
from __future__ import annotations

import argparse
import csv
import io
import subprocess
from collections import defaultdict

ap = argparse.ArgumentParser()
ap.add_argument("report")
ap.add_argument("kernel")
ap.add_argument("--top", type=int, default=25)
ap.add_argument("--by", default="samples", choices=["samples", "inst"])
ap.add_argument("--skip", type=int, default=0, help="launches of the kernel to skip")
a = ap.parse_args()

out = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--kernel-name", a.kernel,
                      "--print-source", "cuda,sass", "--launch-skip", str(a.skip), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
cur = None
agg = defaultdict(lambda: defaultdict(float))
src = {}
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8:
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        src[cur] = r[1]
        continue
    if cur is None:
        continue
    d = dict(zip(hdr[2:], r[2:]))
    def f(k):
        try:
            return float(d.get(k, "0").replace(",", ""))
        except ValueError:
            return 0.0
    agg[cur]["samples"] += f("Warp Stall Sampling (All Samples)")
    agg[cur]["inst"] += f("Instructions Executed")
    for k in d:
        if k.startswith("stall_") and "Not Issued" not in k:
            agg[cur][k] += f(k)

tot_s = sum(v["samples"] for v in agg.values()) or 1
tot_i = sum(v["inst"] for v in agg.values()) or 1
print(f"total samples {tot_s:.0f}, warp instructions {tot_i:.3e}")
for key, v in sorted(agg.items(), key=lambda kv: -kv[1][a.by])[: a.top]:
    stalls = sorted(((k[6:], x) for k, x in v.items() if k.startswith("stall_")), key=lambda t: -t[1])[:3]
    st = " ".join(f"{k}:{x / max(v['samples'], 1):.0%}" for k, x in stalls if x)
    print(f"{key[0]}:{key[1]:<4} {v['samples'] / tot_s:6.1%} smp {v['inst'] / tot_i:6.1%} inst  "
          f"{st:40s} | {src[key].strip()[:90]}")
