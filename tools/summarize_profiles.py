"""Summarise ncu outputs brought back in gpurun_out/ into profiles/ (tracked).

    python tools/summarize_profiles.py --tag r2_cfg1 --config cfg1 \
        --launches gpurun_out/launches_bench.csv --report gpurun_out/prof_frame.ncu-rep

Writes profiles/<tag>_launches.md (per-kernel launch statistics of the bench command),
profiles/<tag>_frame.md (one full-set capture of every kernel of one frame) and, under the
config's key, profiles/traffic.json (DRAM read+write bytes per frame of every pipeline stage)
and profiles/instructions.json (warp instructions per frame), which bench.py reads for the
SAME config only.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import re
import subprocess
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROF = ROOT / "profiles"

STAGES = {
    "preprocess": ["preprocess_kernel"],
    "depth_sort": ["key_hist_kernel", "chunk_table_kernel", "onesweep_kernel"],
    "binning": ["bin_count_kernel", "bin_colscan_kernel", "bin_tilescan_kernel", "bin_campre_kernel"],
    "scatter": ["bin_scatter_kernel"],
    "raster": ["raster_kernel"],
}


def short(name: str) -> str:
    name = re.sub(r"\(.*", "", name)
    name = name.replace("void ", "").replace("gsim_gpu::", "")
    return name.strip()


def launches(path: Path) -> dict:
    rows = list(csv.reader(open(path)))
    hdr = None
    per = defaultdict(lambda: defaultdict(list))
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            try:
                v = float(d["Metric Value"].replace(",", ""))
            except ValueError:
                continue
            key = (d["ID"], short(d["Kernel Name"]))
            per[key][d["Metric Name"]].append(v)
    agg = defaultdict(lambda: defaultdict(list))
    for (lid, name), m in per.items():
        for k, v in m.items():
            agg[name][k].append(v[0])
    return agg


def raw_report(rep: Path) -> list[dict]:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def f(d, k, default=float("nan")):
    try:
        return float(str(d.get(k, "")).replace(",", ""))
    except ValueError:
        return default


def merge_json(path: Path, config: str, entry: dict) -> None:
    """profiles/*.json hold one entry per config (bench.py never reads another config's)."""
    data = {}
    if path.exists():
        try:
            data = json.loads(path.read_text())
        except ValueError:
            data = {}
    data = {k: v for k, v in data.items() if isinstance(v, dict)}  # drop the r1 flat layout
    data[config] = entry
    path.write_text(json.dumps(data, indent=1) + "\n")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--launches")
    ap.add_argument("--report")
    ap.add_argument("--config", default="cfg1")
    a = ap.parse_args()
    PROF.mkdir(exist_ok=True)
    if a.launches:
        agg = launches(Path(a.launches))
        lines = [f"# {a.tag}: launch list of `bench.py --steps 4 --warmup 3 --contexts 1` under "
                 "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                 "--clock-control none` (cold-cache, serialised: compare shares, not absolutes)", "",
                 "| kernel | launches | mean us | share | DRAM read MB/launch | DRAM write MB/launch |",
                 "|---|---|---|---|---|---|"]
        tot = sum(sum(m["gpu__time_duration.sum"]) for m in agg.values())
        for name, m in sorted(agg.items(), key=lambda x: -sum(x[1]["gpu__time_duration.sum"])):
            t = m["gpu__time_duration.sum"]
            rd = m.get("dram__bytes_read.sum", [0])
            wr = m.get("dram__bytes_write.sum", [0])
            lines.append(f"| {name} | {len(t)} | {sum(t) / len(t) / 1e3:.1f} | {sum(t) / tot:.3f} | "
                         f"{sum(rd) / len(rd) / 1e6:.1f} | {sum(wr) / len(wr) / 1e6:.1f} |")
        (PROF / f"{a.tag}_launches.md").write_text("\n".join(lines) + "\n")
        # stage traffic (per frame): sum over the stage's kernels of mean bytes per launch x
        # launches per frame
        frames = sum(len(m["gpu__time_duration.sum"]) for n, m in agg.items()
                     if n.startswith("raster_kernel")) or 1
        traffic = {}
        for stage, kernels in STAGES.items():
            b = 0.0
            for name, m in agg.items():
                if not any(name.startswith(k) for k in kernels):
                    continue
                b += (sum(m.get("dram__bytes_read.sum", [0])) + sum(m.get("dram__bytes_write.sum", [0]))) / frames
            traffic[stage] = int(b)
        merge_json(PROF / "traffic.json", a.config, {
            "source": f"profiles/{a.tag}_launches.md (ncu dram__bytes_read.sum + dram__bytes_write.sum "
                      f"per frame, {a.config})", **traffic})
    if a.report:
        rows, units = raw_report(Path(a.report))
        scale_to = {"us": {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3},
                    "MB": {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3},
                    "GB/s": {"byte/s": 1e-9, "Kbyte/s": 1e-6, "Mbyte/s": 1e-3, "Gbyte/s": 1,
                             "Tbyte/s": 1e3}}
        keys = [("gpu__time_duration.sum", "us", None), ("dram__bytes_read.sum", "MB", None),
                ("dram__bytes_write.sum", "MB", None),
                ("dram__bytes.sum.per_second", "GB/s", None),
                ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "% DRAM", 1),
                ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "% L2", 1),
                ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                 "% smem", 1),
                ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "% SM", 1),
                ("smsp__issue_active.avg.pct_of_peak_sustained_active", "% issue", 1),
                ("sm__warps_active.avg.per_cycle_active", "warps/SM", 1),
                ("launch__registers_per_thread", "regs", 1),
                ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "% fp64 pipe", 1)]
        lines = [f"# {a.tag}: `ncu --set full --clock-control none` of every kernel of one {a.config} "
                 "frame (tools/profile_step.py)", "",
                 "| kernel | " + " | ".join(f"{k.split('__')[-1][:28]} ({u})" for k, u, _ in keys) + " | top stalls |",
                 "|---|" + "---|" * (len(keys) + 1)]
        for d in rows:
            name = short(d.get("Kernel Name", "?"))
            stalls = sorted(((f(d, k), k) for k in d if k.startswith("smsp__average_warps_issue_stalled_")
                             and k.endswith("_per_issue_active.ratio")), reverse=True)[:3]
            st = ", ".join(f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}"
                           f" {v:.1f}" for v, k in stalls)
            vals = " | ".join(
                f"{f(d, k) * (s if s is not None else scale_to[u].get(units.get(k, ''), float('nan'))):.1f}"
                for k, u, s in keys)
            lines.append(f"| {name} | {vals} | {st} |")
        (PROF / f"{a.tag}_frame.md").write_text("\n".join(lines) + "\n")
        # warp instructions per frame of every stage (bench.py's issue-rate roofline)
        inst = {}
        for stage, kernels in STAGES.items():
            inst[stage] = int(sum(f(d, "smsp__inst_executed.sum", 0.0) for d in rows
                                  if any(short(d.get("Kernel Name", "")).startswith(k) for k in kernels)))
        merge_json(PROF / "instructions.json", a.config, {
            "source": f"profiles/{a.tag}_frame.md (ncu smsp__inst_executed.sum per frame, {a.config}, "
                      "one context)", **inst})


if __name__ == "__main__":
    main()
