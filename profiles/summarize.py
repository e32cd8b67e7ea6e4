"""Summarise an ncu report (and optionally a launch-list CSV) into profiles/.

    python profiles/summarize.py gpurun_out/prof_c4.ncu-rep --tag r01_c4 \
        [--launches gpurun_out/launches_c4.csv] [--config C4 --bytes-per-launch N]

Writes profiles/<tag>_ncu.txt (key metrics + top stall reasons) and, with --config,
profiles/ncu_<config>.json holding dram bytes per launch (bench.py's roofline.traffic).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "smsp__inst_executed.sum", "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
    "sm__cycles_elapsed.avg.per_second", "lts__t_sector_hit_rate.pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.min.pct_of_peak_sustained_active",
    "smsp__issue_active.max.pct_of_peak_sustained_active",
]
STALL = ("smsp__average_warps_issue_stalled_", "_per_issue_active.ratio")

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
         "nsecond": 1e-9}


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True,
                         text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def raw_metrics(rep):
    rows = ncu_csv(rep, "raw")
    hdr, units, data = rows[0], rows[1], rows[2:]
    kernels = []
    for row in data:
        d = {}
        for k, u, v in zip(hdr, units, row):
            d[k] = (v, u)
        kernels.append(d)
    return kernels


def to_float(v, u):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    return x * SCALE.get(u, 1.0)


def stall_reasons(rep):
    rows = ncu_csv(rep, "details")
    hdr = rows[0]
    out = []
    for row in rows[1:]:
        d = dict(zip(hdr, row))
        if d.get("Section Name", "").startswith("Warp State") or "Stall" in d.get("Metric Name", ""):
            out.append(f"{d.get('Metric Name')}: {d.get('Metric Value')} {d.get('Metric Unit')}")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--config")
    ap.add_argument("--bytes-per-launch", type=float)
    a = ap.parse_args()
    lines = [f"# ncu summary {a.tag}: {os.path.basename(a.report)}", ""]
    ks = raw_metrics(a.report)
    traffic = None
    for d in ks:
        name = d.get("Kernel Name", ("?", ""))[0]
        lines.append(f"## kernel {name[:160]}")
        for k in KEYS:
            if k in d:
                lines.append(f"{k} = {d[k][0]} {d[k][1]}")
        rd = to_float(*d["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in d else None
        wr = to_float(*d["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in d else None
        dur = to_float(*d["gpu__time_duration.sum"]) if "gpu__time_duration.sum" in d else None
        if rd is not None and wr is not None:
            traffic = rd + wr
            lines.append(f"dram bytes per launch (read+write) = {traffic:.6e}")
            if a.bytes_per_launch:
                lines.append(f"algorithmic bytes per launch = {a.bytes_per_launch:.6e}  "
                             f"(traffic / algorithmic = {traffic / a.bytes_per_launch:.4f})")
            if dur:
                lines.append(f"dram GB/s = {traffic / dur / 1e9:.1f}   "
                             f"algorithmic GB/s (ncu duration) = "
                             f"{(a.bytes_per_launch or 0) / dur / 1e9:.1f}")
        stalls = []
        for k, (v, u) in d.items():
            if k.startswith(STALL[0]) and k.endswith(STALL[1]):
                x = to_float(v, u)
                if x is not None and x >= 0.05:
                    stalls.append((x, k[len(STALL[0]):-len(STALL[1])]))
        if stalls:
            lines.append("stalls per issued instruction: " + ", ".join(
                f"{n} {x:.2f}" for x, n in sorted(stalls, reverse=True)))
        lines.append("")
    lines.append("## warp state / stalls")
    lines.extend(stall_reasons(a.report))
    if a.launches:
        lines.append("")
        lines.append("## launch list (gpu__time_duration.sum, ncu --clock-control none)")
        with open(a.launches) as f:
            text = [ln for ln in f if not ln.startswith("==")]
        rows = list(csv.reader(text))
        hdr = rows[0]
        tot = {}
        for r in rows[1:]:
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            k = d["Kernel Name"].split("(")[0][:90]
            t = to_float(d["Metric Value"], d["Metric Unit"])
            tot.setdefault(k, []).append(t)
        total = sum(sum(v) for v in tot.values())
        for k, v in sorted(tot.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"{k}: {len(v)} launches, {sum(v) * 1e3:.3f} ms total, "
                         f"{sum(v) / total * 100:.1f}% of device time, mean {sum(v) / len(v) * 1e6:.1f} us")
    path = os.path.join(HERE, f"{a.tag}_ncu.txt")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")
    print(path)
    if a.config and traffic is not None:
        with open(os.path.join(HERE, f"ncu_{a.config}.json"), "w") as f:
            json.dump({"dram_bytes_per_launch": traffic, "source": f"{a.tag}_ncu.txt",
                       "report": os.path.basename(a.report)}, f, indent=1)


if __name__ == "__main__":
    main()
