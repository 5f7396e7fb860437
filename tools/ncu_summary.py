"""Summarise ncu reports for profiles/ (run in the build container; ncu -i needs no GPU).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [more.ncu-rep] --out profiles/r01_kernels.md
    python tools/ncu_summary.py --launches gpurun_out/launches.csv --out profiles/r01_launches.md

Writes a markdown table of the key per-kernel metrics, and a JSON sidecar
({kernel: {duration_ns, dram_bytes, ...}}) that bench.py reads to fill the
roofline "traffic" field.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "active_threads_per_warp",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "pipe_xu_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "pipe_fma_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "pipe_alu_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "pipe_lsu_pct",
    "l1tex__t_bytes.sum": "l1_bytes",
    "lts__t_bytes.sum": "l2_bytes",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_sb",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "stall_barrier",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_throughput_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__cycles_active.avg": "sm_cycles_active_avg",
    "sm__cycles_active.max": "sm_cycles_active_max",
    "sm__cycles_elapsed.avg": "sm_cycles_elapsed_avg",
}


def raw_metrics(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3,
             "ms": 1e6, "s": 1e9,
             "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/second": 1,
             "cycle/nsecond": 1e9, "cycle/usecond": 1e6}
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        k = {"kernel": d.get("Kernel Name", "?")[:90]}
        for m, short in KEYS.items():
            if m in d and d[m] not in ("", "n/a"):
                try:
                    k[short] = float(d[m].replace(",", "")) * scale.get(units.get(m, ""), 1)
                except ValueError:
                    pass
        if "duration" in k:
            k["duration_ns"] = k.pop("duration")
        res.append(k)
    return res


def launches(path: str):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    agg = {}
    for r in rows[hdr_i + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0][:70]
        if "k_gate" in name:  # bench.py's timing gate: under ncu it only times out
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "nsecond")
        v *= {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "ns": 1.0, "us": 1e3,
              "ms": 1e6}.get(unit, 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="*")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    args = ap.parse_args()
    lines = [f"# {args.title}", ""]
    side = {}
    if args.launches:
        agg = launches(args.launches)
        tot = sum(v[1] for v in agg.values())
        lines += ["Per-kernel device time from `ncu --metrics gpu__time_duration.sum "
                  "--clock-control none` (cold-cache, serialised: compare shares).", "",
                  "| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
        for name, (cnt, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| `{name}` | {cnt} | {ns / 1e6:.3f} | {ns / tot:.3f} |")
        lines.append("")
    for rep in args.reports:
        for k in raw_metrics(rep):
            name = k.pop("kernel")
            dram = k.get("dram_read", 0) + k.get("dram_write", 0)
            k["dram_bytes"] = dram
            side[name] = k
            lines += [f"## `{name}`", f"source: `{rep}` (`ncu --set full --clock-control none`)", "",
                      "| metric | value |", "|---|---:|"]
            for kk, v in k.items():
                lines.append(f"| {kk} | {v:,.4g} |")
            lines.append("")
    with open(args.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if side:
        with open(args.out.rsplit(".", 1)[0] + ".json", "w") as f:
            json.dump(side, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    sys.exit(main())
