"""Headline metrics and stall mix of every kernel in an ncu --set full report."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(out))
for row in rows[2:]:
    d = dict(zip(rows[0], row))
    print("==", d.get("Kernel Name", "")[:90])
    for k in ["gpu__time_duration.sum", "launch__registers_per_thread",
              "sm__warps_active.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
              "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
              "smsp__thread_inst_executed_per_inst_executed.ratio",
              "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
              "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "l1tex__t_bytes.sum"]:
        print(f"  {k:60s} {d.get(k)}")
    st = {k: float(v.replace(',', '')) for k, v in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued") and v}
    tot = sum(st.values()) or 1
    for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:9]:
        print(f"    {k[33:]:40s} {v / tot:6.3f}")
