# per-kernel times of the bucketed path on C4 (ncu launch list) + one full capture of each kernel
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,l1tex__t_sector_hit_rate.pct --clock-control none -k regex:k_sto_b --csv --log-file gpurun_out/bkt_launch.csv python tools/bkt_check.py C4 > /dev/null 2>&1
python - <<'PY'
import csv
rows = list(csv.DictReader(open("gpurun_out/bkt_launch.csv")))
for r in rows[-12:]:
    print(r["Kernel Name"][:40], r["Metric Name"], r["Metric Value"])
PY
