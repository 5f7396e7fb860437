# Round-2 evidence pass on one B200: ncu --set full of the hot kernels, the bench's
# launch list, then a clean bench run (no profiler).  Outputs in gpurun_out/.
set -x
mkdir -p gpurun_out
N="ncu --set full --import-source on --clock-control none -c 1 -f"
KERNELS=warp $N -k regex:k_sto_warp -o gpurun_out/r02_warp python tools/abk.py > /dev/null 2>&1
KERNELS=fast $N -k regex:k_sto_fast -o gpurun_out/r02_fast python tools/abk.py > /dev/null 2>&1
KERNELS=f64 $N -k regex:k_sto64 -o gpurun_out/r02_sto64 python tools/abk.py > /dev/null 2>&1
$N -k regex:k_bh_units -o gpurun_out/r02_bh python tools/profile_c4.py --what bh --reps 1 > /dev/null 2>&1
FSB_BENCH_NO_GATE=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c5-anchor > gpurun_out/r02_launch_bench.log 2>&1
true
ls -la gpurun_out
