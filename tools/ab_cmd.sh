# A/B timing of library variants under ab/ (tools/build_ab.py), then the GPU tests
for v in ${AB_VARIANTS:-base}; do FSB_LIB=ab/$v.so timeout 300 python tools/ab_sto.py 2>&1 | tail -1; done > gpurun_out/ab.txt
if [ -z "$AB_NOTEST" ]; then
  timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log >> gpurun_out/ab.txt
fi
cat gpurun_out/ab.txt
