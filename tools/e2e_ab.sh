# e2e A/B of library builds on one box: tools/e2e_ab.sh name1 name2 ... (abx/<name>.so)
: > gpurun_out/e2e_ab.txt
for r in 1 2; do for v in "$@"; do echo "== $v" >> gpurun_out/e2e_ab.txt; FSB_LIB=abx/$v.so python tools/e2e_chunks.py >> gpurun_out/e2e_ab.txt 2>&1; done; done
cat gpurun_out/e2e_ab.txt
