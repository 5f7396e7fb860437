# On the GPU box: time every abx/*.so (or $AB) with tools/abk.py; results in gpurun_out/abx.txt
: > gpurun_out/abx.txt
for v in ${AB:-$(ls abx/*.so | xargs -n1 basename | sed 's/\.so$//')}; do
  FSB_LIB=abx/$v.so KERNELS=${KERNELS:-warp,fast,f64} timeout 600 python tools/abk.py >> gpurun_out/abx.txt 2>&1
done
cat gpurun_out/abx.txt
