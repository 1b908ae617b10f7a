# Source-level ncu captures of the 3-D kernels + variant tests.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_variants.py -m gpu -q -x 2>&1 | tail -3
for cfg in "3 16 f32 262144" "3 10 f32 262144" "3 16 f64 131072" "2 10 f32 1048576"; do
  set -- $cfg
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:kron._sq -s 3 -c 1 \
     -o gpurun_out/src_k$1_$3_n$2 python tools/quickbench.py one $1 $2 $3 $4 1 > /dev/null 2>&1
done
ls -la gpurun_out
