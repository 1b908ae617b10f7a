mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py -m gpu -q -x 2>&1 | tail -3
for f in 0 1 2; do
  for cfg in "16 f32 262144" "14 f32 262144" "12 f32 262144" "10 f32 262144" "8 f32 1048576" "16 f64 131072" "12 f64 131072" "10 f64 262144"; do
    set -- $cfg; KB_K3=$f timeout 120 python tools/quickbench.py one 3 $1 $2 $3 10 2>&1 | sed "s/^/K3=$f /"
  done
done
