mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py -m gpu -q -x 2>&1 | tail -3
KB_K3=3 python tests/variant_check.py
for f in 0 1 2 3; do
  for cfg in "16 f32 262144" "14 f32 262144" "12 f32 262144" "10 f32 262144" "8 f32 1048576"; do
    set -- $cfg; KB_K3=$f timeout 120 python tools/quickbench.py one 3 $1 $2 $3 10 2>&1 | sed "s/^/K3=$f /"
  done
done
KB_K3=3 timeout 300 ncu --set full --clock-control none --import-source on -k regex:kron3_cw -s 3 -c 1 -o gpurun_out/cw3_f32_n16 python tools/quickbench.py one 3 16 f32 262144 1 > /dev/null 2>&1
