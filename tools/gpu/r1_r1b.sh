mkdir -p gpurun_out
KB_K3=10 python tests/variant_check.py
for cfg in "16 f32 262144" "12 f32 262144" "10 f32 262144" "16 f64 131072" "14 f64 131072" "12 f64 131072" "10 f64 262144"; do
  set -- $cfg
  for f in 10 3 2; do KB_K3=$f timeout 120 python tools/quickbench.py one 3 $1 $2 $3 10 | sed "s/^/K3=$f /"; done
done
