mkdir -p gpurun_out
KB_K3=6 python tests/variant_check.py
for f in 3 4 6; do
  for cfg in "16 f32 262144" "16 f64 131072"; do
    set -- $cfg; KB_K3=$f timeout 120 python tools/quickbench.py one 3 $1 $2 $3 10 2>&1 | sed "s/^/K3=$f /"
  done
done
KB_K3=6 timeout 300 ncu --set full --clock-control none --import-source on -k regex:kron3_cw -s 3 -c 1 -o gpurun_out/cwpp_f32_n16 python tools/quickbench.py one 3 16 f32 262144 1 > /dev/null 2>&1
