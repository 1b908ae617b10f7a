set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
for v in 0 1 2 3; do KB_VARIANT2=$v KB_VARIANT3=$v timeout 120 python tools/quickbench.py main 2>&1 | sed "s/^/v$v /"; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:kron3_sq -s 3 -c 1 -o gpurun_out/k3b_f32_16 python tools/quickbench.py one 3 16 f32 262144 1 > gpurun_out/ncu_k3b.log 2>&1
