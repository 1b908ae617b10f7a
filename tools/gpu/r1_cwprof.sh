mkdir -p gpurun_out
KB_K3=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:kron3_cw -s 3 -c 1 -o gpurun_out/cw1_f32_n16 python tools/quickbench.py one 3 16 f32 262144 1 > /dev/null 2>&1
KB_K3=2 timeout 300 ncu --set full --clock-control none --import-source on -k regex:kron3_cw -s 3 -c 1 -o gpurun_out/cw2_f32_n16 python tools/quickbench.py one 3 16 f32 262144 1 > /dev/null 2>&1
KB_K3=2 timeout 300 ncu --set full --clock-control none --import-source on -k regex:kron3_cw -s 3 -c 1 -o gpurun_out/cw2_f64_n16 python tools/quickbench.py one 3 16 f64 131072 1 > /dev/null 2>&1
ls gpurun_out
