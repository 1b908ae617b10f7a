for n in 4 5 8; do b=$((1073741824 / (n*n*n*4))); echo "n=$n b=$b"; KB_K3=14 timeout 30 python tools/quickbench.py one 3 $n f32 $b 3 2>&1 | tail -1; done
echo "f64 n=4"; KB_K3=14 timeout 30 python tools/quickbench.py one 3 4 f64 2097152 3 2>&1 | tail -1
for i in 1 2; do for n in 16 14; do timeout 30 python tools/quickbench.py one 3 $n f32 262144 10 2>&1 | tail -1; done; done
KB_K3=14 timeout 300 python tests/variant_check.py
timeout 120 ncu --set full --clock-control none --import-source on -k regex:kron3_ -s 3 -c 1 -o gpurun_out/prof_kron3_f32_n16_v7 python tools/quickbench.py one 3 16 f32 262144 1 > /dev/null 2>&1; ls -la gpurun_out/prof_kron3_f32_n16_v7.ncu-rep
