timeout 1200 python -m pytest tests/test_gpu_kron3.py tests/test_gpu_variants.py tests/test_gpu_parity_full.py -m gpu -q -x 2>&1 | tail -3
for i in 1 2; do for n in 16 14; do timeout 120 python tools/quickbench.py one 3 $n f32 262144 10 2>&1 | tail -1; done; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:kron3_ -s 3 -c 1 -o gpurun_out/prof_kron3_f32_n16_v7 python tools/quickbench.py one 3 16 f32 262144 1 > /dev/null 2>&1
timeout 300 compute-sanitizer --tool racecheck --racecheck-report all python tools/quickbench.py one 3 16 f32 2000 1 2>&1 | grep -E "SUMMARY"
