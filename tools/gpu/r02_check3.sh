mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_sanitizer.py -m gpu -q 2>&1 | tail -4
grep -E "SUMMARY" gpurun_out/sanitize_*.log
python tools/probe_hostreg.py
KB_TF32=1 timeout 120 python tools/quickbench.py one 3 16 f32 262144 5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kron3_tc -s 2 -c 1 -o gpurun_out/prof_tc_r1 env KB_TF32=1 python tools/quickbench.py one 3 16 f32 262144 3 > gpurun_out/ncu_tc.log 2>&1; tail -3 gpurun_out/ncu_tc.log
ls -la gpurun_out/*.ncu-rep
