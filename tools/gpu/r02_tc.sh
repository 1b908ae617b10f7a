mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -m gpu -q -x 2>&1 | tail -3
for w in 3 4 5; do echo "WGS=$w"; KB_TC_WGS=$w KB_TF32=1 timeout 120 python tools/quickbench.py one 3 16 f32 262144 10; done
timeout 120 python tools/quickbench.py one 3 16 f32 262144 10
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kron3_tc -s 2 -c 1 -o gpurun_out/prof_tc_r2b env KB_TC_WGS=${PROF_WGS:-5} KB_TF32=1 python tools/quickbench.py one 3 16 f32 262144 3 > gpurun_out/ncu_tc.log 2>&1; tail -1 gpurun_out/ncu_tc.log
