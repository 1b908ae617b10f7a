mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -m gpu -q -x 2>&1 | tail -3
for w in 4 5; do echo "WGS=$w"; KB_TC_WGS=$w KB_TF32=1 timeout 120 python tools/quickbench.py one 3 16 f32 262144 10; done
./build/tc_trace 5
