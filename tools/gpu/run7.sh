set -x
./tools/microbench/mma_tput
timeout 600 python -m pytest tests/test_gpu_kron3.py -q -x 2>&1 | tail -3
for v in 0 1 3; do KB_VARIANT3=$v timeout 120 python tools/quickbench.py one 3 16 f32 262144 10 2>&1 | sed "s/^/v$v /"; done
timeout 120 python tools/quickbench.py one 3 16 f64 131072 10
timeout 120 python tools/quickbench.py one 3 10 f32 262144 10
