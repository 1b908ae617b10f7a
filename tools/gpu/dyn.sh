KB_K3=14 timeout 600 python tests/variant_check.py
timeout 900 python -m pytest tests/test_gpu_kron3.py tests/test_gpu_runtime.py tests/test_gpu_parity_full.py -m gpu -q -x 2>&1 | tail -2
timeout 300 python tools/bench_one.py kron3-f32-n16 sleep1 kron3-f32-n16 sleep1 kron3-f32-n10 sleep1 kron3-f64-n16
for n in 16 14; do for b in 262144 1048576; do timeout 60 python tools/quickbench.py one 3 $n f32 $b 10 2>&1 | tail -1; done; done
