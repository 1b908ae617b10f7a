KB_K3=14 timeout 600 python tests/variant_check.py
timeout 900 python -m pytest tests/test_gpu_kron3.py tests/test_gpu_runtime.py -m gpu -q -x 2>&1 | tail -2
timeout 300 python tools/bench_one.py kron3-f32-n16 sleep1 kron3-f32-n16 sleep1 kron3-f32-n10
for n in 9 10 11 12 13 15; do b=$((2147483648 / (n*n*n*4))); for f in 14 ""; do echo "K3=${f:-default} n=$n"; if [ -z "$f" ]; then unset KB_K3; else export KB_K3=$f; fi; timeout 60 python tools/quickbench.py one 3 $n f32 $b 10 2>&1 | tail -1; done; done
unset KB_K3
for n in 10 12 16; do b=$((2147483648 / (n*n*n*8))); for f in 14 ""; do echo "K3=${f:-default} f64 n=$n"; if [ -z "$f" ]; then unset KB_K3; else export KB_K3=$f; fi; timeout 60 python tools/quickbench.py one 3 $n f64 $b 10 2>&1 | tail -1; done; done
