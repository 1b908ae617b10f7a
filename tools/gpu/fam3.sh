timeout 1800 python -m pytest tests/test_gpu_variants.py tests/test_gpu_kron3.py -m gpu -q 2>&1 | tail -3
timeout 300 python tools/bench_one.py kron3-f64-n16 sleep2 kron3-f32-n16 sleep2 kron3-f64-n16
for n in 14 15 16; do echo "3d f64 n=$n: $(timeout 60 python tools/quickbench.py one 3 $n f64 $((1073741824 / (n*n*n*8))) 10 2>&1 | tail -1)"; done
echo "3d f32 n=14: $(timeout 60 python tools/quickbench.py one 3 14 f32 97827 10 2>&1 | tail -1)"
