for e in "KB_K2=0" "KB_K2=1" "KB_K2=2" "KB_YSTAGE=1" "KB_YSTAGE=0" "X=1"; do echo "$e: $(env $e timeout 600 python tests/variant_check.py | tail -1)"; done
timeout 900 python -m pytest tests/test_gpu_kron2.py tests/test_gpu_golden.py -m gpu -q -x 2>&1 | tail -2
for n in 16 10 15 13 11 9 8 6; do b=$((2147483648 / (n*n*4))); for d in 0 1; do echo "DYN=$d 2d n=$n"; KB_DYN=$d timeout 60 python tools/quickbench.py one 2 $n f32 $b 10 2>&1 | tail -1; done; done
for n in 16 11 13; do b=$((2147483648 / (n*n*8))); for d in 0 1; do echo "DYN=$d 2d f64 n=$n"; KB_DYN=$d timeout 60 python tools/quickbench.py one 2 $n f64 $b 10 2>&1 | tail -1; done; done
timeout 300 python tools/bench_one.py kron2-f32-n16 sleep1 kron2-f32-n10 sleep1 kron2-f32-n16
