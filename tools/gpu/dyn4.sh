for n in 5 6 13 15; do b=$((2147483648 / (n*n*n*4))); for d in 0 1; do echo "DYN=$d n=$n"; KB_DYN=$d timeout 60 python tools/quickbench.py one 3 $n f32 $b 10 2>&1 | tail -1; done; done
for n in 5 7 9 11 13 15; do b=$((2147483648 / (n*n*n*8))); for d in 0 1; do echo "DYN=$d f64 n=$n"; KB_DYN=$d timeout 60 python tools/quickbench.py one 3 $n f64 $b 10 2>&1 | tail -1; done; done
timeout 300 python tools/bench_one.py kron3-f32-n16 sleep1 kron3-f32-n10 sleep1 kron3-f64-n16 sleep1 kron2-f32-n16
