for i in 1 2; do KB_K3=14 timeout 120 python tools/quickbench.py one 3 8 f32 524288 10 2>&1 | tail -1; done
KB_K3=14 timeout 900 python tests/variant_check.py
for n in 16 14 8; do for f in 14 3; do echo "K3=$f n=$n"; KB_K3=$f timeout 120 python tools/quickbench.py one 3 $n f32 $((2147483648 / (n*n*n*4))) 10; done; done
for f in 14 3; do echo "K3=$f n=16 262144"; KB_K3=$f timeout 120 python tools/quickbench.py one 3 16 f32 262144 10; done
