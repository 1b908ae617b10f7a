for f in "" 0 1 2 3 10 11 13 14; do if [ -z "$f" ]; then unset KB_K3; else export KB_K3=$f; fi; echo "K3=${f:-default}: $(timeout 600 python tests/variant_check.py | tail -1)"; done
unset KB_K3
for n in 5 7 9 10 11 12; do b=$((2147483648 / (n*n*n*4))); for d in 0 1; do echo "DYN=$d n=$n"; KB_DYN=$d timeout 60 python tools/quickbench.py one 3 $n f32 $b 10 2>&1 | tail -1; done; done
for n in 10 12 16; do b=$((2147483648 / (n*n*n*8))); for d in 0 1; do echo "DYN=$d f64 n=$n"; KB_DYN=$d timeout 60 python tools/quickbench.py one 3 $n f64 $b 10 2>&1 | tail -1; done; done
