for n in 4 5 7 9 11 13 15; do b=$((1073741824 / (n*n*n*4))); echo "n=$n b=$b"; KB_K3=14 timeout 60 python tools/quickbench.py one 3 $n f32 $b 3 2>&1 | tail -1; done
for n in 4 8; do b=$((1073741824 / (n*n*n*8))); echo "f64 n=$n b=$b"; KB_K3=14 timeout 60 python tools/quickbench.py one 3 $n f64 $b 3 2>&1 | tail -1; done
