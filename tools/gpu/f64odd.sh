for n in 5 9 11 13 15; do b=$((1073741824 / (n*n*n*8)))
  for e in "X=1" "KB_K3=1" "KB_K3=2" "KB_K3=3" "KB_K3=11" "KB_YS=1" "KB_YS=1 KB_K3=1" "KB_YS=1 KB_K3=3"; do echo "3d f64 n=$n $e: $(env $e timeout 60 python tools/quickbench.py one 3 $n f64 $b 10 2>&1 | tail -1)"; done
done
for n in 5 9 11 15; do b=$((1073741824 / (n*n*n*4)))
  for e in "X=1" "KB_K3=1" "KB_K3=3" "KB_K3=13" "KB_YS=0"; do echo "3d f32 n=$n $e: $(env $e timeout 60 python tools/quickbench.py one 3 $n f32 $b 10 2>&1 | tail -1)"; done
done
