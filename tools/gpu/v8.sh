# V8 (V2 tiles on a 4-stage ring): correctness, then odd / small n and fp32 n = 14 family timings
echo "KB_K3=15: $(KB_K3=15 timeout 600 python tests/variant_check.py | tail -1)"
for dt in f32 f64; do es=4; [ $dt = f64 ] && es=8
 for n in 5 6 7 9 11 13 15; do b=$((1073741824 / (n*n*n*es)))
  for f in -1 15 3; do echo "3d $dt n=$n K3=$f: $(KB_K3=$f timeout 60 python tools/quickbench.py one 3 $n $dt $b 10 2>&1 | tail -1)"; done
 done
done
for f in -1 1 2 3 10 11 14 15; do echo "3d f32 n=14 K3=$f: $(KB_K3=$f timeout 60 python tools/quickbench.py one 3 14 f32 97827 10 2>&1 | tail -1)"; done
for f in -1 1 2 3 10 11 15; do echo "3d f64 n=14 K3=$f: $(KB_K3=$f timeout 60 python tools/quickbench.py one 3 14 f64 48914 10 2>&1 | tail -1)"; done
for f in -1 1 3 10 11 15; do echo "3d f64 n=16 K3=$f: $(KB_K3=$f timeout 60 python tools/quickbench.py one 3 16 f64 131072 10 2>&1 | tail -1)"; done
