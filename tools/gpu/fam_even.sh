for dt in f32 f64; do es=4; [ $dt = f64 ] && es=8
 for n in 6 10 12 14; do b=$((1073741824 / (n*n*n*es)))
  for f in -1 0 1 2 3 10 11 13 14; do echo "3d $dt n=$n K3=$f: $(KB_K3=$f timeout 60 python tools/quickbench.py one 3 $n $dt $b 10 2>&1 | tail -1)"; done
 done
done
