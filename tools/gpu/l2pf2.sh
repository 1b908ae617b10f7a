echo "L2PF=3 check: $(KB_L2PF=3 timeout 600 python tests/variant_check.py | tail -1)"
for dt in f32 f64; do es=4; [ $dt = f64 ] && es=8
 for n in 5 7 9 10 11 13 15 16; do b=$((1073741824 / (n*n*es)))
  for pf in 1 2 3; do echo "L2PF=$pf 2d $dt n=$n: $(KB_L2PF=$pf timeout 60 python tools/quickbench.py one 2 $n $dt $b 10 2>&1 | tail -1)"; done
 done
done
