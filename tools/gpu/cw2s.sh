# 2-D column-wise kernel ring depth: main (3 stages) vs variant libraries built with -DKB_CW2_STAGES=2 / 4
for lib in "" build/var_s2/libkronbatch_b200.so build/var_s4/libkronbatch_b200.so; do
 for dt in f32 f64; do es=4; [ $dt = f64 ] && es=8
  for n in 6 9 10 11 12 13 15; do b=$((1073741824 / (n*n*es)))
   for f in 1 2; do echo "lib=${lib:-main} $dt n=$n K2=$f: $(KB_LIB_PATH=$lib KB_K2=$f timeout 60 python tools/quickbench.py one 2 $n $dt $b 10 2>&1 | tail -1)"; done
  done
 done
done
echo "S2 check: $(KB_LIB_PATH=build/var_s2/libkronbatch_b200.so KB_K2=1 timeout 600 python tests/variant_check.py | tail -1)"
