# 3-D kernel family sweep: even n = 4..16, fp32/fp64, KB_K3 = 0..3, 2 GiB of X per config
for t in f32 f64; do for n in 4 6 8 10 12 14 16; do
  es=4; [ $t = f64 ] && es=8
  b=$(( 2147483648 / (n*n*n*es) ))
  for f in 0 1 2 3; do KB_K3=$f timeout 120 python tools/quickbench.py one 3 $n $t $b 5 2>&1 | sed "s/^/K3=$f /"; done
done; done
