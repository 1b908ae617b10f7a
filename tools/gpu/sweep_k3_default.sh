# Default 3-D dispatch, every n = 3..16, fp32 / fp64, 2 GiB of X per point.
for t in f32 f64; do
  for n in $(seq 3 16); do
    es=4; [ $t = f64 ] && es=8
    b=$(( 2147483648 / (n*n*n*es) ))
    timeout 120 python tools/quickbench.py one 3 $n $t $b 5 2>&1
  done
done
