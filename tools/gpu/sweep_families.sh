# Kernel-family sweeps that set the per-size dispatch tables
# (profiles/r01_k2_families.txt, r01_k3_families.txt): every family forced
# with KB_K2 / KB_K3 at 2 GiB of X per (dims, dtype, n).
mkdir -p gpurun_out
for t in f32 f64; do
  for f in 0 1 2; do KB_K2=$f timeout 300 python tools/quickbench.py sweepd 2 $t 2>&1 | sed "s/^/K2=$f /"; done
  for n in $(seq 1 16); do
    es=4; [ $t = f64 ] && es=8
    b=$(( 2147483648 / (n*n*n*es) ))
    for f in 0 1 2 3 9 10; do KB_K3=$f timeout 120 python tools/quickbench.py one 3 $n $t $b 5 2>&1 | sed "s/^/K3=$f /"; done
  done
done
