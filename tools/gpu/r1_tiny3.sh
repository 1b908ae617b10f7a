mkdir -p gpurun_out
KB_K3=9 python tests/variant_check.py
timeout 900 python -m pytest tests/test_gpu_kron3.py tests/test_gpu_variants.py -m gpu -q -x 2>&1 | tail -2
for t in f32 f64; do for n in 1 2 3 4; do
  es=4; [ $t = f64 ] && es=8
  b=$(( 2147483648 / (n*n*n*es) ))
  for f in 9 0 3; do KB_K3=$f timeout 120 python tools/quickbench.py one 3 $n $t $b 5 2>&1 | sed "s/^/K3=$f /"; done
done; done
