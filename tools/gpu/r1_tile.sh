mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_kron3.py -m gpu -q -x 2>&1 | tail -2
bash tools/quicksweep3.sh > gpurun_out/sweep3_tile.txt 2>&1; cat gpurun_out/sweep3_tile.txt
for t in f32 f64; do for n in 9 11 13 15; do
  es=4; [ $t = f64 ] && es=8
  b=$(( 2147483648 / (n*n*n*es) ))
  for f in 1 2 3; do KB_K3=$f timeout 120 python tools/quickbench.py one 3 $n $t $b 5 2>&1 | sed "s/^/K3=$f /"; done
done; done
