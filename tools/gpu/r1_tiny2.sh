mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py -m gpu -q -x 2>&1 | tail -3
for f in 0 1 2; do for t in f32 f64; do for n in 1 2 3 4 5 7; do
  es=4; [ $t = f64 ] && es=8
  b=$(( 2147483648 / (n*n*es) ))
  KB_K2=$f timeout 120 python tools/quickbench.py one 2 $n $t $b 5 2>&1 | sed "s/^/K2=$f /"
done; done; done
for lib in paper_1304_7054_b200 build/altf64; do KB_LIB_PATH=$PWD/$lib/libkronbatch_b200.so timeout 120 python tools/quickbench.py one 3 16 f64 131072 10 | sed "s#^#$lib #"; done
KB_LIB_PATH=$PWD/build/altf64/libkronbatch_b200.so KB_K3=2 python tests/variant_check.py
