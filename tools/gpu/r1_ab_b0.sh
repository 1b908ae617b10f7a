mkdir -p gpurun_out
for lib in build/nob0 paper_1304_7054_b200; do for i in 1 2; do
  KB_LIB_PATH=$PWD/$lib/libkronbatch_b200.so timeout 120 python tools/quickbench.py one 2 16 f32 4194304 20 | sed "s#^#$lib #"
  KB_LIB_PATH=$PWD/$lib/libkronbatch_b200.so timeout 120 python tools/quickbench.py one 2 10 f32 4194304 20 | sed "s#^#$lib #"
  KB_LIB_PATH=$PWD/$lib/libkronbatch_b200.so timeout 120 python tools/quickbench.py one 2 16 f64 2097152 20 | sed "s#^#$lib #"
done; done
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_kron2.py -m gpu -q -x 2>&1 | tail -2
