mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_blas.py tests/test_gpu_variants.py tests/test_gpu_kron2.py -m gpu -q -x 2>&1 | tail -3
for t in f32 f64; do
  KB_K2=0 KB_YSTAGE=0 timeout 300 python tools/quickbench.py sweepd 2 $t 2>&1 | sed "s/^/K2=0 YS=0 /"
  KB_K2=0 KB_YSTAGE=1 timeout 300 python tools/quickbench.py sweepd 2 $t 2>&1 | sed "s/^/K2=0 YS=1 /"
  KB_K2=1 timeout 300 python tools/quickbench.py sweepd 2 $t 2>&1 | sed "s/^/K2=1 /"
  KB_K2=2 timeout 300 python tools/quickbench.py sweepd 2 $t 2>&1 | sed "s/^/K2=2 /"
done
timeout 120 python tools/launch_overhead.py 65536
