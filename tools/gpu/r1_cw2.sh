mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py -m gpu -q -x 2>&1 | tail -3
for f in 0 1 2; do for t in f32 f64; do KB_K2=$f timeout 300 python tools/quickbench.py sweepd 2 $t 2>&1 | sed "s/^/K2=$f /"; done; done
for f in 0 1 2; do KB_K2=$f timeout 120 python tools/launch_overhead.py 65536 2>&1 | sed "s/^/K2=$f /"; done
