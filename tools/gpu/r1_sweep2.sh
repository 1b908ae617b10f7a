mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_kron2.py -m gpu -q -x 2>&1 | tail -3
for ys in 0 1; do for t in f32 f64; do KB_YSTAGE=$ys timeout 300 python tools/quickbench.py sweepd 2 $t 2>&1 | sed "s/^/YS=$ys /"; done; done
timeout 120 python tools/launch_overhead.py 65536
KB_YSTAGE=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:kron2_sq -s 3 -c 1 -o gpurun_out/k2_n10_small python tools/quickbench.py one 2 10 f32 65536 1 > /dev/null 2>&1
