set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
for v in 0 1 3; do KB_VARIANT2=$v KB_VARIANT3=$v timeout 120 python tools/quickbench.py main 2>&1 | sed "s/^/v$v /"; done
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; tail -c 3000 gpurun_out/bench_r01.json; tail -5 gpurun_out/bench_r01.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:kron3_sq -s 3 -c 1 -o gpurun_out/k3c_f32_16 python tools/quickbench.py one 3 16 f32 262144 1 > /dev/null 2>&1
