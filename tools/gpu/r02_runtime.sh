# Round-2 runtime checks: new runtime / parity tests, the full GPU suite, bench
# (1 GPU, and 2 parts on one GPU through the parts API), reference arm.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_parity_full.py tests/test_multiprocess_gloo.py -m gpu -q -x -s 2>&1 | tail -25
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 python bench.py --gpus 2 --devices 0,0 --no-cpu --steps 20 > gpurun_out/bench_2parts.json 2> gpurun_out/bench_2parts.err; cat gpurun_out/bench_2parts.json; tail -3 gpurun_out/bench_2parts.err
timeout 300 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.json 2>&1; cat gpurun_out/bench_ref.json
