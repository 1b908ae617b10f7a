# Round-1 re-entry check: GPU tests, smoke, kernel timings (CUDA-core + TF32), bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -8
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"
timeout 300 python tools/quickbench.py main 2>&1
KB_TF32=1 timeout 120 python tools/quickbench.py one 3 16 f32 262144 10 2>&1 | sed 's/^/TF32 /'
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
