mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_acceptance.py tests/test_kronbench.py -m gpu -q -x -s 2>&1 | grep -E "criterion|passed|failed|Error" | head -20
timeout 1500 python tools/sweep_configs4.py > gpurun_out/sweep_configs4.md 2> gpurun_out/sweep.err; cat gpurun_out/sweep_configs4.md; tail -3 gpurun_out/sweep.err
