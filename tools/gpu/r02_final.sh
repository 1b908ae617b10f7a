# End-of-round: full GPU suite, smoke, bench + reference arm, configs[4] sweep
bash tools/gpu/r02_full.sh > gpurun_out/r02_full.log 2>&1
timeout 1500 python tools/sweep_configs4.py > gpurun_out/sweep_configs4.md 2> gpurun_out/sweep.err; tail -3 gpurun_out/sweep.err
