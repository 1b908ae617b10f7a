mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
./tools/microbench/fma_tput > gpurun_out/fma_tput.txt 2>&1; cat gpurun_out/fma_tput.txt
timeout 600 python -m pytest tests/test_gpu_variants.py -m gpu -q -x 2>&1 | tail -2
bash tools/quicksweep3.sh > gpurun_out/sweep3_families.txt 2>&1; cat gpurun_out/sweep3_families.txt
