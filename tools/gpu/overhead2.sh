build/microbench/call_overhead
timeout 1500 python -m pytest tests/test_gpu_kron2.py tests/test_gpu_kron3.py tests/test_gpu_blas.py tests/test_gpu_runtime.py tests/test_gpu_shard.py -m gpu -q 2>&1 | tail -1
