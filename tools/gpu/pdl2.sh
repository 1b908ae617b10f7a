for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_kron3.py -m gpu -q -x -k "generated_bitwise" 2>&1 | grep -E "Error|error|passed|failed|assert" | head -8; done
for i in 1 2 3; do KB_PDL=0 timeout 300 python -m pytest tests/test_gpu_kron3.py -m gpu -q -x -k "generated_bitwise" 2>&1 | tail -1; done
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_kron3.py -m gpu -q 2>&1 | tail -1; done
