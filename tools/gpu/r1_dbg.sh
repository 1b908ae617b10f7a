mkdir -p gpurun_out
KB_K2=1 timeout 300 python -m pytest "tests/test_gpu_kron2.py::test_square_generated_bitwise" -m gpu -q -x 2>&1 | grep -E "assert|Error|passed|failed" | head -20
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for f in 1 2 3; do KB_K3=$f timeout 120 python tools/quickbench.py one 3 16 f32 262144 10; done
for f in 1 2; do KB_K3=$f timeout 120 python tools/quickbench.py one 3 16 f64 131072 10; done
timeout 120 python tools/quickbench.py one 3 10 f32 262144 10
