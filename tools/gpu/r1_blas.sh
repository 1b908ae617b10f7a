mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_blas.py tests/test_gpu_variants.py tests/test_kronbench.py -m gpu -q -x 2>&1 | tail -5
for i in 1 2 3; do timeout 120 python tools/quickbench.py one 2 16 f32 4194304 20; done
timeout 600 python bench.py --no-extra --no-cpu --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline'])"
