for e in "X=1" "KB_OM=0"; do echo "$e: $(env $e timeout 600 python tests/variant_check.py | tail -1)"; done
timeout 900 python -m pytest tests/test_gpu_kron3.py tests/test_gpu_golden.py tests/test_gpu_sanitizer.py -m gpu -q 2>&1 | tail -1
echo "f32 n=9: $(timeout 60 python tools/quickbench.py one 3 9 f32 368224 10 2>&1 | tail -1)"
echo "f64 n=9: $(timeout 60 python tools/quickbench.py one 3 9 f64 184112 10 2>&1 | tail -1)"
