for e in "X=1" "KB_K2=1" "KB_K2=2"; do echo "$e: $(env $e timeout 600 python tests/variant_check.py | tail -1)"; done
timeout 1500 python -m pytest tests/test_gpu_kron2.py tests/test_gpu_golden.py tests/test_gpu_sanitizer.py -m gpu -q 2>&1 | tail -1
for c in "9 f32" "13 f32" "10 f64" "13 f64"; do set -- $c; es=4; [ $2 = f64 ] && es=8; echo "2d $2 n=$1: $(timeout 60 python tools/quickbench.py one 2 $1 $2 $((1073741824 / ($1*$1*es))) 10 2>&1 | tail -1)"; done
