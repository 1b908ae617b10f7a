# 3-D odd-n family re-pick + Y staging, 2-D bulk Y stores: correctness then sweeps
for e in "X=1" "KB_K3=1" "KB_K3=3" "KB_K3=14" "KB_K2=0" "KB_K2=1" "KB_K2=2" "KB_YSTAGE=1" "KB_YS=0"; do echo "$e: $(env $e timeout 600 python tests/variant_check.py | tail -1)"; done
timeout 1500 python -m pytest tests/test_gpu_kron2.py tests/test_gpu_kron3.py tests/test_gpu_golden.py tests/test_gpu_sanitizer.py -m gpu -q 2>&1 | tail -3
for dt in f32 f64; do es=4; [ $dt = f64 ] && es=8
 for n in 3 5 6 7 8 9 10 11 12 13 14 15; do b=$((1073741824 / (n*n*es)))
  echo "2d $dt n=$n default: $(timeout 60 python tools/quickbench.py one 2 $n $dt $b 10 2>&1 | tail -1)"
  for e in "KB_K2=0 KB_YSTAGE=0" "KB_K2=0 KB_YSTAGE=1" "KB_K2=1" "KB_K2=2"; do echo "2d $dt n=$n $e: $(env $e timeout 60 python tools/quickbench.py one 2 $n $dt $b 10 2>&1 | tail -1)"; done
 done
 for n in 5 7 9 11 13 15; do b=$((1073741824 / (n*n*n*es))); echo "3d $dt n=$n default: $(timeout 60 python tools/quickbench.py one 3 $n $dt $b 10 2>&1 | tail -1)"; done
done
