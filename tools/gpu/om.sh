for e in "X=1" "KB_OM=0" "KB_K3=1" "KB_K3=2" "KB_K3=3" "KB_K3=13" "KB_K3=14" "KB_YS=0"; do echo "$e: $(env $e timeout 600 python tests/variant_check.py | tail -1)"; done
timeout 1500 python -m pytest tests/test_gpu_kron3.py tests/test_gpu_golden.py tests/test_gpu_sanitizer.py -m gpu -q 2>&1 | tail -1
for dt in f32 f64; do es=4; [ $dt = f64 ] && es=8
 for n in 5 7 9 11 13 15; do b=$((1073741824 / (n*n*n*es)))
  for om in 0 1; do echo "OM=$om 3d $dt n=$n: $(KB_OM=$om timeout 60 python tools/quickbench.py one 3 $n $dt $b 10 2>&1 | tail -1)"; done
 done
done
