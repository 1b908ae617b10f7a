# odd-n 3-D Y staging (KB_YS): correctness over every odd-n family, then A/B and a family re-pick
for e in "X=1" "KB_K3=0" "KB_K3=1" "KB_K3=2" "KB_K3=3" "KB_K3=11" "KB_K3=13" "KB_K3=14"; do echo "$e: $(env $e timeout 600 python tests/variant_check.py | tail -1)"; done
timeout 1200 python -m pytest tests/test_gpu_kron3.py tests/test_gpu_golden.py tests/test_gpu_sanitizer.py -m gpu -q -x 2>&1 | tail -3
for dt in f32 f64; do es=4; [ $dt = f64 ] && es=8
 for n in 5 7 9 11 13 15; do b=$((1073741824 / (n*n*n*es)))
  for y in 0 1; do echo "YS=$y $dt n=$n default: $(KB_YS=$y timeout 60 python tools/quickbench.py one 3 $n $dt $b 10 2>&1 | tail -1)"; done
  for f in 0 1 2 3 11 13 14; do echo "YS=1 $dt n=$n K3=$f: $(KB_K3=$f timeout 60 python tools/quickbench.py one 3 $n $dt $b 10 2>&1 | tail -1)"; done
 done
done
