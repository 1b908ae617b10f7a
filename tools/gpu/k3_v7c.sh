KB_K3=14 timeout 600 compute-sanitizer --tool memcheck --print-limit 3 python tools/quickbench.py one 3 8 f32 524288 1 2>&1 | grep -v "^$" | grep -v "Host Frame" | head -30
for rep in 1 2; do
for n in 16 10 12 14; do
  for f in 14 3; do echo "K3=$f n=$n"; KB_K3=$f timeout 120 python tools/quickbench.py one 3 $n f32 $((2147483648 / (n*n*n*4))) 10; done
done
done
