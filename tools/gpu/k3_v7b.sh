KB_K3=14 timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python tools/quickbench.py one 3 8 f32 20000 2 2>&1 | grep -v "^$" | head -30
for rep in 1 2; do
for n in 16 10 12 14; do
  for f in 14 ""; do echo "K3=$f n=$n"; KB_K3=$f timeout 120 python tools/quickbench.py one 3 $n f32 $((1073741824 / (n*n*n*4))) 10; done
done
done
for n in 16 10; do for f in 14 ""; do echo "K3=$f f32 262144"; KB_K3=$f timeout 120 python tools/quickbench.py one 3 $n f32 262144 10; done; done
