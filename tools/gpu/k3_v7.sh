KB_K3=14 timeout 600 python tests/variant_check.py
for n in 16 10 12 14 8; do
  for f in "" 14; do echo "K3=$f"; KB_K3=$f timeout 120 python tools/quickbench.py one 3 $n f32 $((1073741824 / (n*n*n*4))) 10; done
done
for n in 16 10; do for f in "" 14; do echo "K3=$f f64"; KB_K3=$f timeout 120 python tools/quickbench.py one 3 $n f64 $((1073741824 / (n*n*n*8))) 10; done; done
