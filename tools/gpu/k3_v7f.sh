for b in 50000 100000 200000 400000; do echo "n=8 b=$b"; KB_K3=14 timeout 60 python tools/quickbench.py one 3 8 f32 $b 3 2>&1 | tail -1; done
for b in 524288 1048576; do echo "n=16 b=$b"; KB_K3=14 timeout 60 python tools/quickbench.py one 3 16 f32 $b 3 2>&1 | tail -1; done
for b in 1000000 3000000; do echo "n=12 b=$b"; KB_K3=14 timeout 60 python tools/quickbench.py one 3 12 f32 $b 3 2>&1 | tail -1; done
for b in 2000000 8000000; do echo "n=6 b=$b"; KB_K3=14 timeout 60 python tools/quickbench.py one 3 6 f32 $b 3 2>&1 | tail -1; done
