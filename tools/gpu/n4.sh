for f in -1 0 1 2 3 9 10 11; do echo "3d f32 n=4 K3=$f: $(KB_K3=$f timeout 60 python tools/quickbench.py one 3 4 f32 4194304 10 2>&1 | tail -1)"; done
for f in -1 0 1 2 3 9; do echo "3d f32 n=3 K3=$f: $(KB_K3=$f timeout 60 python tools/quickbench.py one 3 3 f32 9942054 10 2>&1 | tail -1)"; done
for f in -1 0 1 2 3 9; do echo "3d f64 n=3 K3=$f: $(KB_K3=$f timeout 60 python tools/quickbench.py one 3 3 f64 4971027 10 2>&1 | tail -1)"; done
for f in -1 0 1 2 3 10 11; do echo "3d f32 n=6 K3=$f: $(KB_K3=$f timeout 60 python tools/quickbench.py one 3 6 f32 1242757 10 2>&1 | tail -1)"; done
for f in -1 0 1 2 3 13; do echo "3d f32 n=7 K3=$f: $(KB_K3=$f timeout 60 python tools/quickbench.py one 3 7 f32 782611 10 2>&1 | tail -1)"; done
