mkdir -p gpurun_out
L=$PWD/build/var/libkronbatch_b200.so
for f in 3 4 5 6 7 8; do KB_LIB_PATH=$L KB_K3=$f timeout 120 python tools/quickbench.py one 3 16 f32 262144 10 | sed "s/^/K3=$f /"; done
for f in 1 2 4 5 7 8; do KB_LIB_PATH=$L KB_K3=$f timeout 120 python tools/quickbench.py one 3 16 f64 131072 10 | sed "s/^/K3=$f /"; done
KB_LIB_PATH=$L KB_K3=4 python tests/variant_check.py; KB_LIB_PATH=$L KB_K3=8 python tests/variant_check.py
