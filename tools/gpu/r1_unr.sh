mkdir -p gpurun_out
KB_LIB_PATH=$PWD/build/alt4/libkronbatch_b200.so KB_K3=3 python tests/variant_check.py
for lib in paper_1304_7054_b200/libkronbatch_b200.so build/alt4/libkronbatch_b200.so; do
for f in 1 2 3; do
  for cfg in "16 f32 262144" "14 f32 262144" "12 f32 262144" "10 f32 262144" "16 f64 131072" "12 f64 131072" "10 f64 262144"; do
    set -- $cfg; KB_LIB_PATH=$PWD/$lib KB_K3=$f timeout 120 python tools/quickbench.py one 3 $1 $2 $3 10 2>&1 | sed "s#^#$(basename $(dirname $lib)) K3=$f #"
  done
done
done
