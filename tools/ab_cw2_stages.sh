# A/B: 2-D column-wise kernel with 3 (default) vs 4 smem stages (build/s4)
for lib in paper_1304_7054_b200 build/s4; do
  L=$PWD/$lib/libkronbatch_b200.so
  KB_LIB_PATH=$L timeout 120 python tools/launch_overhead.py 65536 | sed "s#^#$lib #"
  for cfg in "10 f32 4194304" "12 f32 4194304" "1 f32 268435456" "4 f32 33554432" "9 f64 3314017"; do
    set -- $cfg; KB_LIB_PATH=$L timeout 120 python tools/quickbench.py one 2 $1 $2 $3 10 | sed "s#^#$lib #"
  done
done
