timeout 300 python tools/bench_one.py kron2-f32-n16 sleep1 kron3-f32-n16 kron2-f32-n16 sleep3 kron3-f32-n16 kron2-f32-n16 sleep6 kron3-f32-n16
