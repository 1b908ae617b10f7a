# configs[0] (2-D fp32 n = 10, 65,536 entries, 7 rotating sets): CUDA-graph time per launch by family / ring depth
for lib in "" build/var_s2/libkronbatch_b200.so; do for f in 0 1 2; do
KB_LIB_PATH=$lib KB_K2=$f timeout 300 python - <<'PY'
import os, sys
sys.path.insert(0, ".")
import torch, bench
import paper_1304_7054_b200 as kb
topo = bench.Topo([0], 1, 0)
ms = [bench.time_graph(kb, torch, topo, "kron2-f32-n10", 200, 7) for _ in range(3)]
print(f"lib={os.environ.get('KB_LIB_PATH') or 'main'} K2={os.environ['KB_K2']}: graph {min(ms)*1e3:.2f} us/launch (runs {[round(m*1e3,2) for m in ms]})", flush=True)
PY
done; done
