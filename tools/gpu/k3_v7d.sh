for n in 8 16; do KB_K3=14 timeout 600 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 4 python tools/quickbench.py one 3 $n f32 3000 1 2>&1 | grep -v "Host Frame" | grep -v "^$" | head -24; done
for n in 8 16; do KB_K3=14 timeout 600 compute-sanitizer --tool synccheck --print-limit 4 python tools/quickbench.py one 3 $n f32 3000 1 2>&1 | grep -v "Host Frame" | grep -v "^$" | head -12; done
for i in 1 2 3; do KB_K3=14 timeout 120 python tools/quickbench.py one 3 8 f32 524288 10 2>&1 | tail -1; done
KB_K3=14 CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/quickbench.py one 3 8 f32 524288 3 2>&1 | tail -3
