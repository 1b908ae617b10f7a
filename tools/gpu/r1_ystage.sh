# Y-staging check: GPU tests, size sweep with staging forced off / auto, launch overhead.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"
KB_YSTAGE=0 timeout 600 python tools/quickbench.py sweep > gpurun_out/sweep_ys0.txt 2>&1
timeout 600 python tools/quickbench.py sweep > gpurun_out/sweep_auto.txt 2>&1
KB_YSTAGE=1 timeout 300 python tools/quickbench.py main > gpurun_out/main_ys1.txt 2>&1
paste gpurun_out/sweep_ys0.txt gpurun_out/sweep_auto.txt | awk '{print $1,$2,$3,$7,$9,"->",$21,$23}'
cat gpurun_out/main_ys1.txt
timeout 120 python tools/launch_overhead.py 65536
