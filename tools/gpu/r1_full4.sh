mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"
timeout 120 python tools/launch_overhead.py 65536
timeout 300 ./tools/kronbench/kronbench --resident --batch 65536 --reps 20 --sizes 10 --dims 2d --precision single --format csv
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json | head -c 600; echo
timeout 900 ./tools/kronbench/kronbench --resident --batch 1048576 --reps 5 --sizes 1..16 > gpurun_out/kronbench_1m.txt 2>&1; cat gpurun_out/kronbench_1m.txt
