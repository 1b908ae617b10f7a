mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 ./tools/kronbench/kronbench --resident --batch 262144 --reps 5 --sizes 1..16 --dims 3d > gpurun_out/kronbench_3d.txt 2>&1; cat gpurun_out/kronbench_3d.txt
