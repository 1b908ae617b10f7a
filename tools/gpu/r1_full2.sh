mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 120 python tools/launch_overhead.py 65536
timeout 300 ./tools/kronbench/kronbench --resident --batch 65536 --reps 20 --sizes 10 --dims 2d --precision single --format csv
timeout 300 ./tools/kronbench/kronbench --batch 65536 --reps 20 --sizes 10 --dims 2d --precision single --format csv
timeout 600 ./tools/kronbench/kronbench --resident --batch 262144 --reps 5 --sizes 1..16 > gpurun_out/kronbench_all.txt 2>&1; cat gpurun_out/kronbench_all.txt
