# Round profiling: tests, bench, reference arm, ncu launch list of the bench
# command, full ncu (+ source) of the default kernel of each bench workload.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>&1; cat gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu --no-extra > gpurun_out/bench_under_ncu.log 2>&1
P="ncu --set full --clock-control none --import-source on -s 3 -c 1"
timeout 300 $P -k regex:kron2_ -o gpurun_out/prof_kron2_f32_n16 python tools/quickbench.py one 2 16 f32 4194304 1 > /dev/null 2>&1
timeout 300 $P -k regex:kron3_ -o gpurun_out/prof_kron3_f32_n16 python tools/quickbench.py one 3 16 f32 262144 1 > /dev/null 2>&1
timeout 300 $P -k regex:kron3_ -o gpurun_out/prof_kron3_f64_n16 python tools/quickbench.py one 3 16 f64 131072 1 > /dev/null 2>&1
timeout 300 $P -k regex:kron3_ -o gpurun_out/prof_kron3_f32_n10 python tools/quickbench.py one 3 10 f32 262144 1 > /dev/null 2>&1
timeout 300 $P -k regex:kron2_ -o gpurun_out/prof_kron2_f32_n10 python tools/quickbench.py one 2 10 f32 65536 1 > /dev/null 2>&1
ls -la gpurun_out
