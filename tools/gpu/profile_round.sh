# Round profiling (PART=A / PART=B runs half, so each call stays under the 64 MiB gpurun_out limit): ncu launch list of the bench command, full ncu (+ source) of
# the default kernel of each bench workload, the odd-n / tensor-core kernels.
set -x
mkdir -p gpurun_out
[ "${PART:-AB}" != "${PART/A/}" ] && timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu > gpurun_out/bench_under_ncu.log 2>&1
P="ncu --set full --clock-control none --import-source on -s 3 -c 1"
[ "${PART:-AB}" != "${PART/A/}" ] && timeout 300 $P -k regex:kron2_ -o gpurun_out/prof_kron2_f32_n16 python tools/quickbench.py one 2 16 f32 4194304 1 > /dev/null 2>&1
[ "${PART:-AB}" != "${PART/A/}" ] && timeout 300 $P -k regex:kron3_ -o gpurun_out/prof_kron3_f32_n16 python tools/quickbench.py one 3 16 f32 262144 1 > /dev/null 2>&1
[ "${PART:-AB}" != "${PART/A/}" ] && timeout 300 $P -k regex:kron3_ -o gpurun_out/prof_kron3_f64_n16 python tools/quickbench.py one 3 16 f64 131072 1 > /dev/null 2>&1
[ "${PART:-AB}" != "${PART/A/}" ] && timeout 300 $P -k regex:kron3_ -o gpurun_out/prof_kron3_f32_n10 python tools/quickbench.py one 3 10 f32 262144 1 > /dev/null 2>&1
[ "${PART:-AB}" != "${PART/A/}" ] && timeout 300 $P -k regex:kron2_ -o gpurun_out/prof_kron2_f32_n10 python tools/quickbench.py one 2 10 f32 65536 1 > /dev/null 2>&1
[ "${PART:-AB}" != "${PART/B/}" ] && timeout 300 $P -k regex:kron3_ -o gpurun_out/prof_kron3_f32_n9 python tools/quickbench.py one 3 9 f32 368225 1 > /dev/null 2>&1
[ "${PART:-AB}" != "${PART/B/}" ] && timeout 300 $P -k regex:kron3_ -o gpurun_out/prof_kron3_f32_n15 python tools/quickbench.py one 3 15 f32 79537 1 > /dev/null 2>&1
[ "${PART:-AB}" != "${PART/B/}" ] && timeout 300 $P -k regex:kron2_ -o gpurun_out/prof_kron2_f32_n15 python tools/quickbench.py one 2 15 f32 1193047 1 > /dev/null 2>&1
[ "${PART:-AB}" != "${PART/B/}" ] && timeout 300 $P -k regex:kron2_ -o gpurun_out/prof_kron2_f32_n13 python tools/quickbench.py one 2 13 f32 1588376 1 > /dev/null 2>&1
[ "${PART:-AB}" != "${PART/B/}" ] && timeout 300 $P -k regex:kron3_ -o gpurun_out/prof_kron3_f32_n13 python tools/quickbench.py one 3 13 f32 122183 1 > /dev/null 2>&1
[ "${PART:-AB}" != "${PART/B/}" ] && timeout 300 $P -k regex:kron3_tc -o gpurun_out/prof_kron3tc_f32_n16 env KB_TF32=1 KB_TC_WGS=5 python tools/quickbench.py one 3 16 f32 262144 1 > /dev/null 2>&1
ls -la gpurun_out
