"""One gemm_a square timing point (profiling aid): python tools/ga_one.py <n> <f32|f64> <N|T>."""
import runpy
import sys

qb = runpy.run_path(__file__.rsplit("/", 1)[0] + "/quickbench.py")
qb["bench_gemm_a"](int(sys.argv[1]), sys.argv[2], sys.argv[3], reps=1)
