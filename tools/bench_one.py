"""Time bench.py workloads exactly as bench.py does, in order (development aid):
    python tools/bench_one.py kron2-f32-n16 kron3-f32-n16 ..."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import bench  # noqa: E402
import paper_1304_7054_b200 as kb  # noqa: E402

topo = bench.Topo([0], 1, 0)
import time

for name in sys.argv[1:]:
    if name.startswith("sleep"):
        time.sleep(float(name[5:]))
        continue
    with bench.ClockSampler([0]) as clk:
        ms, launch_ms, launches, path, entries = bench.time_device(kb, torch, topo, name, 25, 5)
    d3, n, dt, b, sc = bench.WORKLOADS[name]
    print(f"{name}: {ms:.4f} ms/step, per-launch {launch_ms:.4f} ms, "
          f"{bench.flops_per_entry(d3, n) * b / (launch_ms * 1e-3) / 1e12:.1f} TF/s, path {path}, clocks {clk.summary()}",
          flush=True)
