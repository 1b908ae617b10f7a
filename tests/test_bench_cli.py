"""bench.py's host-side logic (no GPU): the multi-GPU batch split (weak /
strong scaling) and the refusal to report GPUs that did not run."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


@pytest.mark.parametrize("world, parts", [(1, 1), (1, 3), (2, 1), (4, 2), (8, 1)])
def test_strong_scaling_parts_tile_the_fixed_batch(world, parts):
    batch = bench.WORKLOADS["kron3-f64-n16"][3]
    assert bench.WORKLOADS["kron3-f64-n16"][4] == "strong"  # configs[3]: fixed batch over 1/2/4/8 GPUs
    total = 0
    for rank in range(world):
        topo = bench.Topo([0] * parts, world, rank)
        for i in range(parts):
            total += bench.part_batch(topo, "strong", batch, i)
    assert total == batch


def test_weak_scaling_parts_keep_the_per_gpu_batch():
    topo = bench.Topo([0, 1, 2], 1, 0)
    assert [bench.part_batch(topo, "weak", 4194304, i) for i in range(3)] == [4194304] * 3


def test_single_process_topology_counts_distinct_devices():
    assert bench.Topo([0, 0], 1, 0).n_gpus == 1
    assert bench.Topo([0, 1, 2, 3], 1, 0).n_gpus == 4


def test_refuses_more_gpus_than_visible():
    import torch

    if torch.cuda.device_count() >= 64:
        pytest.skip("machine with >= 64 GPUs")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "64", "--no-cpu"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert "CUDA device(s) visible" in line["error"]
