"""compute-sanitizer over one small call of every kernel family (-m gpu).

SURVEY.md §5: the reference has no sanitizers (proj/CMakeLists.txt:1-52), but
the sm_100a kernels double-buffer shared memory behind mbarriers and bulk
(TMA) copies, so memcheck (out-of-bounds / misaligned accesses -- including
the odd-n group spans, which must not read past the batch), racecheck
(shared-memory hazards) and synccheck (barrier misuse) run over
tools/sanitize/kb_sanitize.cpp: every square size n = 1..16 in fp32/fp64 for
2-D (op_x N and T) and 3-D, the generic, scale, kron1, gemm_a and 3xTF32
tensor-core kernels, on exactly-sized device buffers.
"""
import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(ROOT, "build", "sanitize", "kb_sanitize")
CS = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


def _run(tool, mode, timeout):
    if not os.path.exists(DRIVER):
        pytest.skip("build/sanitize/kb_sanitize not built (make sanitize)")
    cmd = [CS, "--tool", tool, "--error-exitcode", "97", "--print-limit", "20"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    cmd += [DRIVER, mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    out = r.stdout + r.stderr
    logdir = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(logdir):  # keep the full report next to the GPU run's other outputs
        with open(os.path.join(logdir, f"sanitize_{tool}.log"), "w") as f:
            f.write(out)
    assert r.returncode == 0, out[-4000:]
    assert ("ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out), out[-4000:]
    assert "0 failures" in out, out[-4000:]
    return out


def test_memcheck_every_kernel_family():
    _run("memcheck", "full", 1500)


def test_racecheck_kernel_families():
    _run("racecheck", "full", 2400)


def test_synccheck_kernel_families():
    _run("synccheck", "full", 1500)
