"""The reference's OWN acceptance binary on B200 (drop-in proof).

oracle/_ref/acceptance is /root/reference/proj/tests/acceptance.cpp,
tools/bench_support.cpp and src/reference.cpp compiled UNMODIFIED against this
repo's drop-in headers (include/kronbatch/*.hpp -> libkronbatch_b200.so); only
the reference's brute-force oracle header is taken from the reference tree
(oracle/Makefile `accept`). Its seven criteria (acceptance.cpp:1169-1196):
C1 oracle equivalence n = 1..16 x 22 op combos x both precisions (:82-339),
C2 50 rectangular tuples (:345-534), C3 kron3 == kron2 + gemm_a composition
(:540-641), C4 flop model (:647-659), C5 affine / NaN / padding / determinism
(:782-989), C6 the bench CSV -- driven through tools/kronbench as
KRONBATCH_BENCH (:1003-1084), C7 fused kron2 >= the unfused two-GEMM CPU
baseline at n = 16 double (:1104-1165).
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ACCEPT = os.path.join(ROOT, "oracle", "_ref", "acceptance")
BENCH = os.path.join(ROOT, "tools", "kronbench", "kronbench")

needs_bin = pytest.mark.skipif(not os.path.exists(ACCEPT), reason="oracle/_ref/acceptance not built (make accept)")


@needs_bin
def test_acceptance_binary_calls_the_b200_library():
    """The kron2/kron3/kron1/gemm_a calls in the reference's acceptance code
    resolve to the C ABI of libkronbatch_b200.so (undefined symbols bound at
    load time), not to the reference's CPU templates."""
    out = subprocess.run(["nm", "-D", ACCEPT], capture_output=True, text=True).stdout
    und = {ln.split()[-1] for ln in out.splitlines() if " U " in ln}
    assert {"kb_skron2", "kb_dkron2", "kb_skron3", "kb_dkron3", "kb_sgemm_a", "kb_dgemm_a"} <= und
    ldd = subprocess.run(["ldd", ACCEPT], capture_output=True, text=True).stdout
    assert "libkronbatch_b200.so" in ldd


@needs_bin
@pytest.mark.gpu
def test_reference_acceptance_all_criteria_pass_on_b200():
    env = dict(os.environ, KRONBATCH_BENCH=BENCH)
    r = subprocess.run([ACCEPT], capture_output=True, text=True, timeout=2400, env=env, cwd=ROOT)
    print(r.stdout)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("criterion")]
    assert len(lines) == 7, r.stdout + r.stderr[-2000:]
    for ln in lines:
        assert ": pass" in ln, ln
    assert r.returncode == 0
