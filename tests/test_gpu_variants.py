"""Kernel-selection switches that are not the default for every size must stay
bit-exact too: Y staged through shared memory (KB_YSTAGE=1) and direct R-row
stores (KB_YSTAGE=0); the 3-D kernel families (KB_K3=0 row-owner, 1/2
column-wise double/single stage, 3 128-thread tiles, 9 tiny-entry, 10 one row per
task, 11 one entry per CTA, 13 warp-plane, 14 two groups per CTA on a 3-stage ring), the
odd-n 3-D Y image off / on for every size (KB_YS), static tile order (KB_DYN=0) and
plain launches without programmatic dependent launch (KB_PDL=0), no first-group L2 prefetch (KB_L2PF=0) -- every square n,
2-D/3-D, fp32/fp64 (-m gpu)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("env", [{"KB_YSTAGE": "1"}, {"KB_YSTAGE": "0"}] + [{"KB_K3": str(f)} for f in (0, 1, 2, 3, 9, 10, 11, 13, 14)] + [{"KB_K2": str(f)} for f in range(3)]
                         + [{"KB_YS": "0"}, {"KB_YS": "1"}, {"KB_DYN": "0"}, {"KB_PDL": "0"}, {"KB_L2PF": "0"}],
                         ids=lambda e: "_".join(f"{k[3:]}-{v}" for k, v in e.items()))
def test_kernel_switches_bitwise(env):
    r = subprocess.run([sys.executable, os.path.join(HERE, "variant_check.py")], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("warp", ["0", "1"])
def test_gemm_a_square_kernels_both(warp):
    """Both square gemm_a kernels (CTA tile / warp-granular, KB_GA_WARP) stay bit-exact vs the oracle."""
    env = dict(os.environ, KB_GA_WARP=warp)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu",
                        os.path.join(HERE, "test_gpu_blas.py"), "-k", "gemm_a"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
