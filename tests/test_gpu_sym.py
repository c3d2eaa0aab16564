"""-m gpu: both implementations of kernel (b) against the oracle.

Exact sweeps use the symmetric kernel (each unordered pair evaluated once and
applied to both vertices) when the triangular schedule is large
enough (n >~ 60K at 148 SMs), else the one-sided kernel.  The library reads
MM_SYM once per process, so the exact-sweep parity suite of
test_gpu_sweep.py is re-run in a subprocess with each kernel forced:
MM_SYM=2 (symmetric at every size: TB = 1, ragged tail chunks, 3-D, q > 0)
and MM_SYM=0 (one-sided, including the full-size cfg2 case)."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("mode", ["2", "0"])
def test_exact_suite_per_kernel(mode):
    env = dict(os.environ, MM_SYM=mode)
    cmd = [sys.executable, "-m", "pytest", "tests/test_gpu_sweep.py", "-m", "gpu", "-q", "-x",
           "-p", "no:cacheprovider", "-k", "exact or ring or determinism or translation or orbit"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, f"MM_SYM={mode}:\n{tail}"
    assert " passed" in r.stdout, tail
