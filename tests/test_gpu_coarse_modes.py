"""-m gpu: kernel (c)'s optional paths against the oracle (Q27, Q28).

The library reads its switches once per process, so the Eq.(3) parity suite of
test_gpu_sweep.py is re-run in a subprocess per mode:
  MM_FAR_PAIRS=1      the far-tile path (frame origin, tile boxes, lo-free far tiles) at
                      every size (by default only when n k >= 1e9 pairs per sweep, so the
                      scaled cases of the default run take the plain hi/lo path);
  + MM_REORDER_PAIRS=1  re-sorts targets / representatives before every sweep
                      (by default only when n k >= 1e11, i.e. cfg4's finest level);
  MM_FAR_TILES=0      keeps the hi/lo differencing on every tile, full sizes included."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{"MM_FAR_PAIRS": "1"}, {"MM_FAR_PAIRS": "1", "MM_REORDER_PAIRS": "1"},
                                 {"MM_FAR_TILES": "0"}])
def test_approx_suite_per_mode(env):
    e = dict(os.environ, **env)
    cmd = [sys.executable, "-m", "pytest", "tests/test_gpu_sweep.py", "-m", "gpu", "-q", "-x",
           "-p", "no:cacheprovider", "-k", "approx or determinism"]
    r = subprocess.run(cmd, cwd=ROOT, env=e, capture_output=True, text=True, timeout=1200)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, f"{env}:\n{tail}"
    assert " passed" in r.stdout, tail
