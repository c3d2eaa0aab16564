"""The C-ABI from plain C: examples/c_abi_ring.c links libmm_b200.so with no
Python or torch in the process, runs one exact sweep of the ring C_n against
the closed form of pin P3 and mm_energy on the 3-path worked
example.  CPU: the program builds, loads the library and fails cleanly
without a device.  GPU: it passes."""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "examples", "c_abi_ring")


@pytest.fixture(scope="module")
def exe():
    import __graft_entry__ as g

    g.build_c_example()
    return EXE


def test_c_example_builds_and_loads(exe):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu test")
    r = subprocess.run([exe, "64", "0"], capture_output=True, text=True, timeout=60)
    assert "mm_b200" in r.stdout  # the library loaded and answered mm_version()
    assert r.returncode == 2, (r.returncode, r.stdout, r.stderr)  # no device: clean failure


@pytest.mark.gpu
@pytest.mark.parametrize("n,q", [(65536, "0"), (4099, "0.8"), (1000, "0")])
def test_c_example_ring(exe, n, q):
    r = subprocess.run([exe, str(n), q], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.stdout, r.stderr)
    assert r.stdout.count("PASS") == 2, r.stdout
