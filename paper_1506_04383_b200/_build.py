"""Build libmm_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libmm_b200.so")
BUILD = os.path.join(HERE, "csrc", "build")
SOURCES = ["k_repulse.cu", "k_gather.cu", "k_hier.cu", "k_fullstress.cu", "k_sclap.cu", "k_small.cu", "k_perm.cu", "k_sort.cu", "api.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include"),
         # host code: an uninitialised status on an error path is a build error
         "-Xcompiler", "-Wmaybe-uninitialized", "-Xcompiler", "-Werror=maybe-uninitialized"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh"))]
    deps.append(os.path.join(ROOT, "include", "mm.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = None, extra=()) -> str:
    """Build libmm_b200.so (or `out` with `extra` nvcc flags, for experiments)."""
    lib = out or LIB
    if not force and out is None and not extra and not _stale():
        return LIB
    bdir = BUILD if out is None else out + ".objs"
    os.makedirs(bdir, exist_ok=True)
    procs = []
    objs = []
    for src in SOURCES:
        obj = os.path.join(bdir, src.replace(".cu", ".o"))
        objs.append(obj)
        cmd = [NVCC, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = False
    for cmd, p in procs:
        log, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(log.decode(errors="replace"))
        if p.returncode != 0:
            failed = True
            sys.stderr.write("FAILED: " + " ".join(cmd) + "\n")
    if failed:
        raise RuntimeError("nvcc failed")
    tmp = lib + ".tmp"
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-o", tmp, *objs,
            "-Xlinker", "--exclude-libs,ALL"]
    subprocess.check_call(link)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if a not in ("--force", "-v")]
    out = None
    if args and args[0] == "--out":
        out, args = os.path.abspath(args[1]), args[2:]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=out, extra=args))
