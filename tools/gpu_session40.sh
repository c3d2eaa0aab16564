# hierarchy: edge-parallel edge_keys / coarse_sset, grouped match_pick; bitwise tests + timing
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_hierarchy.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_h.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_h.log | tail -5
timeout 600 python tools/bench_hier.py cfg5 cfg4 cfg3 2>&1 | grep -v Warn | cut -c1-600
for g in 4 8 32; do echo "== MM_MATCH_G=$g"; MM_MATCH_G=$g timeout 600 python tools/bench_hier.py cfg5 cfg4 2>&1 | grep -o '^[a-z0-9 ]*\|"match_pick_ms": [0-9.]*\|"kernel_ms": [0-9.]*' | tr '\n' ' '; echo; done
