# hierarchy: heavy-row matching path; bitwise tests + timing (matching and SCLaP)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_hierarchy.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_h.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_h.log | tail -5
timeout 600 python tools/bench_hier.py cfg5 cfg4 cfg3 2>&1 | grep -v Warn | cut -c1-700
SCLAP=1 timeout 600 python tools/bench_hier.py cfg5 cfg4 cfg3 2>&1 | grep -v Warn | cut -c1-700
