mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu.log | tail -5
timeout 900 python tools/bench_hier.py cfg5 cfg4 cfg3 2>&1 | cut -c1-400
timeout 600 python tools/bench_gather.py cfg5 cfg4 cfg3 cfg2 2>&1 | grep "^cfg" | cut -c1-300
