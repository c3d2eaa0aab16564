# kernel (a) with TMA-staged S stream: parity + timing vs direct loads
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_layout.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_g.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_g.log | tail -5
for t in 1 0; do echo "== MM_GATHER_TMA=$t"; MM_GATHER_TMA=$t timeout 600 python tools/bench_gather.py cfg5 cfg4 cfg3 cfg2 2>&1 | grep -o '^cfg[0-9] .*"GBps": [0-9.]*' | sed 's/{.*"gather_ms"/ms/'; done
