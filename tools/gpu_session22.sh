mkdir -p gpurun_out
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|^E  " gpurun_out/pytest_gpu.log | tail -10
SCLAP=1 timeout 900 python tools/bench_hier.py cfg5 cfg4 cfg3 2>&1 | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 2>&1 | tail -1 | cut -c1-600
