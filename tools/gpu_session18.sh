mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|^E  " gpurun_out/pytest_gpu.log | tail -25
