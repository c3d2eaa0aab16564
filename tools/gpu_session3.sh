mkdir -p gpurun_out
timeout 300 python tools/debug_approx.py cfg3_mesh128 3 > gpurun_out/debug3.log 2>&1; cat gpurun_out/debug3.log | tail -30
timeout 300 python tools/debug_approx.py cfg3_mesh128 2 2>&1 | head -3
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -20
