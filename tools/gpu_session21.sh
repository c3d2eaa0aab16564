mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|^E  " gpurun_out/pytest_gpu.log | tail -10
timeout 300 python tools/sanitize_case.py > gpurun_out/san_plain.log 2>&1 && \
timeout 900 compute-sanitizer --tool memcheck --leak-check full python tools/sanitize_case.py > gpurun_out/memcheck.log 2>&1; echo memcheck_rc=$?
grep -E "ERROR SUMMARY|sanitize case ok|Invalid|leak" gpurun_out/memcheck.log | head -20
