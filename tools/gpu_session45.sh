# kernel (d) centroid with G lanes per representative: parity + timing
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_schedule.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_c.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_c.log | tail -3
timeout 600 python tools/bench_centroid.py cfg5 cfg4 cfg3 2>&1 | grep "^cfg"
for a in "cfg2 7" "cfg3 7" "cfg4 7"; do timeout 300 python tools/sched_overhead.py $a 2>&1 | tail -2 | cut -c1-300; done
