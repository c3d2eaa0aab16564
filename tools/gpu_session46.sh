# device-driven schedule loop (conditional WHILE/IF graph per level): parity + timing
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_schedule.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_s.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|Error|error" gpurun_out/pytest_s.log | tail -6
for a in "cfg2 7" "cfg2 0" "cfg3 7" "cfg4 7"; do timeout 300 python tools/sched_overhead.py $a 2>&1 | tail -2 | cut -c1-200; done
echo "== host loop"
for a in "cfg2 7" "cfg3 7"; do MM_SCHED_GRAPH=0 timeout 300 python tools/sched_overhead.py $a 2>&1 | tail -2 | cut -c1-200; done
