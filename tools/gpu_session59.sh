timeout 900 python -m pytest tests/test_gpu_layout.py tests/test_gpu_schedule.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/bench_hier.py cfg5 cfg4 2>&1 | grep -v Warn | cut -c1-300
for a in "cfg2 7" "cfg3 7"; do timeout 200 python tools/sched_overhead.py $a 2>&1 | tail -2 | cut -c1-110; done
