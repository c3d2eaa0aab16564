timeout 900 python -m pytest tests/test_gpu_small.py tests/test_gpu_schedule.py tests/test_gpu_layout.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for N in 8192 20000; do echo "== MM_SMALL_N=$N"; MM_SMALL_N=$N MM_TRACE=1 timeout 300 python tools/trace_levels.py cfg2 7 2>&1 | sed -n "/---- timed/,\$p" | grep level; done
for a in "cfg2 7" "cfg3 7"; do timeout 300 python tools/sched_overhead.py $a 2>&1 | tail -2 | cut -c1-120; done
timeout 300 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg1', d['ms_per_step'], d['e2e']['ms_per_step'], d['value'])"
