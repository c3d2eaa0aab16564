for a in "cfg2 7" "cfg3 7" "cfg4 7"; do timeout 300 python tools/sched_overhead.py $a 2>&1 | tail -2 | cut -c1-150; done
timeout 300 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg1', d['ms_per_step'], d['e2e']['ms_per_step'], d['value'])"
MM_TRACE=1 timeout 300 python tools/trace_levels.py cfg2 7 2>&1 | sed -n "/---- timed/,\$p" | head -14
