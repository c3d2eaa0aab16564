# cached schedule graphs: full GPU suite + timing
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|chaos" gpurun_out/pytest_gpu.log | tail -6
for a in "cfg2 7" "cfg2 0" "cfg3 7" "cfg4 7"; do timeout 300 python tools/sched_overhead.py $a 2>&1 | tail -2 | cut -c1-150; done
timeout 600 python bench.py --schedule --h 7 --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sched bench', d['ms_per_step'], d['gpu_launches'], d['value'])"
