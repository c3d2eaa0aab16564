# full suite + all bench lines + schedule timings after the small-level kernel
mkdir -p gpurun_out/r01_bench
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|chaos" gpurun_out/pytest_gpu.log | tail -6
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r01_bench/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo cfg2_rc=$?
timeout 300 python bench.py --config cfg1 --steps 5 --warmup 3 > gpurun_out/r01_bench/bench_cfg1.json 2>/dev/null; echo cfg1_rc=$?
for c in cfg3 cfg4 cfg5; do timeout 900 python bench.py --config $c --steps 1 --warmup 1 > gpurun_out/r01_bench/bench_$c.json 2>/dev/null; echo ${c}_rc=$?; done
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do python -c "
import json; d=json.load(open('gpurun_out/r01_bench/bench_$c.json')); r=d['roofline']
print('$c', 'value %.4g'%d['value'], 'ms %.2f'%d['ms_per_step'], r['kernel'], 'pairs/s %.4g'%r['pairs_per_s_kernel'], 'frac %.3f'%r['frac'], 'e2e ms %.2f'%d['e2e']['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'], 'cpu', (d['cpu_baseline'] or {}).get('value'))"; done
