# full GPU suite + bench cfg2 + launch list (sym kernel, sub-tile units)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|chaos" gpurun_out/pytest_gpu.log | tail -6
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo bench_rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg2.json'))
r=d['roofline']; print('value %.4g'%d['value'], 'ms %.2f'%d['ms_per_step'], 'frac %.3f exec %.3f'%(r['frac'], r['executed_frac']), r['kernel_variant'], 'e2e', d['e2e']['ms_per_step'], 'clocks', d['clocks'], 'cpu', d['cpu_baseline']['value'])
print({k: round(v,4) for k,v in d['kernel_share_of_gpu_time'].items() if v > 0.002})"
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain.json 2>&1; echo plain_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu_rc=$?
