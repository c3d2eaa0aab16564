mkdir -p gpurun_out
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -2
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|chaos|Error" gpurun_out/pytest_gpu.log | tail -10
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo bench_rc=$?; tail -2 gpurun_out/bench7.err
for c in cfg2 cfg3 cfg5 cfg4; do
  if [ $c != cfg2 ]; then timeout 900 python bench.py --config $c --steps 1 --warmup 1 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_${c}_rc=$?; tail -2 gpurun_out/bench_$c.err; fi
  f=gpurun_out/bench_$c.json; [ $c = cfg2 ] && f=gpurun_out/bench7.json
  python -c "
import json; d=json.load(open('$f'))
print('$c', 'value %.4g'%d['value'], 'ms %.1f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], 'pairs/s %.4g'%d['roofline']['pairs_per_s_kernel'], 'pairs/step %.4g'%d['pair_interactions_per_step'], 'e2e ms %.1f'%d['e2e']['ms_per_step'], 'E', d['energy_last_step'])
print({k: round(v,4) for k,v in d['kernel_share_of_step'].items() if v > 0.002})"
done
