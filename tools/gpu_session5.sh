mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|chaos" gpurun_out/pytest_gpu.log | tail -10
for c in cfg3 cfg5 cfg4; do
  timeout 900 python bench.py --config $c --steps 1 --warmup 1 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_${c}_rc=$?; tail -2 gpurun_out/bench_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json'))
print('$c', 'value %.4g'%d['value'], 'ms %.1f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], 'pairs/s %.4g'%d['roofline']['pairs_per_s_kernel'], 'pairs/step %.4g'%d['pair_interactions_per_step'], 'e2e ms %.1f'%d['e2e']['ms_per_step'])
print({k: round(v,4) for k,v in d['kernel_share_of_step'].items()}); print(d['levels'], d['k_levels'])"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_repulse -s 8 -c 1 -o gpurun_out/prof_repulse_exact python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu_full_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_repulseILi2ELb0ELb1" -s 4 -c 1 -o gpurun_out/prof_repulse_coarse python bench.py --config cfg3 --steps 1 --warmup 1 > gpurun_out/ncu_full2.log 2>&1; echo ncu_full2_rc=$?
tail -2 gpurun_out/ncu_full2.log
