mkdir -p gpurun_out
timeout 300 ./tools/ubench_repulse 65428 2>&1 | tee gpurun_out/ubench_repulse.txt
timeout 300 ./tools/ubench_repulse 262144 2>&1 | tail -18 | tee gpurun_out/ubench_repulse_262k.txt
for c in cfg3 cfg5 cfg4; do
  timeout 900 python bench.py --config $c --steps 1 --warmup 1 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_${c}_rc=$?; tail -2 gpurun_out/bench_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json'))
print('$c', 'value %.4g'%d['value'], 'ms %.1f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], 'pairs/s %.4g'%d['roofline']['pairs_per_s_kernel'], 'pairs/step %.4g'%d['pair_interactions_per_step'], 'e2e ms %.1f'%d['e2e']['ms_per_step'])
print({k: round(v,4) for k,v in d['kernel_share_of_step'].items()}); print(d['levels'], d['k_levels'])"
done
