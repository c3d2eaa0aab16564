mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|chaos" gpurun_out/pytest_gpu.log | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench9.json 2> gpurun_out/bench9.err; echo bench_rc=$?
for c in cfg2 cfg3 cfg4 cfg5; do
  if [ $c != cfg2 ]; then timeout 900 python bench.py --config $c --steps 1 --warmup 1 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_${c}_rc=$?; fi
  f=gpurun_out/bench_$c.json; [ $c = cfg2 ] && f=gpurun_out/bench9.json
  python -c "
import json; d=json.load(open('$f'))
print('$c', 'value %.4g'%d['value'], 'ms %.1f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], 'pairs/s %.4g'%d['roofline']['pairs_per_s_kernel'], 'e2e ms %.1f'%d['e2e']['ms_per_step'], 'E', d['energy_last_step'])
print({k: round(v,4) for k,v in d['kernel_share_of_gpu_time'].items() if v > 0.002})"
done
CMD3="python bench.py --config cfg3 --steps 1 --warmup 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_repulse -s 305 -c 1 -o gpurun_out/prof_r01_repulse_coarse $CMD3 > gpurun_out/ncu_c.log 2>&1; echo ncu_c_rc=$?
CMD5="python bench.py --config cfg5 --steps 1 --warmup 1"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_gather|k_centroid|k_repulse" -s 540 -c 3 -o gpurun_out/prof_r01_cfg5 $CMD5 > gpurun_out/ncu_5.log 2>&1; echo ncu_5_rc=$?
