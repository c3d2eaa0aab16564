# mass-ordered representatives (Q26): parity + A/B of kernel (c)
mkdir -p gpurun_out/s61
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s61/pytest.log 2>&1; tail -3 gpurun_out/s61/pytest.log
for v in old new old new; do
  if [ $v = new ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  for c in cfg3 cfg4; do
    timeout 300 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s61/b_${v}_$c.json 2>/dev/null
    python -c "
import json,sys; d=json.load(open('gpurun_out/s61/b_${v}_$c.json')); r=d['roofline']
print('$v $c ms %.1f'%d['ms_per_step'], 'pairs/s %.4g'%r['pairs_per_s_kernel'], 'frac %.3f'%r['frac'], d['clocks'].get('sm_mhz'))"
  done
done
unset MM_LIB_PATH
timeout 300 python bench.py --config cfg5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s61/b_new_cfg5.json 2>/dev/null
python -c "
import json,sys; d=json.load(open('gpurun_out/s61/b_new_cfg5.json')); r=d['roofline']
print('new cfg5 ms %.1f'%d['ms_per_step'], 'pairs/s %.4g'%r['pairs_per_s_kernel'], 'frac %.3f'%r['frac'])"
