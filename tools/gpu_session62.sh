# kernel (c) variants after Q26: targets per thread / unroll; ncu of the default on cfg3
mkdir -p gpurun_out/s62
for v in new t8 u2 u8 t8u2 t6 new; do
  if [ $v = new ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  c=cfg3
  timeout 300 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s62/b_${v}_$c.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/s62/b_${v}_$c.json')); r=d['roofline']
print('$v $c ms %.1f'%d['ms_per_step'], 'pairs/s %.4g'%r['pairs_per_s_kernel'], 'frac %.3f'%r['frac'], d['clocks'].get('sm_mhz'))"
done
for v in new t3_4 u8; do
  if [ $v = new ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  timeout 300 python bench.py --config cfg5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s62/b_${v}_cfg5.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/s62/b_${v}_cfg5.json')); r=d['roofline']
print('$v cfg5 ms %.1f'%d['ms_per_step'], 'pairs/s %.4g'%r['pairs_per_s_kernel'], 'frac %.3f'%r['frac'])"
done
unset MM_LIB_PATH
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_repulse -s 40 -c 1 -o gpurun_out/s62/prof_coarse_cfg3 python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s62/ncu.log 2>&1; echo ncu_rc=$?
