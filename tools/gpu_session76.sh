# 2-D coarse kernel occupancy variants (MINB 3 -> <= 85 regs, 3 CTAs/SM)
mkdir -p gpurun_out/s76
for v in new m3 m3u2 u2 m3t2 new; do
  if [ $v = new ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  timeout 600 python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s76/b_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/s76/b_$v.json')); r=d['roofline']
print('$v cfg3 ms %.2f'%d['ms_per_step'], 'pairs/s %.4g'%r['pairs_per_s_kernel'])"
done
