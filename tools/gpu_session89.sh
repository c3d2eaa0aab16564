# kernel (a): S rows evict-first (default) vs normal loads (L2 retention across sweeps)
mkdir -p gpurun_out/s89
for v in new sload new sload; do
  if [ $v = new ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  timeout 300 python tools/bench_gather.py cfg5 cfg4 cfg3 cfg2 2>&1 | grep -E "^cfg" | sed "s|^|$v |" | python -c "
import sys,json
for l in sys.stdin:
    v,c,j=l.split(' ',2); d=json.loads(j); print(v,c,'%.4f ms'%d['gather_ms'],'%.0f GB/s'%d['GBps'],'%.3f'%d['hbm_frac'])"
  for c in cfg3 cfg2; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s89/b_${v}_$c.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/s89/b_${v}_$c.json')); k=d['kernels']['gather_update']
print('$v $c ms/step %.3f'%d['ms_per_step'], 'gather total ms %.3f'%k['total_ms'], k['launches'])"; done
done
