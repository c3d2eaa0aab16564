# kernel (a) unroll / occupancy re-check with the prefetch and lane split
for v in new u2 u8 minb3 new u2 u8 minb3; do
  if [ $v = new ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  timeout 300 python tools/bench_gather.py cfg5 cfg4 cfg3 cfg2 2>&1 | grep -E "^cfg" | sed "s|^|$v |" | python -c "
import sys,json
for l in sys.stdin:
    v,c,j=l.split(' ',2); d=json.loads(j); print(v,c,'%.4f ms'%d['gather_ms'],'%.0f GB/s'%d['GBps'],'%.3f'%d['hbm_frac'])"
done
