mkdir -p gpurun_out
for L in tools/gvar/*.so; do
  MM_LIB_PATH=$L timeout 600 python tools/bench_gather.py cfg5 cfg4 cfg3 2>&1 | grep -E "^cfg" | sed "s|^|$(basename $L) |" | python -c "
import sys, json
for l in sys.stdin:
    pre, js = l.split('{',1); d=json.loads('{'+js)
    print(pre, 'ms %.4f GB/s %.0f frac %.3f'%(d['gather_ms'], d['GBps'], d['hbm_frac']))"
done
timeout 900 python tools/bench_hier.py cfg5 cfg4 cfg3 2>&1 | tee gpurun_out/bench_hier.txt | cut -c1-600
