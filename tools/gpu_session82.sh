# kernel (a): next-vertex index prefetch (MM_GATHER_PREFETCH) A/B, parity suites for sweeps and layouts
mkdir -p gpurun_out/s82
timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_layout.py tests/test_gpu_small.py -m gpu -q -x -p no:cacheprovider > gpurun_out/s82/pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/s82/pytest.log
for v in new nopf new nopf; do
  if [ $v = new ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  timeout 300 python tools/bench_gather.py cfg5 cfg4 cfg3 cfg2 2>&1 | grep -E "^cfg" | sed "s|^|$v |" | python -c "
import sys,json
for l in sys.stdin:
    v,c,j=l.split(' ',2); d=json.loads(j); print(v,c,'%.4f ms'%d['gather_ms'],'%.0f GB/s'%d['GBps'],'%.3f'%d['hbm_frac'])"
done
unset MM_LIB_PATH
for c in cfg3 cfg5; do timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s82/b_$c.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/s82/b_$c.json')); print('$c ms %.2f'%d['ms_per_step'])"; done
