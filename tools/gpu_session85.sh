# kernel (a) after the symmetric kernel: partial slots / j-side rows split over the group's lanes, G >= GMIN; A/B GMIN
mkdir -p gpurun_out/s85
timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_sym.py tests/test_gpu_layout.py -m gpu -q -x -p no:cacheprovider > gpurun_out/s85/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/s85/pytest.log
for v in new sg2 sg4 sg16 new sg2 sg4 sg16; do
  if [ $v = new ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s85/b_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/s85/b_$v.json')); k=d['kernels']['gather_update']
print('$v ms/step %.3f'%d['ms_per_step'], 'gather us %.2f'%(1e3*k['total_ms']/k['launches']), 'e2e %.4g'%d['e2e']['value'])"
done
unset MM_LIB_PATH
timeout 300 python tools/bench_gather.py cfg5 cfg4 cfg3 2>&1 | grep -E "^cfg" | python -c "
import sys,json
for l in sys.stdin:
    c,j=l.split(' ',1); d=json.loads(j); print(c,'%.4f ms'%d['gather_ms'],'%.0f GB/s'%d['GBps'],'%.3f'%d['hbm_frac'])"
