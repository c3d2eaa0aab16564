# kernel (a): unroll 2 for one-lane groups (G = 1) vs 4; parity suites; cfg5 bench
mkdir -p gpurun_out/s88
timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_layout.py tests/test_gpu_small.py tests/test_gpu_schedule.py -m gpu -q -x -p no:cacheprovider > gpurun_out/s88/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/s88/pytest.log
for v in new g1u4 new g1u4; do
  if [ $v = new ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  timeout 300 python tools/bench_gather.py cfg5 cfg3 2>&1 | grep -E "^cfg" | sed "s|^|$v |" | python -c "
import sys,json
for l in sys.stdin:
    v,c,j=l.split(' ',2); d=json.loads(j); print(v,c,'%.4f ms'%d['gather_ms'],'%.0f GB/s'%d['GBps'],'%.3f'%d['hbm_frac'])"
done
unset MM_LIB_PATH
timeout 1500 python bench.py --config cfg5 --steps 2 --warmup 3 > gpurun_out/s88/bench_cfg5.json 2>/dev/null; echo cfg5 rc=$?
python -c "
import json; d=json.load(open('gpurun_out/s88/bench_cfg5.json')); r=d['roofline']; k=d['kernels']['gather_update']
print('cfg5 ms %.2f'%d['ms_per_step'], 'value %.4g'%d['value'], 'frac %.3f'%r['frac'], 'gather total ms %.2f'%k['total_ms'], k['launches'])"
