# concurrency: threads calling layouts / hierarchy builds at once (with and without the state lock);
# gather occupancy variants; full GPU suite; headline bench
mkdir -p gpurun_out/s83
export MM_LIB_PATH=$PWD/tools/gvar/nolock.so
timeout 180 python -m pytest tests/test_gpu_layout.py -k concurrent -m gpu -q -x -p no:cacheprovider > gpurun_out/s83/nolock.log 2>&1; echo nolock rc=$?; tail -5 gpurun_out/s83/nolock.log | cut -c1-300
unset MM_LIB_PATH
timeout 300 python -m pytest tests/test_gpu_layout.py -k concurrent -m gpu -q -x -p no:cacheprovider > gpurun_out/s83/lock.log 2>&1; echo lock rc=$?; tail -2 gpurun_out/s83/lock.log
for v in new minb5 minb6; do
  if [ $v = new ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  timeout 300 python tools/bench_gather.py cfg5 cfg4 cfg3 2>&1 | grep -E "^cfg" | sed "s|^|$v |" | python -c "
import sys,json
for l in sys.stdin:
    v,c,j=l.split(' ',2); d=json.loads(j); print(v,c,'%.4f ms'%d['gather_ms'],'%.0f GB/s'%d['GBps'],'%.3f'%d['hbm_frac'])"
done
unset MM_LIB_PATH
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/s83/pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/s83/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/s83/bench_cfg2.json 2> gpurun_out/s83/e2.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/s83/bench_cfg2.json')); r=d['roofline']
print('cfg2 ms %.2f'%d['ms_per_step'], 'value %.4g'%d['value'], 'frac %.3f'%r['frac'], 'e2e %.4g'%d['e2e']['value'], d['clocks'])"
