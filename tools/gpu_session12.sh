mkdir -p gpurun_out
for ST in 0 1; do
 export MM_GATHER_STAGED=$ST
 for G in auto 1 2 4 8; do
  if [ $G = auto ]; then unset MM_GATHER_G; else export MM_GATHER_G=$G; fi
  timeout 600 python tools/bench_gather.py cfg5 cfg4 cfg3 cfg2 2>&1 | grep -E "^cfg" | sed "s/^/staged=$ST G=$G /" | python -c "
import sys, json
for l in sys.stdin:
    pre, js = l.split('{',1); d=json.loads('{'+js)
    print(pre, 'ms %.4f GB/s %.0f frac %.3f'%(d['gather_ms'], d['GBps'], d['hbm_frac']))"
 done
done
unset MM_GATHER_G MM_GATHER_STAGED
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu.log | tail -5
