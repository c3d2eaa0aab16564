# kernel (a): FP64-quotient slot divisions (MM_FASTDIV) A/B + ncu --set full of the gather at cfg5
mkdir -p gpurun_out/s81
timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_sym.py -m gpu -q -x -p no:cacheprovider > gpurun_out/s81/pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/s81/pytest.log
for v in new slowdiv new slowdiv; do
  if [ $v = new ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  timeout 300 python tools/bench_gather.py cfg5 cfg4 cfg3 2>&1 | grep -E "^cfg" | sed "s|^|$v |" | python -c "
import sys,json
for l in sys.stdin:
    v,c,j=l.split(' ',2); d=json.loads(j); print(v,c,'%.4f ms'%d['gather_ms'],'%.0f GB/s'%d['GBps'],'%.3f'%d['hbm_frac'])"
done
unset MM_LIB_PATH
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather -s 3 -c 1 -o gpurun_out/s81/prof_r01_gather_cfg5 python tools/bench_gather.py cfg5 > gpurun_out/s81/ncu_g5.log 2>&1; echo ncu_rc=$?
