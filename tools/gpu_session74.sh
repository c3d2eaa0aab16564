# gather: 8 j-side partial rows in flight (symmetric mode)
mkdir -p gpurun_out/s74
timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_sym.py tests/test_gpu_layout.py -m gpu -q -x -p no:cacheprovider > gpurun_out/s74/pytest.log 2>&1; tail -2 gpurun_out/s74/pytest.log
for v in new prev new prev; do
  if [ $v = new ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s74/b_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/s74/b_$v.json')); sh=d['kernel_share_of_step']; ms=d['ms_per_step']
print('$v cfg2 ms %.3f'%ms, 'e2e %.4g'%d['e2e']['value'], {k: round(v*ms,3) for k,v in sorted(sh.items(), key=lambda kv:-kv[1])[:4]})"
done
