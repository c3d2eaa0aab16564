# kernel (c): hi-only fast pass with tau test + per-tile lo redo vs lo always
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_layout.py tests/test_gpu_schedule.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_c.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|Error|chaos" gpurun_out/pytest_c.log | tail -8
for v in default loalways; do
  if [ $v = default ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  for c in cfg3 cfg4; do
    timeout 900 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bc_${v}_$c.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/bc_${v}_$c.json')); r=d['roofline']
print('$v $c', 'ms %.1f'%d['ms_per_step'], 'coarse pairs/s %.4g'%r['pairs_per_s_kernel'], 'frac %.3f'%r['frac'], 'E', d['energy_last_step'])"
  done
done
