# symmetric kernel (b): packed j-side partials vs scalar FFMAs
mkdir -p gpurun_out/s69
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s69/pytest.log 2>&1; tail -3 gpurun_out/s69/pytest.log
for v in new jp0 new jp0; do
  if [ $v = new ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  echo "$v $(timeout 300 python tools/bench_sym.py cfg2 2>&1 | tail -1 | cut -c1-160)"
done
unset MM_LIB_PATH
timeout 600 python bench.py > gpurun_out/s69/bench_cfg2.json 2> gpurun_out/s69/e2.err; echo rc=$?
python -c "
import json; d=json.load(open('gpurun_out/s69/bench_cfg2.json')); r=d['roofline']
print('cfg2 ms %.2f'%d['ms_per_step'], 'frac %.3f'%r['frac'], 'exec %.3f'%r['executed_frac'], d['clocks'])"
timeout 600 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s69/bench_cfg3.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/s69/bench_cfg3.json')); r=d['roofline']; sh=d['kernel_share_of_step']; ms=d['ms_per_step']
print('cfg3 ms %.2f'%ms, 'frac %.3f'%r['frac'], {k: round(v*ms,2) for k,v in sorted(sh.items(), key=lambda kv:-kv[1])[:8]})"
