mkdir -p gpurun_out
for G in auto 1 2 4 8 16 32; do
  if [ $G = auto ]; then unset MM_GATHER_G; else export MM_GATHER_G=$G; fi
  timeout 600 python tools/bench_gather.py cfg5 cfg4 cfg3 cfg2 2>&1 | grep -E "^cfg" | sed "s/^/G=$G /"
done
unset MM_GATHER_G
MM_TRACE=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline 2> gpurun_out/trace.err > gpurun_out/trace.json; grep mm_trace gpurun_out/trace.err | tail -24
python -c "
import json; d=json.load(open('gpurun_out/trace.json'))
print('value %.4g'%d['value'], 'ms %.2f'%d['ms_per_step'], 'e2e ms %.2f'%d['e2e']['ms_per_step'], d['kernels'])"
