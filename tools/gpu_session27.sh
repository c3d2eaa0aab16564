# symmetric exact kernel (unroll 8, 3 CTAs/SM): parity suites + bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sym.py tests/test_gpu_sweep.py tests/test_gpu_layout.py tests/test_gpu_schedule.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_sym.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|Error|chaos" gpurun_out/pytest_sym.log | tail -12
for m in 1 0; do MM_SYM=$m timeout 300 python tools/bench_sym.py cfg2 2>&1 | tail -1; done
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_sym.json 2> gpurun_out/bench_sym.err; echo bench_rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_sym.json'))
print('value %.4g'%d['value'], 'ms %.2f'%d['ms_per_step'], 'roofline', d['roofline'], 'e2e', d['e2e'], 'clocks', d['clocks'])
print({k: round(v,4) for k,v in d['kernel_share_of_gpu_time'].items() if v > 0.002})"
