# entropy (e): one MUFU per 4 pairs for q = 0; energy parity incl. extreme scales; cfg2 bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_layout.py tests/test_gpu_metrics.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_e.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|Error|assert" gpurun_out/pytest_e.log | tail -8
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e.json 2>/dev/null; echo bench_rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_e.json'))
print('ms %.2f'%d['ms_per_step'], {k: (v['launches'], round(v['total_ms']/v['launches'],4)) for k,v in d['kernels'].items()})"
