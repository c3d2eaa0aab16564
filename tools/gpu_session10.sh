mkdir -p gpurun_out
timeout 600 ./tools/ubench_repulse 65428 2>&1 | grep -E "COARSE|T=4 BMASK=1 MINB=1" | tee gpurun_out/ubench_coarse.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|chaos" gpurun_out/pytest_gpu.log | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench10.json 2> gpurun_out/bench10.err; echo bench_rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench10.json'))
print('value %.4g'%d['value'], 'ms %.2f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], 'e2e ms %.2f'%d['e2e']['ms_per_step'], 'E', d['energy_last_step'], d['kernels'])"
