mkdir -p gpurun_out
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -3
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -20
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo bench_rc=$?; tail -3 gpurun_out/bench4.err
python -c "
import json; d=json.load(open('gpurun_out/bench4.json'))
print('value', d['value'], 'ms', d['ms_per_step'], 'frac', d['roofline']['frac'], 'pairs/s', d['roofline']['pairs_per_s_kernel'], 'e2e', d['e2e']['value'])
print(d['kernel_share_of_step']); print(d['clocks']); print(d['cpu_baseline'])"
