# round-1 re-entry check: full GPU suite, smoke, headline bench on a fresh box
mkdir -p gpurun_out/s80
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/s80/pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/s80/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/s80/bench_cfg2.json 2> gpurun_out/s80/e2.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/s80/bench_cfg2.json')); r=d['roofline']
print('cfg2 ms %.2f'%d['ms_per_step'], 'value %.4g'%d['value'], 'frac %.3f'%r['frac'], 'e2e %.4g'%d['e2e']['value'], d['clocks'])"
timeout 300 python tools/bench_gather.py 2>&1 | tail -30
