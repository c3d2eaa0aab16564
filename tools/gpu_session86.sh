# round-1 re-entry final refresh: full GPU suite, smoke, bench lines of every config, cfg2 launch list
mkdir -p gpurun_out/s86/r01_bench
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/s86/pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/s86/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/s86/r01_bench/bench_cfg2.json 2> gpurun_out/s86/e2.err; echo bench rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s86/r01_launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s86/ncul2.log 2>&1; echo ncul2=$?
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 > gpurun_out/s86/r01_bench/bench_cfg3.json 2>/dev/null; echo cfg3 rc=$?
timeout 1200 python bench.py --config cfg4 --steps 2 --warmup 3 > gpurun_out/s86/r01_bench/bench_cfg4.json 2>/dev/null; echo cfg4 rc=$?
timeout 1500 python bench.py --config cfg5 --steps 2 --warmup 3 > gpurun_out/s86/r01_bench/bench_cfg5.json 2>/dev/null; echo cfg5 rc=$?
timeout 600 python bench.py --config cfg1 > gpurun_out/s86/r01_bench/bench_cfg1.json 2>/dev/null; echo cfg1 rc=$?
for c in 1 2 3 4 5; do python -c "
import json; d=json.load(open('gpurun_out/s86/r01_bench/bench_cfg$c.json')); r=d['roofline']
print('cfg$c ms %.2f'%d['ms_per_step'], 'value %.4g'%d['value'], r.get('kernel'), 'frac %.3f'%r['frac'], 'pairs/s %.4g'%r.get('pairs_per_s_kernel', 0), 'e2e %.4g'%d['e2e'].get('value'), d['clocks'])"; done
