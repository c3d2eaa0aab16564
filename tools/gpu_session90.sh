# final: full GPU suite, smoke, bench lines (cfg2, cfg3, cfg4, cfg5) with the final kernel (a), ncu of the gather at cfg5
mkdir -p gpurun_out/s90/r01_bench
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/s90/pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/s90/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/s90/r01_bench/bench_cfg2.json 2> gpurun_out/s90/e2.err; echo bench rc=$?
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 > gpurun_out/s90/r01_bench/bench_cfg3.json 2>/dev/null; echo cfg3 rc=$?
timeout 1200 python bench.py --config cfg4 --steps 2 --warmup 3 > gpurun_out/s90/r01_bench/bench_cfg4.json 2>/dev/null; echo cfg4 rc=$?
timeout 1500 python bench.py --config cfg5 --steps 2 --warmup 3 > gpurun_out/s90/r01_bench/bench_cfg5.json 2>/dev/null; echo cfg5 rc=$?
for c in 2 3 4 5; do python -c "
import json; d=json.load(open('gpurun_out/s90/r01_bench/bench_cfg$c.json')); r=d['roofline']
print('cfg$c ms %.2f'%d['ms_per_step'], 'value %.4g'%d['value'], r.get('kernel'), 'frac %.3f'%r['frac'], 'pairs/s %.4g'%r.get('pairs_per_s_kernel', 0), 'e2e %.4g'%d['e2e'].get('value'), d['clocks'])"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather -s 3 -c 1 -o gpurun_out/s90/prof_r01_gather_cfg5 python tools/bench_gather.py cfg5 > gpurun_out/s90/ncu_g5.log 2>&1; echo ncu_rc=$?
