# refresh: bench lines for every config (steps timed without profiling events), ncu finest-level kernel (c)
mkdir -p gpurun_out/s70/r01_bench
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/s70/r01_bench/bench_cfg2.json 2> gpurun_out/s70/e2.err; echo cfg2 rc=$?
timeout 600 python bench.py --config cfg1 > gpurun_out/s70/r01_bench/bench_cfg1.json 2> gpurun_out/s70/e1.err; echo cfg1 rc=$?
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 > gpurun_out/s70/r01_bench/bench_cfg3.json 2> gpurun_out/s70/e3.err; echo cfg3 rc=$?
timeout 1200 python bench.py --config cfg4 --steps 2 --warmup 3 > gpurun_out/s70/r01_bench/bench_cfg4.json 2> gpurun_out/s70/e4.err; echo cfg4 rc=$?
timeout 1500 python bench.py --config cfg5 --steps 2 --warmup 3 > gpurun_out/s70/r01_bench/bench_cfg5.json 2> gpurun_out/s70/e5.err; echo cfg5 rc=$?
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/s70/ref_cfg2.json 2> gpurun_out/s70/eref.err; echo ref rc=$?; cut -c1-300 gpurun_out/s70/ref_cfg2.json
for c in 1 2 3 4 5; do python -c "
import json; d=json.load(open('gpurun_out/s70/r01_bench/bench_cfg$c.json')); r=d['roofline']
print('cfg$c ms %.2f'%d['ms_per_step'], 'value %.4g'%d['value'], r.get('kernel'), 'frac %.3f'%r['frac'], 'pairs/s %.4g'%r.get('pairs_per_s_kernel', 0), 'e2e %.4g'%d['e2e'].get('value'), 'cpu', (d.get('cpu_baseline') or {}).get('value'), d['clocks'])"; done
for c in cfg3 cfg4 cfg5; do
timeout 900 ncu --nvtx --nvtx-include "finest/" --set full --clock-control none --import-source on -k regex:k_repulse -c 1 -o gpurun_out/s70/prof_r01_repulse_coarse_$c python tools/profile_finest.py $c > gpurun_out/s70/ncu_$c.log 2>&1; echo ncu $c rc=$?; tail -1 gpurun_out/s70/ncu_$c.log
done
