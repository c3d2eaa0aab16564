# round-1 refresh after Q26-Q29: bench lines for every config, ncu of kernel (c) at the finest levels
mkdir -p gpurun_out/s68/r01_bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python bench.py > gpurun_out/s68/r01_bench/bench_cfg2.json 2> gpurun_out/s68/e2.err; echo cfg2 rc=$?
timeout 600 python bench.py --config cfg1 > gpurun_out/s68/r01_bench/bench_cfg1.json 2> gpurun_out/s68/e1.err; echo cfg1 rc=$?
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 > gpurun_out/s68/r01_bench/bench_cfg3.json 2> gpurun_out/s68/e3.err; echo cfg3 rc=$?
timeout 1200 python bench.py --config cfg4 --steps 2 --warmup 3 > gpurun_out/s68/r01_bench/bench_cfg4.json 2> gpurun_out/s68/e4.err; echo cfg4 rc=$?
timeout 1500 python bench.py --config cfg5 --steps 2 --warmup 3 > gpurun_out/s68/r01_bench/bench_cfg5.json 2> gpurun_out/s68/e5.err; echo cfg5 rc=$?
for c in 1 2 3 4 5; do python -c "
import json; d=json.load(open('gpurun_out/s68/r01_bench/bench_cfg$c.json')); r=d['roofline']
print('cfg$c ms %.2f'%d['ms_per_step'], 'value %.4g'%d['value'], 'kernel', r.get('kernel'), 'frac %.3f'%r['frac'], 'pairs/s %.4g'%r.get('pairs_per_s_kernel', 0), 'e2e', d['e2e'].get('value'), d['clocks'])"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_repulse -s 100 -c 1 -o gpurun_out/s68/prof_r01_repulse_coarse_cfg3 python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s68/ncu3.log 2>&1; echo ncu3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_repulse -s 105 -c 1 -o gpurun_out/s68/prof_r01_repulse_coarse_cfg4 python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s68/ncu4.log 2>&1; echo ncu4=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_repulse -s 95 -c 1 -o gpurun_out/s68/prof_r01_repulse_coarse_cfg5 python bench.py --config cfg5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s68/ncu5.log 2>&1; echo ncu5=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s68/r01_launches_cfg3.csv python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s68/ncul3.log 2>&1; echo ncul3=$?
