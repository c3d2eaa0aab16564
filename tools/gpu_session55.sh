# sym kernel with plain reciprocals: parity, bench, launch list + ncu
mkdir -p gpurun_out/r01_bench
timeout 1200 python -m pytest tests/test_gpu_sym.py tests/test_gpu_sweep.py tests/test_gpu_c_abi.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r01_bench/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo bench_rc=$?
python -c "
import json; d=json.load(open('gpurun_out/r01_bench/bench_cfg2.json')); r=d['roofline']
print('value %.4g'%d['value'], 'ms %.2f'%d['ms_per_step'], 'frac %.3f exec %.3f'%(r['frac'], r['executed_frac']), 'e2e', round(d['e2e']['ms_per_step'],2), d['clocks'], {k: round(v,4) for k,v in d['kernel_share_of_gpu_time'].items() if v > 0.002})"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_repulse_sym -s 70 -c 1 -o gpurun_out/prof_r01_repulse_sym python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_sym.log 2>&1; echo ncu_rc=$?
