mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|chaos" gpurun_out/pytest_gpu.log | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench8.json 2> gpurun_out/bench8.err; echo bench_rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench8.json'))
print('value %.4g'%d['value'], 'ms %.2f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], 'e2e ms %.2f'%d['e2e']['ms_per_step'], 'launches', d['gpu_launches'])"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_cfg2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo ncu_list_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_repulse -s 8 -c 1 -o gpurun_out/prof_r01_repulse_exact $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu_full_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_entropy -s 1 -c 1 -o gpurun_out/prof_r01_entropy $CMD > gpurun_out/ncu_full_e.log 2>&1; echo ncu_full_e_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gather -s 8 -c 1 -o gpurun_out/prof_r01_gather $CMD > gpurun_out/ncu_full_g.log 2>&1; echo ncu_full_g_rc=$?
CMD3="python bench.py --config cfg3 --steps 1 --warmup 1"
timeout 600 $CMD3 > gpurun_out/plain_cfg3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_repulseILi2ELb0ELb1" -s 4 -c 1 -o gpurun_out/prof_r01_repulse_coarse $CMD3 > gpurun_out/ncu_full2.log 2>&1; echo ncu_full2_rc=$?
