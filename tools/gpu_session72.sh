# far-tile threshold (MM_FAR_PAIRS): parity (all modes) + schedules + bench cfg3
mkdir -p gpurun_out/s72
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s72/pytest.log 2>&1; tail -3 gpurun_out/s72/pytest.log
bash tools/gpu_session71.sh > /dev/null 2>&1
for f in gpurun_out/s71/*.json; do python -c "
import json; d=json.load(open('$f')); print(d['config'], d['h'], {k: round(v['seconds'],3) for k,v in d.items() if isinstance(v, dict)})"; done
timeout 600 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s72/bench_cfg3.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/s72/bench_cfg3.json')); r=d['roofline']
print('cfg3 ms %.2f'%d['ms_per_step'], 'frac %.3f'%r['frac'])"
