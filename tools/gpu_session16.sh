mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_schedule.py -q -p no:cacheprovider 2>&1 | tail -3
for h in 0 2 7; do
  timeout 900 python bench.py --config cfg2 --schedule --h $h --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/sched_cfg2_h$h.json 2>/dev/null; echo rc=$?
  python -c "
import json; d=json.load(open('gpurun_out/sched_cfg2_h$h.json'))
print('cfg2 MulMent_$h', 'ms %.1f'%d['ms_per_step'], 'vu/s %.3g'%d['value'], 'levels', len(d['levels']), 'E', d['energy_last_step'])"
done
for c in cfg3 cfg4; do for h in 2 7; do
  timeout 900 python bench.py --config $c --schedule --h $h --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/sched_${c}_h$h.json 2>/dev/null; echo rc=$?
  python -c "
import json; d=json.load(open('gpurun_out/sched_${c}_h$h.json'))
print('$c MulMent_$h', 'ms %.1f'%d['ms_per_step'], 'vu/s %.3g'%d['value'], 'levels', len(d['levels']), 'E', d['energy_last_step'])"
done; done
