# Q28 frame origin + centroid-keyed representative order: parity + A/B
mkdir -p gpurun_out/s66
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s66/pytest.log 2>&1; tail -3 gpurun_out/s66/pytest.log
run() { # name config [env...]
  timeout 300 env "${@:3}" python bench.py --config $2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s66/b_$1_$2.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/s66/b_$1_$2.json')); r=d['roofline']
print('$1 $2 ms %.1f'%d['ms_per_step'], 'pairs/s %.4g'%r['pairs_per_s_kernel'], 'frac %.3f'%r['frac'])"
}
run new cfg4
run level cfg4 MM_REORDER_PAIRS=1e30
run every cfg4 MM_REORDER_PAIRS=1e9
run new cfg3
run new cfg5
