# Q27: spatial orders + lo-free far tiles in kernel (c): parity + A/B
mkdir -p gpurun_out/s63
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s63/pytest.log 2>&1; tail -3 gpurun_out/s63/pytest.log
run() { # name config [env...]
  timeout 300 env "${@:3}" python bench.py --config $2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s63/b_$1_$2.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/s63/b_$1_$2.json')); r=d['roofline']
print('$1 $2 ms %.1f'%d['ms_per_step'], 'pairs/s %.4g'%r['pairs_per_s_kernel'], 'frac %.3f'%r['frac'], 'E %.8g'%d.get('energy', {}).get('total', float('nan')) if isinstance(d.get('energy'),dict) else d.get('energy'))"
}
for c in cfg3 cfg4; do
  run q26 $c MM_LIB_PATH=$PWD/tools/gvar/q26.so
  run new $c
  run lo $c MM_FAR_TILES=0
  run nobatch $c MM_LIB_PATH=$PWD/tools/gvar/nobatch.so
done
run q26 cfg5 MM_LIB_PATH=$PWD/tools/gvar/q26.so
run new cfg5
