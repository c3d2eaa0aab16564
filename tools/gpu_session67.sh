# Q29 polynomial 2^y share in the 3-D q>0 coarse kernel: parity + variants on cfg5
mkdir -p gpurun_out/s67
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s67/pytest.log 2>&1; tail -3 gpurun_out/s67/pytest.log
run() { # name config [env...]
  timeout 300 env "${@:3}" python bench.py --config $2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s67/b_$1_$2.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/s67/b_$1_$2.json')); r=d['roofline']
print('$1 $2 ms %.1f'%d['ms_per_step'], 'pairs/s %.4g'%r['pairs_per_s_kernel'], 'frac %.3f'%r['frac'])"
}
run new cfg5
for v in m3 p49 p11 p0 p55; do run $v cfg5 MM_LIB_PATH=$PWD/tools/gvar/$v.so; done
