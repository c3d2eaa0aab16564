# partials at the vertex id (coalesced gather reads) + polynomial 2^y share in the q>0 energy
mkdir -p gpurun_out/s73
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s73/pytest.log 2>&1; tail -3 gpurun_out/s73/pytest.log
run() { # name config steps [env...]
  timeout 900 env "${@:4}" python bench.py --config $2 --steps $3 --warmup 3 --no-cpu-baseline > gpurun_out/s73/b_$1_$2.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/s73/b_$1_$2.json')); r=d['roofline']; sh=d['kernel_share_of_step']; ms=d['ms_per_step']
print('$1 $2 ms %.1f'%ms, 'pairs/s %.4g'%r['pairs_per_s_kernel'], {k: round(v*ms,2) for k,v in sorted(sh.items(), key=lambda kv:-kv[1])[:4]})"
}
run new cfg4 2
run prev cfg4 2 MM_LIB_PATH=$PWD/tools/gvar/prev.so
run new cfg5 1
run prev cfg5 1 MM_LIB_PATH=$PWD/tools/gvar/prev.so
