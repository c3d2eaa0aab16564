for v in default cb0 cb3; do
  if [ $v = default ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  timeout 900 python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v cfg3', round(d['ms_per_step'],1), '%.4g'%r['pairs_per_s_kernel'])"
done
