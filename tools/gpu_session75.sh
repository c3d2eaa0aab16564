# symmetric kernel: source sub-tile 128 / 512 (units per CTA: load balance) and 5 CTAs/SM
for v in new src128 src512 minb5 new src128; do
  if [ $v = new ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  echo "$v $(timeout 300 python tools/bench_sym.py cfg2 2>&1 | tail -1 | cut -c1-150)"
done
