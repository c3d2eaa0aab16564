for v in default q_s128 q_m5 q_u4 default; do
  if [ $v = default ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  echo "$v $(timeout 300 python tools/bench_sym.py cfg2 2>&1 | tail -1 | cut -c1-100)"
done
