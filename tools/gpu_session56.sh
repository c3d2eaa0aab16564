for v in default p_sg4 p_sg4m6 p_sg4m5 p_sg4u4 p_sg4s512; do
  if [ $v = default ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  echo "$v $(timeout 300 python tools/bench_sym.py cfg2 2>&1 | tail -1 | cut -c1-100)"
done
