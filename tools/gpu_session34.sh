# kernel (a) gather: streaming loads + 32-bit offsets; waves / unroll / occupancy variants
for v in default gu8 gu8m3 gu2 gm6; do
  if [ $v = default ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  for wv in 1 2 4; do
    echo "== $v waves=$wv"; MM_GATHER_WAVES=$wv timeout 600 python tools/bench_gather.py cfg4 cfg5 cfg3 2>&1 | grep -o '^cfg[0-9] .*"GBps": [0-9.]*' | sed 's/{.*"gather_ms"/ms/'
  done
done
