# symmetric exact kernel: rotation-loop unroll / occupancy variants on cfg2
mkdir -p gpurun_out
for v in u4m4 u4m2 u8m2 u8m3 u4m2s512 u4sg4; do
  export MM_LIB_PATH=$PWD/tools/gvar/$v.so
  echo "== $v"; timeout 300 python tools/bench_sym.py cfg2 2>&1 | tail -1
done
