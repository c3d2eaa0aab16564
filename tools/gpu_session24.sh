# symmetric exact kernel: SG=2 vs SG=4 timing, ncu of SG=2 on cfg2
mkdir -p gpurun_out
for v in default sg4; do
  if [ $v = default ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  echo "== $v"; timeout 300 python tools/bench_sym.py cfg2 2>&1 | tail -1
done
unset MM_LIB_PATH
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_repulse_sym -s 3 -c 1 -o gpurun_out/prof_r01_repulse_sym python tools/bench_sym.py cfg2 > gpurun_out/ncu_sym.log 2>&1; echo ncu_rc=$?
