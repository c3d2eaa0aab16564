# kernel (a) software-pipelined row loop vs plain; parity + timing
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sweep.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_g.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_g.log | tail -3
for v in default nopipe pipe2 pipem3; do
  if [ $v = default ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  echo "== $v"; timeout 600 python tools/bench_gather.py cfg5 cfg4 cfg3 cfg2 2>&1 | grep -o '^cfg[0-9] .*"GBps": [0-9.]*' | sed 's/{.*"gather_ms"/ms/'
done
