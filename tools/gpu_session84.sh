# concurrency test with and without the state lock
mkdir -p gpurun_out/s84
export MM_LIB_PATH=$PWD/tools/gvar/nolock.so
for r in 1 2; do timeout 180 python -m pytest tests/test_gpu_layout.py -k concurrent -m gpu -q -x -p no:cacheprovider > gpurun_out/s84/nolock$r.log 2>&1; echo nolock rc=$?; grep -E "^E " gpurun_out/s84/nolock$r.log | head -3 | cut -c1-300; tail -1 gpurun_out/s84/nolock$r.log; done
unset MM_LIB_PATH
for r in 1 2; do timeout 300 python -m pytest tests/test_gpu_layout.py -k concurrent -m gpu -q -x -p no:cacheprovider > gpurun_out/s84/lock$r.log 2>&1; echo lock rc=$?; grep -E "^E " gpurun_out/s84/lock$r.log | head -3 | cut -c1-300; tail -1 gpurun_out/s84/lock$r.log; done
