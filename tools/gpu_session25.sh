# symmetric exact kernel variants (sub-tile, SG, occupancy) on cfg2
mkdir -p gpurun_out
for v in default src512 sg4 sg4b minb2; do
  if [ $v = default ]; then unset MM_LIB_PATH; else export MM_LIB_PATH=$PWD/tools/gvar/$v.so; fi
  echo "== $v"; timeout 300 python tools/bench_sym.py cfg2 2>&1 | tail -1
done
unset MM_LIB_PATH
MM_SYM=0 timeout 300 python tools/bench_sym.py cfg2 2>&1 | tail -1
python -c "
import numpy as np
a=np.load('gpurun_out/sym_cfg2_1.npy'); b=np.load('gpurun_out/sym_cfg2_0.npy'); print('rel', float(np.abs(a-b).max()/np.abs(b).max()))"
