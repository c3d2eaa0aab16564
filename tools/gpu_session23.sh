# symmetric exact kernel: parity tests + per-mode timing
mkdir -p gpurun_out
for m in 1 0; do
  for c in cfg2 cfg1_grid64 cfg5_grid16; do
    MM_SYM=$m timeout 300 python tools/bench_sym.py $c 2>&1 | tail -2
  done
done
python - <<'PY'
import numpy as np
for c in ["cfg2", "cfg1_grid64", "cfg5_grid16"]:
    a = np.load(f"gpurun_out/sym_{c}_1.npy"); b = np.load(f"gpurun_out/sym_{c}_0.npy")
    print(c, "max|sym-plain| / max|x|", float(np.abs(a - b).max() / np.abs(b).max()))
PY
timeout 1200 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_layout.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_sym.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_sym.log | tail -8
