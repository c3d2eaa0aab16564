# symmetric kernel with sub-tile units: timing vs one-sided across n; parity
mkdir -p gpurun_out
for c in cfg2 cfg2_rgg32768 cfg2_rgg16384; do
  for m in 2 0; do MM_SYM=$m timeout 300 python tools/bench_sym.py $c 2>&1 | tail -1; done
done
timeout 900 python -m pytest tests/test_gpu_sym.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2
