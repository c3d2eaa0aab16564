timeout 120 python tools/bench_hier.py cfg3 2>&1 | grep -v Warn | cut -c1-200; echo rc=$?
timeout 400 python -m pytest tests/test_gpu_hierarchy.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
