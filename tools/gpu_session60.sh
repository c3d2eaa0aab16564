# re-entry check: full GPU suite, smoke, default bench
mkdir -p gpurun_out/s60
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
( time timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider ) > gpurun_out/s60/pytest.log 2>&1; tail -15 gpurun_out/s60/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/s60/bench.json 2> gpurun_out/s60/bench.err; echo bench_rc=$?; cut -c1-600 gpurun_out/s60/bench.json
