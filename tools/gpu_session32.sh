# full GPU suite after the sym threshold fix + ncu --set full of k_repulse_sym inside bench.py
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|chaos" gpurun_out/pytest_gpu.log | tail -6
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_repulse_sym -s 70 -c 1 -o gpurun_out/prof_r01_repulse_sym python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_sym.log 2>&1; echo ncu_rc=$?
