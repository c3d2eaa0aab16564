set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | grep -E "Model name|^CPU\(s\)"
timeout 60 ./tools/ubench_pipes > gpurun_out/ubench.txt 2>&1; cat gpurun_out/ubench.txt
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -20 gpurun_out/smoke.log
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-s 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench_rc=$?; tail -5 gpurun_out/bench1.err; cat gpurun_out/bench1.json
