# ncu --set full of kernel (a) gather at cfg4 (bench_gather: Eq.(3) sweeps with k = 1)
mkdir -p gpurun_out
timeout 600 python tools/bench_gather.py cfg4 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather -s 3 -c 1 -o gpurun_out/prof_r01_gather_cfg4 python tools/bench_gather.py cfg4 > gpurun_out/ncu_g4.log 2>&1; echo ncu_rc=$?
