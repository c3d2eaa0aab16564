# smoke, reference arm, ncu of the new kernel (c) at cfg3
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 2>/dev/null | tail -1 | cut -c1-400
CMD3="python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_repulse -s 305 -c 1 -o gpurun_out/prof_r01_repulse_coarse_cfg3 $CMD3 > gpurun_out/ncu_c.log 2>&1; echo ncu_c_rc=$?
