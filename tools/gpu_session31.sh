for m in 2 0; do MM_SYM=$m timeout 600 python tools/sym_accuracy.py cfg2_rgg4096 cfg2_rgg16384 cfg2_rgg32768 2>&1 | tail -3; done
timeout 300 python tools/sched_energy_probe.py cfg3_mesh64 2 200 25 2>&1 | tail -1
