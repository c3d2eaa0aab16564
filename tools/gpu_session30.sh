for lib in current prev; do
  if [ $lib = prev ]; then export MM_LIB_PATH=$PWD/tools/gvar/prev.so; fi
  timeout 300 python tools/sched_energy_probe.py cfg3_mesh64 2 200 25 2>&1 | tail -2
done
unset MM_LIB_PATH
MM_SYM=0 timeout 300 python tools/sched_energy_probe.py cfg3_mesh64 2 200 25 2>&1 | tail -2
