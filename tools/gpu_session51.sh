for N in 20000 40000; do echo "== MM_SMALL_N=$N"; MM_SMALL_N=$N MM_TRACE=1 timeout 300 python tools/trace_levels.py cfg2 7 2>&1 | sed -n "/---- timed/,\$p" | grep "level [0-3] "; done
for N in 20000 40000; do echo "== MM_SMALL_N=$N cfg3"; MM_SMALL_N=$N MM_TRACE=1 timeout 300 python tools/trace_levels.py cfg3 7 2>&1 | sed -n "/---- timed/,\$p" | grep "level"; done
