mkdir -p gpurun_out/r01
B=gpurun_out/r01
timeout 600 python bench.py --steps 5 --warmup 3 > $B/bench_cfg2.json 2> $B/bench_cfg2.err; echo cfg2 rc=$?
timeout 600 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline > $B/bench_cfg1.json 2>/dev/null; echo cfg1 rc=$?
for c in cfg3 cfg4 cfg5; do timeout 900 python bench.py --config $c --steps 1 --warmup 1 > $B/bench_$c.json 2>/dev/null; echo $c rc=$?; done
for c in cfg2 cfg3 cfg4; do for h in 0 7 10; do
  if [ $c = cfg4 ] && [ $h = 0 ]; then continue; fi
  timeout 900 python - > $B/sched_${c}_h$h.json 2>/dev/null <<PY
import json, time, sys, torch
sys.path.insert(0, '.')
import paper_1506_04383_b200 as mm
from workloads import configs
w = configs.make('$c')
G = mm.graph_to_device(w.graph); S = mm.sset_to_device(w.S)
sch = mm.paper_schedule(max_final_iters=200)
out = {}
for sc, dc in ((False, False), (True, True)):
    mm.layout_schedule(G, S, w.dim, w.q, $h, sch, w.seed, sclap=sc, disc=dc)  # warm-up (also builds caches)
    torch.cuda.synchronize(); t = time.perf_counter()
    x, rep = mm.layout_schedule(G, S, w.dim, w.q, $h, sch, w.seed, sclap=sc, disc=dc)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    fs = mm.full_stress(G, x) if w.n <= 300000 else None
    out['sclap' if sc else 'matching'] = {'seconds': dt, 'levels': rep['levels'], 'sweeps': rep['sweeps_level'],
        'M_alpha_min': rep['energy'], 'coincident': rep['coincident_pairs'], 'full_stress': fs}
print(json.dumps({'config': '$c', 'h': $h, **out}))
PY
  echo sched $c h=$h rc=$?
done; done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > $B/plain_cfg2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $B/launches_cfg2.csv $CMD > $B/ncu_list.log 2>&1; echo ncu_list_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_repulse -s 8 -c 1 -o $B/prof_repulse_exact $CMD > /dev/null 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gather -s 8 -c 1 -o $B/prof_gather_cfg2 $CMD > /dev/null 2>&1; echo ncu2=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_entropy -s 1 -c 1 -o $B/prof_entropy $CMD > /dev/null 2>&1; echo ncu3=$?
CMD3="python bench.py --config cfg3 --steps 1 --warmup 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_repulse -s 305 -c 1 -o $B/prof_repulse_coarse_cfg3 $CMD3 > /dev/null 2>&1; echo ncu4=$?
