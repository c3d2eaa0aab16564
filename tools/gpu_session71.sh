# refresh the MulMent_h schedule timings after the kernel (c) changes (Q26-Q29)
mkdir -p gpurun_out/s71
B=gpurun_out/s71
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
