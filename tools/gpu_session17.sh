mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|^E  " gpurun_out/pytest_gpu.log | tail -20
timeout 600 python - <<'PY'
import time, torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_1506_04383_b200 as mm
from workloads import configs
for name in ['cfg2', 'cfg3']:
    w = configs.make(name)
    g = mm.graph_to_device(w.graph)
    x = mm.coords_to_device(w.x0 if w.x0 is not None else configs.random_state(w.n, w.dim, 1, w.n ** 0.5))
    mm.full_stress(g, x); torch.cuda.synchronize()
    t = time.perf_counter(); r = mm.full_stress(g, x); dt = time.perf_counter() - t
    print(name, 'full stress', r, '%.3f s' % dt, 'pairs/s %.3g' % (r[3] / dt))
PY
