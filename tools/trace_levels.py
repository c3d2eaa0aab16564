import sys, torch
sys.path.insert(0, '.')
import paper_1506_04383_b200 as mm
from workloads import configs
w = configs.make(sys.argv[1]); h = int(sys.argv[2]); sc = len(sys.argv) > 3 and sys.argv[3] == "sclap"
G, S = mm.graph_to_device(w.graph), mm.sset_to_device(w.S)
sch = mm.paper_schedule(max_final_iters=200)
mm.layout_schedule(G, S, w.dim, w.q, h, sch, w.seed, sclap=sc, disc=sc)
torch.cuda.synchronize()
print("---- timed", flush=True)
mm.layout_schedule(G, S, w.dim, w.q, h, sch, w.seed, sclap=sc, disc=sc)
torch.cuda.synchronize()
