"""Device time of bicadmm_solve on configs[0] (launch-bound): device loop vs host loop."""
import os, sys
import torch
sys.path.insert(0, ".")
from paper_2405_16267_b200 import bicadmm as bc, datagen as dg
P = dg.generate(2, 100, 50, 5, "ls", seed=3)
cs = dg.block_partition(50, 1)
for g in ("1", "0", "1", "0"):
    os.environ["BICADMM_GRAPH"] = g
    s = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "ls",
                   bc.Params(kappa=5, max_outer=2000, inner_fixed=10, refit=0, eps_p=1e-7, eps_d=1e-7, eps_b=1e-7), cs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep = s.solve()
    e1.record()
    torch.cuda.synchronize()
    print(f"BICADMM_GRAPH={g}: {rep.outer_iters} outer iterations, solve {e0.elapsed_time(e1):.2f} ms "
          f"({1e3 * e0.elapsed_time(e1) / rep.outer_iters:.1f} us per outer iteration)", flush=True)
    s.close()
