import sys, time
sys.path.insert(0, '/root/repo')
import torch, numpy as np
from paper_2405_16267_b200 import bicadmm as bc, datagen as dg
for rep in range(3):
    P = dg.generate(2, 100, 50, 5, "ls", seed=rep)
    cs = dg.block_partition(50, 1)
    A = [a.cuda() for a in P.A]; b = [x.cuda() for x in P.b]
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    s = bc.BiCADMM(A, b, "ls", bc.Params(kappa=5, max_outer=2000, inner_fixed=10, refit=1), cs)
    e[1].record()
    r = s.solve()
    e[2].record()
    torch.cuda.synchronize()
    print("setup %.3f ms solve %.3f ms outer %d launches %d" % (e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), r.outer_iters, s.launches()))
    s.close()
