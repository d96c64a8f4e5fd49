"""configs[0] time-to-tolerance anatomy: setup, solve with and without the LS refit
(device time between CUDA events; wall time brackets host work)."""
import sys, time
sys.path.insert(0, '/root/repo')
import torch  # noqa: E402
from paper_2405_16267_b200 import bicadmm as bc, datagen as dg  # noqa: E402

for refit in (1, 0):
    for rep in range(4):
        P = dg.generate(2, 100, 50, 5, "ls", seed=rep)
        cs = dg.block_partition(50, 1)
        A = [a.cuda() for a in P.A]; b = [x.cuda() for x in P.b]
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        t0 = time.perf_counter()
        e[0].record()
        s = bc.BiCADMM(A, b, "ls", bc.Params(kappa=5, max_outer=2000, inner_fixed=10, refit=refit), cs)
        e[1].record()
        t1 = time.perf_counter()
        r = s.solve()
        e[2].record()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print("refit %d setup %.3f ms (wall %.3f) solve %.3f ms (wall %.3f) outer %d launches %d"
              % (refit, e[0].elapsed_time(e[1]), (t1 - t0) * 1e3, e[1].elapsed_time(e[2]), (t2 - t1) * 1e3,
                 r.outer_iters, s.launches()))
        s.close()
