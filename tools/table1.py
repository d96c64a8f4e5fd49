"""All twelve Table-1 rows: synthetic SLS, N = 4 nodes, n in {2000, 4000},
m in {1e5, 2e5, 3e5}, s_l in {0.6, 0.9}; solved to p_r, d_r, b_r <= 1e-4 with K_in = 10
and the LS refit; device time (CUDA events) of setup + solve.  Prints a markdown table."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2405_16267_b200 import bicadmm as bc, datagen as dg

PAPER = {(2000, 100000, 0.6): 1.1, (4000, 100000, 0.6): 1.8, (2000, 200000, 0.6): 1.7, (4000, 200000, 0.6): 3.0,
         (2000, 300000, 0.6): 2.2, (4000, 300000, 0.6): 4.0, (2000, 100000, 0.9): 1.1, (4000, 100000, 0.9): 1.9,
         (2000, 200000, 0.9): 1.7, (4000, 200000, 0.9): 2.9, (2000, 300000, 0.9): 2.2, (4000, 300000, 0.9): 4.1}
N = 4
print("| n | m | s_l | kappa | B200 s (setup + solve) | outer its | support recovered | paper s (RTX 4070) |")
print("|---|---|---|---|---|---|---|---|")
for sl in (0.6, 0.9):
    for m in (100000, 200000, 300000):
        for n in (2000, 4000):
            kappa = int(round(n * (1 - sl)))
            P = dg.generate(N, m // N, n, kappa, "ls", seed=0, device="cuda")
            cs = dg.block_partition(n, 1)
            prm = bc.Params(kappa=kappa, max_outer=3000, inner_fixed=10, refit=1)
            torch.cuda.synchronize()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record()
            s = bc.BiCADMM(P.A, P.b, "ls", prm, cs)
            e[1].record()
            rep = s.solve()
            e[2].record()
            torch.cuda.synchronize()
            sup = s.support()
            truth = np.nonzero(P.x_true.cpu().numpy())[0]
            ok = bool(np.array_equal(np.sort(sup), truth))
            print(f"| {n} | {m:.0e} | {sl} | {kappa} | {e[0].elapsed_time(e[2]) / 1e3:.2f} "
                  f"({e[0].elapsed_time(e[1]) / 1e3:.2f} + {e[1].elapsed_time(e[2]) / 1e3:.2f}) | {rep.outer_iters} | "
                  f"{ok} | {PAPER[(n, m, sl)]} |", flush=True)
            s.close()
            del P
            torch.cuda.empty_cache()
