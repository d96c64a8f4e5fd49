"""Phase breakdown of the Table-1 time-to-tolerance row (bench.py time_to_tol)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2405_16267_b200 import bicadmm as bc, datagen as dg

n, m, N, sl = int(os.environ.get("TTT_N", "4000")), 300_000, 4, 0.9
kappa = int(round(n * (1 - sl)))
P = dg.generate(N, m // N, n, kappa, "ls", seed=0, device="cuda")
cs = dg.block_partition(n, 1)
for refit in (1, 0):
    prm = bc.Params(kappa=kappa, max_outer=3000, inner_fixed=10, refit=refit, sweep=int(os.environ.get("SWEEP", "0")))
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    s = bc.BiCADMM(P.A, P.b, "ls", prm, cs)
    ev[1].record()
    s.set_profiling(True)
    info = None
    while True:
        info = s.iterate(1)
        if info.converged or info.outer_iters >= 3000:
            break
    ev[2].record()
    rep = s.finalize()
    ev[3].record()
    torch.cuda.synchronize()
    print(f"refit={refit} setup {ev[0].elapsed_time(ev[1]):.1f} ms, iterate {ev[1].elapsed_time(ev[2]):.1f} ms "
          f"({info.outer_iters} outer), finalize {ev[2].elapsed_time(ev[3]):.1f} ms", flush=True)
    print({k: (round(v[0], 2), v[1]) for k, v in s.phases().items() if v[1]}, flush=True)
    s.close()
