"""Time-to-tolerance on Table-1-shaped SLS problems and configs[0].

    python tools/ttt.py [--n 2000] [--m 100000] [--sl 0.6] [--inner 10]
Device time (CUDA events) of setup (Gram + factor) and solve (iterations to
p_r, d_r, b_r <= 1e-4 plus finalize).  Diagnostic; bench.py reports the default row.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2405_16267_b200 import bicadmm as bc  # noqa: E402
from paper_2405_16267_b200 import datagen as dg  # noqa: E402


def run(n, m, sl, N=4, inner=10, refit=1, max_outer=3000, seed=0, loss="ls", tol_inner=False):
    kappa = int(round(n * (1 - sl)))
    P = dg.generate(N, m // N, n, kappa, loss, seed=seed, device="cuda")
    cs = dg.block_partition(n, 1)
    prm = bc.Params(kappa=kappa, max_outer=max_outer, inner_fixed=0 if tol_inner else inner, refit=refit,
                    eps_inner=1e-6, max_inner=200)
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    s = bc.BiCADMM(P.A, P.b, loss, prm, cs)
    e1.record()
    rep = s.solve()
    e2.record()
    torch.cuda.synchronize()
    sup = s.support()
    truth = np.nonzero(P.x_true.cpu().numpy())[0]
    out = dict(n=n, m=m, N=N, s_l=sl, kappa=kappa, K_in=("tol" if tol_inner else inner), setup_s=e0.elapsed_time(e1) / 1e3,
               solve_s=e1.elapsed_time(e2) / 1e3, total_s=e0.elapsed_time(e2) / 1e3, outer=rep.outer_iters,
               inner_sweeps=int(rep.inner_sweeps), converged=bool(rep.converged),
               support_recovered=bool(sup.size == truth.size and np.array_equal(np.sort(sup), truth)),
               objective=rep.objective, residuals=[rep.p_r, rep.d_r, rep.b_r])
    s.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", default="table1")
    ap.add_argument("--inner", type=int, default=10)
    a = ap.parse_args()
    rows = [(2000, 100000, 0.6), (4000, 100000, 0.6), (2000, 300000, 0.9), (4000, 300000, 0.9)]
    for (n, m, sl) in rows:
        print(json.dumps(run(n, m, sl, inner=a.inner)), flush=True)
    print(json.dumps(run(4000, 100000, 0.6, tol_inner=True)), flush=True)


if __name__ == "__main__":
    main()
