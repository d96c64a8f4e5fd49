"""Debug: per-sweep comparison (p, nu, r, x) of the fused sweep against the two-pass sweep."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2405_16267_b200 import bicadmm as bc
from paper_2405_16267_b200 import datagen as dg
N, m, n = 1, int(os.environ.get('DBG_M', 600)), int(os.environ.get('DBG_N', 300))
NO = int(sys.argv[1]) if len(sys.argv) > 1 else 3
P = dg.generate(N, m, n, 10, "logistic", seed=0)
cs = dg.block_partition(n, 1)
res = {}
for sweep in (1, 2):
    s = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "logistic",
                   bc.Params(kappa=10, max_outer=50, inner_fixed=1, refit=0, eps_p=0, eps_d=0, eps_b=0, sweep=sweep), cs)
    res[sweep] = []
    for o in range(NO):
        s.iterate(1)
        res[sweep].append({f: s.get(getattr(bc, "FIELD_" + f)) for f in ("P_LOCAL", "NU", "R_LOCAL", "X_LOCAL")})
    s.close()
for o in range(NO):
    line = []
    for f in ("P_LOCAL", "NU", "R_LOCAL", "X_LOCAL"):
        a, b = res[2][o][f], res[1][o][f]
        d = np.abs(a - b)
        bad = np.nonzero(~(d <= 1e-9 * (np.abs(b) + 1e-12)))[0]
        line.append("%s bad %d first %s" % (f, len(bad), bad[:6]))
    print("sweep", o + 1, " | ".join(line))

a, b = res[2][1]["R_LOCAL"], res[1][1]["R_LOCAL"]
a3, b3 = res[2][2]["R_LOCAL"], res[1][2]["R_LOCAL"]
for lo, hi in ((0, 64), (64, 128), (128, 152), (152, 216), (216, 300)):
    print("cols %d-%d: sweep2 r max|d| %.3g  sweep3 r max|d| %.3g  |r| %.3g" % (lo, hi, np.abs(a[lo:hi] - b[lo:hi]).max(),
          np.nanmax(np.abs(a3[lo:hi] - b3[lo:hi])) if not np.isnan(a3[lo:hi]).all() else float('nan'), np.abs(b3[lo:hi]).max()))
