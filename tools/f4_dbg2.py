"""Debug: which rows of p differ after a few fused sweeps (env selects R / groups)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2405_16267_b200 import bicadmm as bc
from paper_2405_16267_b200 import datagen as dg
N, m, n, K = 1, 600, 300, int(sys.argv[1]) if len(sys.argv) > 1 else 1
NO = int(sys.argv[2]) if len(sys.argv) > 2 else 1
P = dg.generate(N, m, n, 10, "logistic", seed=0)
cs = dg.block_partition(n, 1)
out = {}
for sweep in (1, 2):
    s = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "logistic",
                   bc.Params(kappa=10, max_outer=5, inner_fixed=K, refit=0, eps_p=0, eps_d=0, eps_b=0, sweep=sweep), cs)
    for o in range(NO):
        s.iterate(1)
        pp = s.get(bc.FIELD_P_LOCAL); nu = s.get(bc.FIELD_NU); r = s.get(bc.FIELD_R_LOCAL)
        print(sweep, o, 'z norm', np.linalg.norm(s.z), 'x nan', int(np.isnan(s.get(bc.FIELD_X_LOCAL)).sum()),
              'p nan rows', np.nonzero(np.isnan(pp))[0][:12], 'nu nan', int(np.isnan(nu).sum()), 'r nan', int(np.isnan(r).sum()))
    out[sweep] = (s.get(bc.FIELD_P_LOCAL), s.get(bc.FIELD_X_LOCAL), s.get(bc.FIELD_NU))
    s.close()
p2, p1 = out[2][0], out[1][0]
bad = np.nonzero(~np.isclose(p2, p1, rtol=1e-9, atol=1e-12))[0]
print("K", K, "p rows bad:", len(bad), bad[:40], "nan:", int(np.isnan(p2).sum()))
x2, x1 = out[2][1], out[1][1]
badx = np.nonzero(~np.isclose(x2, x1, rtol=1e-6, atol=1e-9))[0]
print("x cols bad:", len(badx), badx[:20], "nan:", int(np.isnan(x2).sum()))
