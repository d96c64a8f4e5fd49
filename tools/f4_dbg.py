"""Debug: one small fused-sweep case vs the two-pass kernels (R / group overrides via env)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2405_16267_b200 import bicadmm as bc
from paper_2405_16267_b200 import datagen as dg
N, m, n = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (4, 600, 300))]
P = dg.generate(N, m, n, 10, "logistic", seed=0)
cs = dg.block_partition(n, 1)
out = {}
for sweep in (1, 2):
    s = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "logistic",
                   bc.Params(kappa=10, max_outer=5, inner_fixed=2, refit=0, eps_p=0, eps_d=0, eps_b=0, sweep=sweep), cs)
    s.iterate(2)
    out[sweep] = (s.z, s.get(bc.FIELD_X_LOCAL), s.get(bc.FIELD_P_LOCAL), s.sweep_kind())
    s.close()
for k, nm in enumerate(("z", "x", "p")):
    a, b = out[2][k], out[1][k]
    print(nm, "fused norm %.6g two-pass norm %.6g rel diff %.3g" % (np.linalg.norm(a), np.linalg.norm(b),
          np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)))
print("kinds", out[2][3], out[1][3], "env", {k: v for k, v in os.environ.items() if k.startswith("BICADMM_F4")})
