"""Per-row timeline of the single-pass sweep (k_fused4) from a trace build.

    tools/build_variant.sh f4trace k_fused4.cu -DBIC_F4_TRACE
    BICADMM_LIB_PATH=build_ab/f4trace.so python tools/f4_trace.py [--dtype f32] [--loss ls]

Records clock64 stamps for the first 1024 rows of cluster 0 (both CTAs) during the last
sweep of a C2-shaped run and prints the median per-row intervals (cycles)."""
import argparse
import ctypes as ct
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2405_16267_b200 import bicadmm as bc  # noqa: E402
from paper_2405_16267_b200 import datagen as dg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dtype", default="f64")
ap.add_argument("--loss", default="logistic")
ap.add_argument("--n", type=int, default=10_000)
ap.add_argument("--m", type=int, default=25_000)
ap.add_argument("--nodes", type=int, default=4)
ap.add_argument("--out", default=None)
a = ap.parse_args()
dt = torch.float64 if a.dtype == "f64" else torch.float32
L = bc.lib()
fn = L.bicadmm_debug_f4_trace
fn.argtypes = [ct.c_void_p]
R = 1024
buf = torch.zeros(2 * R * 8, dtype=torch.int64, device="cuda")
assert fn(buf.data_ptr()) == 0
P = dg.generate(a.nodes, a.m, a.n, 100, a.loss, seed=1000, device="cuda", dtype=dt)
cs = dg.block_partition(a.n, 1)
s = bc.BiCADMM(P.A, P.b, a.loss, bc.Params(kappa=100, max_outer=100, inner_fixed=10, sweep=2), cs)
s.iterate(3)
torch.cuda.synchronize()
T = buf.view(2, R, 8).cpu().numpy().astype(np.float64)
out = {}
for h in range(2):
    t = T[h]
    ok = (t[:, 1] > 0) & (t[:, 2] > 0)
    rows = np.nonzero(ok)[0]
    r = rows[(rows > 50) & (rows < rows.max() - 50)]
    per = np.diff(t[r, 1])
    lag_rows = 2  # informational
    res = {
        "row_period": float(np.median(per)),
        "dot (start->published, warp 0)": float(np.median(t[r, 2] - t[r, 1])),
        "tma issue->dot start": float(np.median(t[r, 1] - t[r, 0])),
        "published->dots complete (prox)": float(np.median(t[r, 5] - t[r, 2])),
        "prox compute (dots complete->q)": float(np.median(t[r, 6] - t[r, 5])),
        "q published->q seen (warp 0)": float(np.median(t[r, 3] - t[r, 6])),
        "dot start->q seen": float(np.median(t[r, 3] - t[r, 1])),
        "q seen->slot released": float(np.median(t[r, 4] - t[r, 3])),
    }
    out[f"cta{h}"] = res
print(json.dumps({"dtype": a.dtype, "loss": a.loss, "n": a.n, **out}, indent=1))
if a.out:
    np.save(a.out, T)
