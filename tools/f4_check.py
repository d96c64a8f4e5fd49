"""Protocol check of the single-pass sweep (k_fused4) on a BIC_F4_CHECK build.

    tools/build_f4_variant.sh f4check -DBIC_F4_CHECK
    BICADMM_LIB_PATH=build_ab/f4check.so python tools/f4_check.py [--quick]

Runs the sweep over row widths, dtypes and forced plans (row batches R, row groups GR, axpy
delay D, ring depth), several ragged nodes so node boundaries fall inside clusters, and
reports the slot-tag mismatches the check build counts (must be 0) plus the deviation of z
from the independent two-pass sweep after a few outer iterations (FP64 <= 1e-9)."""
import argparse
import ctypes as ct
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2405_16267_b200 import bicadmm as bc  # noqa: E402
from paper_2405_16267_b200 import datagen as dg  # noqa: E402


def errors():
    f = bc.lib().bicadmm_debug_f4_errors
    f.restype = ct.c_ulonglong
    return int(f())


def run(n, dt, loss, env, K=3, K_in=3):
    ms = (n + 301, n + 77, n + 504)   # ragged tall nodes (the single pass takes tall blocks)
    for k, v in env.items():
        os.environ[k] = str(v)
    try:
        P = dg.generate(len(ms), list(ms), n, 10, loss, seed=n)
        cs = dg.block_partition(n, 1)
        dtype = torch.float64 if dt == "f64" else torch.float32
        out = {}
        lda = -(-n // 4) * 4   # rows padded to 16 bytes; the padding holds NaN (never read)
        A = []
        for a in P.A:
            t = torch.full((a.shape[0], lda), float("nan"), dtype=dtype, device="cuda")
            t[:, :n] = a.to("cuda", dtype)
            A.append(t[:, :n])
        for sweep in (1, 2):
            s = bc.BiCADMM(A, [b.to("cuda", dtype) for b in P.b], loss,
                           bc.Params(kappa=10, max_outer=50, inner_fixed=K_in, refit=0, eps_p=0, eps_d=0, eps_b=0,
                                     sweep=sweep), cs)
            s.iterate(K)
            out[sweep] = (s.z, s.sweep_kind())
            s.close()
        z2, z1 = out[2][0], out[1][0]
        rel = float(np.linalg.norm(z2 - z1) / max(np.linalg.norm(z1), 1e-300))
        return rel, out[2][1]
    finally:
        for k in env:
            os.environ.pop(k, None)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--widths", default="", help="comma-separated row widths (default: the built-in list)")
    a = ap.parse_args()
    widths = [300, 1000, 1502, 2000, 4000, 6250, 10000] if a.quick else [300, 496, 1000, 1502, 2000, 4000, 6248, 6250, 10000, 12500, 13300]
    if a.widths:
        widths = [int(w) for w in a.widths.split(",")]
    plans = [{}, {"BICADMM_F4_R": 1}, {"BICADMM_F4_R": 2}, {"BICADMM_F4_R": 4}, {"BICADMM_F4_GROUPS": 1},
             {"BICADMM_F4_GROUPS": 2}, {"BICADMM_F4_GROUPS": 6, "BICADMM_F4_R": 2}, {"BICADMM_F4_D": 1},
             {"BICADMM_F4_D": 3}, {"BICADMM_F4_RING": 4}]
    if a.quick:
        plans = plans[:4] + plans[6:7]
    if not bc.lib().bicadmm_debug_f4_check_build():   # a product build counts nothing
        print(json.dumps({"error": "not a BIC_F4_CHECK build: set BICADMM_LIB_PATH to build_ab/f4check.so"}))
        return 2
    rows, worst, total0 = [], 0.0, errors()
    for n, dt, plan in itertools.product(widths, ("f64", "f32"), plans):
        loss = "logistic" if n % 3 else "hinge"
        e0 = errors()
        rel, kind = run(n, dt, loss, plan)
        e1 = errors()
        rows.append({"n": n, "dtype": dt, "loss": loss, "plan": plan, "kind": kind, "tag_errors": e1 - e0,
                     "rel_z_vs_two_pass": rel})
        if dt == "f64":
            worst = max(worst, rel)
        print(json.dumps(rows[-1]), flush=True)
    summary = {"runs": len(rows), "check_build": True, "tag_errors": errors() - total0, "worst_rel_f64": worst,
               "fused_runs": sum(1 for r in rows if r["kind"][0] == 4)}
    print(json.dumps({"summary": summary}))
    return 0 if summary["tag_errors"] == 0 and worst <= 1e-9 else 1


if __name__ == "__main__":
    sys.exit(main())
