"""Kernel microbenchmarks (CUDA events) for the HBM passes at C2 scale.

    python tools/microbench.py [--m 100000] [--n 10000] [--dtype f64]

Times bicadmm_op_gemv (p = A x) and bicadmm_op_gemv_t (r = A^T q + ...) on one
m x n matrix (A larger than L2), reports GB/s of algorithmic bytes vs the
measured HBM peak.  Diagnostic only; bench.py is the contract.
"""
import argparse
import ctypes as ct
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2405_16267_b200 import bicadmm as bc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=100_000)
    ap.add_argument("--n", type=int, default=10_000)
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    tdt = torch.float64 if a.dtype == "f64" else torch.float32
    dt = bc.F64 if a.dtype == "f64" else bc.F32
    s = 8 if a.dtype == "f64" else 4
    L = bc.lib()
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(a.m, a.n, generator=g, device="cuda", dtype=torch.float64).to(tdt)
    x = torch.randn(a.n, device="cuda", dtype=torch.float64)
    y = torch.zeros(a.m, device="cuda", dtype=torch.float64)
    p = torch.randn(a.m, device="cuda", dtype=torch.float64)
    r = torch.zeros(a.n, device="cuda", dtype=torch.float64)
    wsb = L.bicadmm_op_gemv_t_ws(dt, a.m, a.n)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    st = ct.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = lambda t: ct.c_void_p(t.data_ptr())
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)
    res = {}
    for name, fn, byt in [
        ("gemv", lambda: L.bicadmm_op_gemv(dt, a.m, a.n, P(A), a.n, P(x), P(y), st), a.m * a.n * s + 8 * (a.m + a.n)),
        ("gemv_t", lambda: L.bicadmm_op_gemv_t(dt, a.m, a.n, P(A), a.n, P(p), None, None, None, 1.0, 0.0, P(r), P(ws),
                                             wsb, st), a.m * a.n * s + 8 * a.m),
    ]:
        for _ in range(3):
            bc.check(fn())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        res[name] = dict(ms=ms, GBps=byt / ms / 1e6, frac=byt / ms / 1e6 / peak)
    # plain copy reference of the same bytes (torch) for context
    B = torch.empty_like(A)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    B.copy_(A)
    e0.record()
    for _ in range(a.reps):
        B.copy_(A)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    res["torch_copy"] = dict(ms=ms, GBps=2 * A.numel() * s / ms / 1e6)
    res["torch_sum_read"] = {}
    e0.record()
    for _ in range(a.reps):
        A.sum(dim=1)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    res["torch_sum_read"] = dict(ms=ms, GBps=A.numel() * s / ms / 1e6)
    print(json.dumps(dict(m=a.m, n=a.n, dtype=a.dtype, env={k: v for k, v in os.environ.items() if k.startswith("BICADMM")},
                          **res)))


if __name__ == "__main__":
    main()
