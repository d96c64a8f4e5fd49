"""Device time of the one-time Gram (C2 block: 25,000 x 10,000 FP64): DMMA vs tcgen05 Ozaki."""
import ctypes as ct
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2405_16267_b200 import bicadmm as bc

m, n = (int(a) for a in sys.argv[1:3]) if len(sys.argv) > 2 else (25000, 10000)
A = torch.randn(m, n, dtype=torch.float64, device="cuda") / m ** 0.5
G = torch.zeros(n, n, dtype=torch.float64, device="cuda")
G2 = torch.zeros(n, n, dtype=torch.float64, device="cuda")
L = bc.lib()
wsb = L.bicadmm_op_gram_tc_ws(bc.F64, m, n)
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
s = ct.c_void_p(torch.cuda.current_stream().cuda_stream)
p = lambda t: ct.c_void_p(t.data_ptr())
for rep in range(3):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    bc.check(L.bicadmm_op_gram(bc.F64, m, n, p(A), A.stride(0), 1.0, 0.0, p(G), n, s))
    e[1].record()
    bc.check(L.bicadmm_op_gram_tc(bc.F64, m, n, p(A), A.stride(0), 1.0, 0.0, p(G2), n, p(ws), wsb, s))
    e[2].record()
    torch.cuda.synchronize()
    lo = torch.tril(torch.ones(n, n, dtype=torch.bool, device="cuda"))
    d = torch.sqrt(torch.diag(G).abs())
    err = ((G - G2).abs() / torch.outer(d, d))[lo].max().item()
    print(f"{m} x {n}: DMMA {e[0].elapsed_time(e[1]):.1f} ms, tcgen05 Ozaki {e[1].elapsed_time(e[2]):.1f} ms, "
          f"max rel diff {err:.2e}", flush=True)
