"""Error pattern of the tcgen05 Ozaki Gram against the FP64 definition (small shapes)."""
import ctypes as ct
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2405_16267_b200 import bicadmm as bc
L = bc.lib()
s = ct.c_void_p(torch.cuda.current_stream().cuda_stream)
p = lambda t: ct.c_void_p(t.data_ptr())
for (m, nj, sc) in [(517, 70, 0), (517, 70, 6), (40000, 300, 0), (2000, 256, 0), (32, 128, 0), (64, 64, 0)]:
    rng = np.random.default_rng(m + nj)
    An = rng.normal(size=(m, -(-nj // 4) * 4)) * np.exp(rng.uniform(-sc, sc, size=-(-nj // 4) * 4))
    A = torch.tensor(An, device="cuda", dtype=torch.float64)
    G = torch.zeros((nj, nj), dtype=torch.float64, device="cuda")
    wsb = L.bicadmm_op_gram_tc_ws(bc.F64, m, nj)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    bc.check(L.bicadmm_op_gram_tc(bc.F64, m, nj, p(A), A.stride(0), 1.0, 0.0, p(G), nj, p(ws), wsb, s))
    torch.cuda.synchronize()
    Gn = G.cpu().numpy()
    An = An[:, :nj]
    ref = An.T @ An
    lo = np.tril_indices(nj)
    d = np.sqrt(np.abs(np.diag(ref)))
    E = np.abs(Gn - ref) / np.outer(d, d)
    E = np.tril(E)
    i, j = np.unravel_index(np.argmax(E), E.shape)
    print(f"m={m} nj={nj} sc={sc}: max rel err {E.max():.2e} at ({i},{j}); median {np.median(E[lo]):.2e}; "
          f"diag max {np.max(np.diag(E)):.2e}; rows>1e-13: {np.unique(np.where(E > 1e-13)[0])[:12]} "
          f"cols>1e-13: {np.unique(np.where(E > 1e-13)[1])[:12]}", flush=True)
