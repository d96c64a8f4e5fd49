"""Small solves for compute-sanitizer: one case per invocation so each
sanitizer tool runs on a handful of launches of the kernel under test.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py fused4_g3

Cases: fused4_g{1,2,3,4,6} (the CTA-pair single-pass sweep at each compiled row-group
count, several nodes so node boundaries fall inside clusters), fused4_n2000 (ADVICE r1:
26 ring slots, 6 groups, the slot-reuse bound), fused4_f32, gram_tc (the tcgen05 Ozaki
Gram k_oz_mm128 and the factor), gemv_t_tma (C = 10 softmax: k_gemv_t_dmma_tma,
k_gemv_dmma), woodbury (fat blocks), emu2 (two emulated ranks, split block sums).
"""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2405_16267_b200 import bicadmm as bc  # noqa: E402
from paper_2405_16267_b200 import datagen as dg  # noqa: E402


def solve(N, m, n, kappa, loss, M=1, C=1, sweep=0, dtype=torch.float64, K=1, K_in=2):
    P = dg.generate(N, m, n, kappa, loss, C=C, seed=5)
    cs = dg.block_partition(n, M)
    prm = bc.Params(kappa=kappa, max_outer=K, inner_fixed=K_in, refit=0, eps_p=0, eps_d=0, eps_b=0, sweep=sweep)
    s = bc.BiCADMM([a.to("cuda", dtype) for a in P.A], [b.to("cuda", dtype) for b in P.b], loss, prm, cs, C=P.C)
    s.iterate(K)
    torch.cuda.synchronize()
    kind = s.sweep_kind()
    s.close()
    return kind


def emu2():
    P = dg.generate(1, 400, 200, 8, "logistic", seed=5)
    cs = dg.block_partition(200, 2)
    grp = bc.bicadmm_emu_group_create(2)
    out = [None, None]
    comms = [bc.bicadmm_comm_init_emu(grp, r, 0, 0) for r in range(2)]

    def rank(r):
        torch.cuda.set_device(0)
        comm = comms[r]
        prm = bc.Params(kappa=8, max_outer=1, inner_fixed=2, refit=0, eps_p=0, eps_d=0, eps_b=0)
        A = P.A[0].cuda()
        s = bc.BiCADMM(None, [P.b[0].cuda()], "logistic", prm, cs, blocks=[(0, r, A[:, cs[r]:cs[r + 1]])],
                       comm=comm, stream=torch.cuda.Stream())
        s.iterate(1)
        torch.cuda.synchronize()
        out[r] = s.z
        s.close()

    th = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for c in comms:
        bc.bicadmm_comm_destroy(c)
    bc.bicadmm_emu_group_destroy(grp)
    return out[0] is not None and out[1] is not None


def main(case):
    if case.startswith("fused4_g"):
        os.environ["BICADMM_F4_GROUPS"] = case[len("fused4_g"):]
        print(solve(3, 211, 496, 9, "logistic", sweep=2))
    elif case == "fused4_n2000":
        print(solve(1, 700, 2000, 9, "logistic", sweep=2))
    elif case == "fused4_f32":
        print(solve(2, 300, 1000, 9, "hinge", sweep=2, dtype=torch.float32))
    elif case == "gram_tc":
        print(solve(1, 600, 512, 9, "ls", sweep=1))
    elif case == "gemv_t_tma":
        print(solve(1, 300, 96, 9, "softmax", M=2, C=10, sweep=1))
    elif case == "woodbury":
        print(solve(2, 60, 200, 9, "logistic", M=2, sweep=1))
    elif case == "emu2":
        print(emu2())
    else:
        raise SystemExit(f"unknown case {case}")


if __name__ == "__main__":
    main(sys.argv[1])
