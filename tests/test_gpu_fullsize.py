"""Full-size checks at BASELINE.json's configs[1] (the bench workload: logistic, 4 nodes x
25,000 x 10,000 FP64, kappa = 100, K_in = 10) in the launch configuration bench.py times
(the CTA-pair single-pass sweep).  The oracle cannot run this size in seconds, so:

* the single-pass kernel and the independent two-pass GEMV-T / H-apply / GEMV / prox
  kernels must agree to 1e-9 after 3 outer iterations (30 sweeps);
* sampled rows of p_i = A_i x_i are recomputed one by one in FP64 on the host;
* the x-update normal equations (rho_l A^T A + c I) x = r (Eq. (24), DESIGN R17) hold to
  1e-10 on every node (full FP64 host mat-vecs);
* the global step's exact invariants hold at full size.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2405_16267_b200 import datagen as dg  # noqa: E402

N, M_I, NN, KAPPA = 4, 25_000, 10_000, 100


@pytest.fixture(scope="module")
def bc():
    from paper_2405_16267_b200 import build
    build.build()
    from paper_2405_16267_b200 import bicadmm
    bicadmm.lib()
    return bicadmm


def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


def test_configs1_full_size(bc):
    P = dg.generate(N, M_I, NN, KAPPA, "logistic", seed=1000, device="cuda")   # bench.py's data (rank 0)
    cs = dg.block_partition(NN, 1)
    prm = dict(kappa=KAPPA, inner_fixed=10, max_outer=100, eps_p=0.0, eps_d=0.0, eps_b=0.0, refit=0)
    res = {}
    for sweep in (0, 1):
        s = bc.BiCADMM(P.A, P.b, "logistic", bc.Params(sweep=sweep, **prm), cs)
        if sweep == 0:
            assert s.sweep_kind() == (4, 0)   # the bench's launch configuration
        else:
            assert s.sweep_kind() == (0, 0)
        s.iterate(3)
        res[sweep] = dict(z=s.z, svec=s.s, x=s.get(bc.FIELD_X_LOCAL), p=s.get(bc.FIELD_P_LOCAL),
                          r=s.get(bc.FIELD_R_LOCAL), sc=s.scalars(), trace=s.trace())
        s.close()
    f, t = res[0], res[1]
    # 1. two independent kernel paths agree
    assert _rel(f["z"], t["z"]) <= 1e-9
    assert _rel(f["x"], t["x"]) <= 1e-9
    assert _rel(f["p"], t["p"]) <= 1e-9
    for k in ("t", "p_r", "d_r"):
        assert abs(f["sc"][k] - t["sc"][k]) <= 1e-9 * max(abs(t["sc"][k]), 1e-300)
    # 2. p = A x on sampled rows, and 3. (rho_l A^T A + c I) x = r, per node, FP64 on the host
    rho_l, c = 4.0, 1.0 / (100.0 * N) + 4.0
    rng = np.random.default_rng(0)
    for i in range(N):
        A = P.A[i].cpu().numpy()
        x = f["x"][i * NN:(i + 1) * NN]
        p = f["p"][i * M_I:(i + 1) * M_I]
        r = f["r"][i * NN:(i + 1) * NN]
        rows = rng.choice(M_I, 256, replace=False)
        ref_rows = A[rows] @ x
        assert np.max(np.abs(ref_rows - p[rows])) <= 1e-12 * max(1.0, np.max(np.abs(ref_rows)))
        Fx = rho_l * (A.T @ (A @ x)) + c * x
        assert _rel(Fx, r) <= 1e-10, i
    # 4. global-step invariants (exact; App. A.4): s in S^kappa, ||z||_1 <= t, tail_kappa(z) <= b_r
    z, s, sc = f["z"], f["svec"], f["sc"]
    assert np.max(np.abs(s)) <= 1.0 + 1e-15
    assert np.abs(s).sum() <= KAPPA * (1 + 1e-12)
    assert np.count_nonzero(s) <= KAPPA
    assert np.abs(z).sum() <= sc["t"] * (1 + 1e-12) + 1e-12
    tail = np.sort(np.abs(z))[: max(0, z.size - KAPPA)].sum()
    assert tail <= sc["b_r"] * (1 + 1e-9) + 1e-12


def test_configs3_full_size(bc):
    # BASELINE.json configs[3] on one GPU, the bench's C4 launch configuration: softmax, C = 10,
    # 1 node x 500,000 x 20,000 FP64 (80 GB), M = 8 feature blocks (7 x 2,512 + 2,416 columns),
    # the DMMA GEMV-C / GEMV-T-C two-pass sweep.  After one outer iteration of K_in = 2:
    # sampled rows of p_ij = A_ij x_ij recomputed one by one in FP64 on the host, and every
    # block's x-update normal equations (rho_l A_ij^T A_ij + c I) x_ij = r_ij (Eq. (24), R17)
    # checked with FP64 library mat-vecs (torch) on the device.
    free, _ = torch.cuda.mem_get_info()
    if free < 120 * 2**30:
        pytest.skip("needs ~120 GB of free device memory")
    Nn, m, n, C, M, kappa = 1, 500_000, 20_000, 10, 8, 500
    P = dg.generate(Nn, m, n, kappa, "softmax", C=C, seed=1000, device="cuda")
    cs = dg.block_partition(n, M, align=16)
    assert [cs[j + 1] - cs[j] for j in range(M)] == [2512] * 7 + [2416]
    s = bc.BiCADMM(P.A, P.b, "softmax", bc.Params(kappa=kappa, inner_fixed=2, max_outer=10, eps_p=0.0, eps_d=0.0,
                                                  eps_b=0.0, refit=0), cs, C=C)
    assert s.sweep_kind() == (0, 0)
    s.iterate(1)
    x = s.get(bc.FIELD_X_LOCAL)
    p = s.get(bc.FIELD_P_LOCAL)
    r = s.get(bc.FIELD_R_LOCAL)
    s.close()
    A = P.A[0]
    rng = np.random.default_rng(3)
    rows = np.sort(rng.choice(m, 256, replace=False))
    Ar = A[torch.from_numpy(rows).cuda()].cpu().numpy()
    rho_l, c = 4.0, 1.0 / (100.0 * Nn) + 4.0
    xo, po = 0, 0
    for j in range(M):
        nj = cs[j + 1] - cs[j]
        Xj = x[xo:xo + nj * C].reshape(nj, C)
        Pj = p[po:po + m * C].reshape(m, C)
        Rj = r[xo:xo + nj * C].reshape(nj, C)
        ref_rows = Ar[:, cs[j]:cs[j + 1]] @ Xj
        assert np.max(np.abs(ref_rows - Pj[rows])) <= 1e-12 * max(1.0, np.max(np.abs(ref_rows))), j
        Aj = A[:, cs[j]:cs[j + 1]]
        Xt = torch.from_numpy(Xj).cuda()
        F = rho_l * (Aj.T @ (Aj @ Xt)) + c * Xt
        assert _rel(F.cpu().numpy(), Rj) <= 1e-10, j
        xo += nj * C
        po += m * C
