"""Degenerate and boundary cases of the whole path through the C ABI against the oracle
(same seeded inputs, iterate by iterate): kappa at its extremes (0, 1, n), one column,
one node, one-row nodes (fat blocks: the Woodbury path with a 1 x 1 K), very ragged
node sizes, one sweep per outer iteration, all-zero labels, and the rejected empty node.

Bar as in test_gpu_solver.py (north star; DESIGN R22): FP64 outer iterates z^k within
1e-9 relative, identical support."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2405_16267_b200 import datagen as dg  # noqa: E402


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


LOSS_ID = {"ls": 0, "logistic": 1, "hinge": 2}


def _run(bc, orc, A, b, loss, cs, kappa, K, K_in, sweep=0):
    prm = dict(kappa=kappa, max_outer=K, inner_fixed=K_in, refit=0, eps_p=0.0, eps_d=0.0, eps_b=0.0)
    s = bc.BiCADMM([a.cuda() for a in A], [x.cuda() for x in b], loss, bc.Params(sweep=sweep, **prm), cs)
    zs = []
    for _ in range(K):
        s.iterate(1)
        zs.append(s.z)
    s.finalize()
    lid = {"ls": orc.LS, "logistic": orc.LOGISTIC, "hinge": orc.HINGE}[loss]
    # bicadmm_iterate runs a fixed count; the oracle gets negative tolerances so that residuals
    # of exactly 0 (x = z = 0 after the first outer iteration when K_in = 1) do not stop it
    oprm = dict(prm, eps_p=-1.0, eps_d=-1.0, eps_b=-1.0)
    ref = orc.run(orc.Problem([a.numpy() for a in A], [x.numpy() for x in b], lid, 1, np.array(cs)),
                  orc.Params(**oprm), trace_z=True)
    assert len(ref["z_trace"]) == K
    for k in range(K):
        assert np.all(np.isfinite(zs[k])), k
        assert _rel(zs[k], ref["z_trace"][k]) <= 1e-9, (k, _rel(zs[k], ref["z_trace"][k]))
    sup = s.support().tolist()
    assert sup == ref["support"].tolist()
    kind = s.sweep_kind()
    s.close()
    return zs, ref, sup, kind


CASES = [
    # name, N, m_i (int or per-node list), n, kappa (data), kappa (solver), loss, M, K_outer, K_in
    ("kappa_eq_n", 2, 60, 12, 4, 12, "ls", 1, 10, 3),
    ("kappa_one", 2, 80, 20, 3, 1, "logistic", 1, 10, 3),
    ("kappa_zero", 2, 50, 16, 3, 0, "ls", 1, 8, 3),
    ("one_column", 2, 30, 1, 1, 1, "ls", 1, 10, 3),
    ("one_node_two_blocks", 1, 200, 40, 5, 5, "hinge", 2, 10, 3),
    ("one_row_nodes", 3, [1, 1, 1], 8, 2, 2, "ls", 1, 10, 3),
    ("ragged_1_and_500", 2, [1, 500], 24, 4, 4, "logistic", 2, 8, 3),
    ("one_sweep_per_outer", 3, 150, 60, 6, 6, "logistic", 3, 12, 1),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_edge_case_matches_oracle(bc, orc, case):
    _, N, m, n, kd, ks, loss, M, K, K_in = case
    P = dg.generate(N, m, n, kd, loss, seed=101)
    cs = dg.block_partition(n, M)
    zs, ref, sup, _ = _run(bc, orc, P.A, P.b, loss, cs, ks, K, K_in)
    if ks == 0:
        assert sup == []                      # T is empty: s = 0, no support
    if ks == n:
        assert len(sup) == int(np.count_nonzero(zs[-1]))   # every nonzero coordinate is in T


@pytest.mark.parametrize("sweep", [1, 2], ids=["two_pass", "fused"])
def test_zero_labels_stay_at_zero(bc, orc, sweep):
    # LS with b = 0 from x = 0: every iterate of (5)-(15) is exactly zero (the consensus
    # point is the origin; Mcap = 0 takes the guarded branch of (13)); both sweeps
    P = dg.generate(2, 300, 40, 4, "ls", seed=3)
    b = [torch.zeros_like(x) for x in P.b]
    zs, ref, sup, kind = _run(bc, orc, P.A, b, "ls", dg.block_partition(40, 1), 4, 6, 3, sweep=sweep)
    assert all(np.count_nonzero(z) == 0 for z in zs)
    assert sup == []
    if sweep == 2:
        assert kind[0] == 4


def test_empty_node_rejected(bc):
    # m_i = 0: bicadmm_setup returns BICADMM_ERR_DIM (validate: "m_i must be >= 1")
    P = dg.generate(2, 40, 16, 2, "ls", seed=1)
    A = [P.A[0].cuda(), torch.zeros(0, 16, dtype=torch.float64, device="cuda")]
    b = [P.b[0].cuda(), torch.zeros(0, dtype=torch.float64, device="cuda")]
    with pytest.raises(bc.BicadmmError) as e:
        bc.BiCADMM(A, b, "ls", bc.Params(kappa=2), dg.block_partition(16, 1))
    assert e.value.rc == bc.ERR_DIM


def test_solve_stops_where_the_oracle_stops_on_exact_zero_residuals(bc, orc):
    # K_in = 1 from x = 0: q = p + delta = 0 in the first sweep, so x = H r = 0, z = 0 and
    # p_r = d_r = b_r = 0 -- the tests p_r <= eps_p, d_r <= eps_d, b_r <= eps_b (15) hold with
    # eps = 0 after one outer iteration, on the device-side loop as in the oracle
    P = dg.generate(3, 150, 60, 6, "logistic", seed=101)
    cs = dg.block_partition(60, 3)
    prm = dict(kappa=6, max_outer=50, inner_fixed=1, refit=0, eps_p=0.0, eps_d=0.0, eps_b=0.0)
    s = bc.BiCADMM([a.cuda() for a in P.A], [x.cuda() for x in P.b], "logistic", bc.Params(**prm), cs)
    rep = s.solve()
    ref = orc.run(orc.Problem([a.numpy() for a in P.A], [x.numpy() for x in P.b], orc.LOGISTIC, 1, np.array(cs)),
                  orc.Params(**prm))
    assert ref["iters"] == 1 and ref["converged"]
    assert rep.outer_iters == 1 and rep.converged == 1
    assert np.count_nonzero(s.z) == 0
    s.close()


# Capacity boundaries of the launch batching: more nodes than one small-sweeps launch takes
# (24), more local blocks than one descriptor batch (64), the single pass's node table (32),
# and the largest class count (C = 16).
BOUNDARY_CASES = [
    # name, N, m_i, n, kappa, loss, M, K_outer, K_in, C, expected sweep kind (None: any)
    ("small_nodes_30_two_launches", 30, 60, 20, 3, "logistic", 1, 6, 3, 1, 5),
    ("blocks_20x4_two_desc_batches", 20, 120, 64, 6, "ls", 4, 6, 3, 1, None),
    ("fused_32_nodes", 32, 720, 704, 8, "logistic", 1, 3, 2, 1, 4),
    ("fused_33_nodes_falls_back", 33, 720, 704, 8, "logistic", 1, 3, 2, 1, 0),
    ("softmax_c16", 2, 400, 40, 8, "softmax", 2, 6, 3, 16, None),
    ("nine_blocks_past_small_path", 2, 200, 72, 6, "logistic", 9, 6, 3, 1, 0),
    ("fat_at_m_eq_n_minus_1", 2, 63, 64, 5, "ls", 1, 8, 3, 1, None),
    ("tall_at_m_eq_n", 2, 64, 64, 5, "ls", 1, 8, 3, 1, None),
]


@pytest.mark.parametrize("case", BOUNDARY_CASES, ids=[c[0] for c in BOUNDARY_CASES])
def test_capacity_boundaries_match_oracle(bc, orc, case):
    _, N, m, n, kappa, loss, M, K, K_in, C, kind = case
    P = dg.generate(N, m, n, kappa, loss, seed=77, C=C)
    cs = dg.block_partition(n, M)
    prm = dict(kappa=kappa, max_outer=K, inner_fixed=K_in, refit=0, eps_p=0.0, eps_d=0.0, eps_b=0.0)
    s = bc.BiCADMM([a.cuda() for a in P.A], [x.cuda() for x in P.b], loss, bc.Params(**prm), cs, C=C)
    if kind is not None:
        assert s.sweep_kind()[0] == kind, s.sweep_kind()
    zs = []
    for _ in range(K):
        s.iterate(1)
        zs.append(s.z)
    s.finalize()
    lid = {"ls": orc.LS, "logistic": orc.LOGISTIC, "hinge": orc.HINGE, "softmax": orc.SOFTMAX}[loss]
    oprm = dict(prm, eps_p=-1.0, eps_d=-1.0, eps_b=-1.0)
    ref = orc.run(orc.Problem([a.numpy() for a in P.A], [x.numpy() for x in P.b], lid, C, np.array(cs)),
                  orc.Params(**oprm), trace_z=True)
    for k in range(K):
        assert _rel(zs[k], ref["z_trace"][k]) <= 1e-9, (k, _rel(zs[k], ref["z_trace"][k]))
    assert s.support().tolist() == ref["support"].tolist()
    s.close()


def test_tol_mode_on_small_nodes(bc, orc):
    # the inner tolerance mode on a problem whose fixed schedule takes the small-nodes
    # path (kind 5): per-node sweep counts decided on the device values, replayed by the oracle
    P = dg.generate(3, 100, 40, 5, "logistic", seed=12)
    cs = dg.block_partition(40, 1)
    K = 6
    prm = dict(kappa=5, max_outer=K, inner_fixed=0, eps_inner=1e-6, max_inner=40, refit=0,
               eps_p=0.0, eps_d=0.0, eps_b=0.0)
    s = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "logistic", bc.Params(**prm), cs)
    s.iterate(K)
    counts = s.get(bc.FIELD_INNER_COUNTS, np.int32).reshape(K, 3)
    pb = orc.Problem([a.numpy() for a in P.A], [b.numpy() for b in P.b], orc.LOGISTIC, 1, np.array(cs))
    oprm = dict(prm, eps_p=-1.0, eps_d=-1.0, eps_b=-1.0)
    own = orc.run(pb, orc.Params(**oprm))
    rep = orc.run(pb, orc.Params(**oprm), schedule=counts)
    assert counts.min() >= 1 and counts.max() <= 40
    assert _rel(s.z, rep["z"]) <= 1e-9
    assert np.mean(counts == own["inner_counts"]) >= 0.8
    s.close()
    # the same problem with a fixed schedule runs on the small-nodes kernel
    s = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "logistic",
                   bc.Params(**dict(prm, inner_fixed=4)), cs)
    assert s.sweep_kind()[0] == 5
    s.close()
