"""End-to-end GPU parity: the whole hot path through the C ABI (bicadmm_setup /
bicadmm_iterate / bicadmm_finalize) against the oracle's run on the same seeded
inputs, iterate by iterate.

Bar (north star; DESIGN R22): FP64 -> every outer iterate z^k, t^k, v^k and the
residuals within 1e-9 relative, identical support, objective within 1e-9.
FP32 storage -> within 1e-4 against the oracle run on the FP64 data, identical
support."""
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


def run_pair(bc, orc, N, m, n, kappa, loss, M, K, K_in, seed=0, dtype=torch.float64, C=1, sweep=0, **kw):
    P = dg.generate(N, m, n, kappa, loss, seed=seed, C=C)
    cs = dg.block_partition(n, M)
    oprm = dict(kappa=kappa, max_outer=K, inner_fixed=K_in, refit=0, eps_p=0.0, eps_d=0.0, eps_b=0.0, **kw)
    solver = bc.BiCADMM([a.to("cuda", dtype) for a in P.A], [b.to("cuda", dtype) for b in P.b], loss,
                        bc.Params(sweep=sweep, **oprm), cs, C=P.C)
    zs, xs = [], []
    for _ in range(K):
        solver.iterate(1)
        zs.append(solver.z)
        xs.append(solver.get(bc.FIELD_X_LOCAL))
    rep = solver.finalize()
    lid = {"ls": orc.LS, "logistic": orc.LOGISTIC, "hinge": orc.HINGE, "softmax": orc.SOFTMAX}[loss]
    Aref = [a.to(dtype).double().numpy() for a in P.A]
    bref = [b.to(dtype).double().numpy() for b in P.b]
    ref = orc.run(orc.Problem(Aref, bref, lid, P.C, np.array(cs)), orc.Params(**oprm), trace_z=True, trace_x=True)
    return solver, rep, np.array(zs), np.array(xs), ref, P


CASES = [
    # name, N, m_i, n, kappa, loss, M, K_outer, K_in[, C]
    ("c1_ls", 2, 100, 50, 5, "ls", 1, 40, 10),
    ("softmax_c4_replica_M8", 1, 1500, 200, 20, "softmax", 8, 8, 4, 10),
    ("softmax_c3_blocks2", 2, 300, 61, 6, "softmax", 2, 10, 5, 3),
    ("ls_blocks3", 2, 300, 250, 12, "ls", 3, 25, 5),
    ("logistic_c2_replica", 4, 600, 300, 10, "logistic", 1, 20, 10),
    ("hinge_blocks2", 3, 400, 201, 8, "hinge", 2, 20, 5),
    ("logistic_blocks4_ragged", 2, 1037, 1030, 15, "logistic", 4, 8, 4),
]


@pytest.mark.parametrize("sweep", [1, 2], ids=["two_pass", "fused"])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_fp64_iterates_match_oracle(bc, orc, case, sweep):
    _, N, m, n, kappa, loss, M, K, K_in = case[:9]
    C = case[9] if len(case) > 9 else 1
    if sweep == 2 and (C > 1 or M > 1 or n % 2):
        pytest.skip("the single-pass sweep takes one block per node, C == 1 and 16-byte half-rows")
    solver, rep, zs, xs, ref, _ = run_pair(bc, orc, N, m, n, kappa, loss, M, K, K_in, C=C, sweep=sweep)
    _check_fp64(solver, rep, zs, xs, ref, K)


def _check_fp64(solver, rep, zs, xs, ref, K):
    tr_g = solver.trace()
    tr_o = ref["trace"]
    assert tr_g.shape == tr_o.shape
    for k in range(K):
        assert _rel(zs[k], ref["z_trace"][k]) <= 1e-9, (k, _rel(zs[k], ref["z_trace"][k]))
        # x_i (local blocks concatenated in node order = full x_i for single-rank placement)
        assert _rel(xs[k], ref["x_trace"][k].ravel()) <= 1e-9, k
        t_o, v_o = tr_o[k, 3], tr_o[k, 4]
        assert abs(tr_g[k, 3] - t_o) <= 1e-9 * max(abs(t_o), 1e-300)
        assert abs(tr_g[k, 4] - v_o) <= 1e-9 * max(abs(v_o), abs(t_o))
        for c in (0, 1):   # p_r, d_r relative to their first-iteration scale (DESIGN R22)
            assert abs(tr_g[k, c] - tr_o[k, c]) <= 1e-9 * max(abs(tr_o[k, c]), abs(tr_o[0, c]))
        assert abs(tr_g[k, 2] - tr_o[k, 2]) <= 1e-9 * max(abs(tr_o[k, 2]), abs(t_o))
    assert solver.support().tolist() == ref["support"].tolist()
    assert abs(rep.objective - ref["objective"]) <= 1e-9 * abs(ref["objective"])


def test_c1_solve_to_tolerance_recovers_brute_force_support(bc, orc):
    # configs[0]: solve to eps = 1e-4 on the GPU; support equals exhaustive best subset
    P = dg.generate(2, 100, 50, 5, "ls", seed=3)
    cs = dg.block_partition(50, 1)
    solver = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "ls",
                        bc.Params(kappa=5, max_outer=2000, inner_fixed=10), cs)
    rep = solver.solve()
    pb = orc.Problem([a.numpy() for a in P.A], [b.numpy() for b in P.b], orc.LS, 1, np.array(cs))
    sup, _, _ = orc.best_subset(pb, 100.0, 5)
    assert rep.converged == 1
    assert solver.support().tolist() == sup.tolist()
    ref = orc.run(pb, orc.Params(kappa=5, max_outer=2000, inner_fixed=10, refit=0))
    assert rep.outer_iters == ref["iters"]
    assert abs(rep.objective - ref["objective"]) <= 1e-9 * abs(ref["objective"])


@pytest.mark.parametrize("sweep", [1, 2], ids=["two_pass", "fused"])
def test_fp32_mode_within_1e4(bc, orc, sweep):
    # FP32 storage of A, b, H; FP64 iterates and accumulation (DESIGN R23)
    solver, rep, zs, xs, ref, _ = run_pair(bc, orc, 4, 600, 300, 10, "logistic", 1, 15, 10, dtype=torch.float32,
                                           sweep=sweep)
    for k in range(15):
        assert _rel(zs[k], ref["z_trace"][k]) <= 1e-4, k
    assert solver.support().tolist() == ref["support"].tolist()
    assert abs(rep.objective - ref["objective"]) <= 1e-4 * abs(ref["objective"])


FP32_CASES = [
    # name, N, m_i, n, kappa, loss, M, K_outer, K_in[, C]
    ("ls_blocks3", 2, 300, 250, 12, "ls", 3, 12, 5),
    ("hinge_blocks2", 3, 400, 201, 8, "hinge", 2, 12, 5),
    ("softmax_c10_blocks8", 1, 1500, 200, 20, "softmax", 8, 6, 4, 10),
    ("softmax_c3_blocks2", 2, 300, 61, 6, "softmax", 2, 8, 5, 3),
]


@pytest.mark.parametrize("case", FP32_CASES, ids=[c[0] for c in FP32_CASES])
def test_fp32_other_losses_within_1e4(bc, orc, case):
    # FP32 storage (R23) for LS, hinge and softmax (the DMMA GEMV-C / GEMV-T-C kernels read
    # FP32 A for C > 1): iterates within 1e-4 of the oracle run on the FP32-rounded data
    _, N, m, n, kappa, loss, M, K, K_in = case[:9]
    C = case[9] if len(case) > 9 else 1
    solver, rep, zs, xs, ref, _ = run_pair(bc, orc, N, m, n, kappa, loss, M, K, K_in, C=C, dtype=torch.float32)
    for k in range(K):
        assert _rel(zs[k], ref["z_trace"][k]) <= 1e-4, (k, _rel(zs[k], ref["z_trace"][k]))
    assert solver.support().tolist() == ref["support"].tolist()
    assert abs(rep.objective - ref["objective"]) <= 1e-4 * abs(ref["objective"])


def test_schedule_replay_matches_oracle(bc, orc):
    # DESIGN R7: per-(outer, node) inner counts replayed identically on both sides
    P = dg.generate(3, 200, 100, 6, "logistic", seed=5)
    cs = dg.block_partition(100, 2)
    K = 6
    sched = np.array([[1, 4, 2], [3, 3, 1], [5, 1, 1], [2, 2, 2], [1, 1, 6], [4, 0, 3]], dtype=np.int32)
    prm = dict(kappa=6, max_outer=K, inner_fixed=3, refit=0, eps_p=0.0, eps_d=0.0, eps_b=0.0)
    solver = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "logistic", bc.Params(**prm), cs)
    solver.set_schedule(sched)
    solver.iterate(K)
    ref = orc.run(orc.Problem([a.numpy() for a in P.A], [b.numpy() for b in P.b], orc.LOGISTIC, 1, np.array(cs)),
                  orc.Params(**prm), schedule=sched)
    assert _rel(solver.z, ref["z"]) <= 1e-9
    assert np.array_equal(solver.get(bc.FIELD_INNER_COUNTS, np.int32).reshape(K, 3), sched)


def test_errors_and_domain(bc):
    P = dg.generate(1, 40, 16, 2, "logistic", seed=1)
    cs = dg.block_partition(16, 1)
    bad = P.b[0].clone()
    bad[3] = 0.5
    with pytest.raises(bc.BicadmmError) as e:
        bc.BiCADMM([P.A[0].cuda()], [bad.cuda()], "logistic", bc.Params(kappa=2), cs)
    assert e.value.rc == bc.ERR_DOMAIN
    with pytest.raises(bc.BicadmmError) as e:
        bc.BiCADMM([P.A[0].cuda()], [P.b[0].cuda()], "logistic", bc.Params(kappa=17), cs)
    assert e.value.rc == bc.ERR_INVALID
    s = bc.BiCADMM([P.A[0].cuda()], [P.b[0].cuda()], "logistic", bc.Params(kappa=2, inner_fixed=2), cs)
    s.iterate(2)
    with pytest.raises(bc.BicadmmError):
        s.iterate(-1)
    assert s.launches() > 0


@pytest.mark.parametrize("M", [1, 3])
def test_ls_refit_matches_oracle(bc, orc, M):
    # a13 / DESIGN R19: ridge refit on the support; GPU CG vs oracle Cholesky
    P = dg.generate(3, 120, 60, 6, "ls", seed=11)
    cs = dg.block_partition(60, M)
    prm = dict(kappa=6, max_outer=30, inner_fixed=8, refit=1, eps_p=0.0, eps_d=0.0, eps_b=0.0)
    solver = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "ls", bc.Params(**prm), cs)
    solver.iterate(30)
    rep = solver.finalize()
    ref = orc.run(orc.Problem([a.numpy() for a in P.A], [b.numpy() for b in P.b], orc.LS, 1, np.array(cs)),
                  orc.Params(**prm))
    assert solver.support().tolist() == ref["support"].tolist()
    xf = solver.get(bc.FIELD_X_FINAL)
    assert _rel(xf, ref["x_final"]) <= 1e-9
    assert abs(rep.objective - ref["objective"]) <= 1e-9 * abs(ref["objective"])


@pytest.mark.parametrize("sweep,n,m", [(1, 120, 300), (2, 120, 300), (2, 4000, 4100)],
                         ids=["two_pass", "fused", "fused_n4000_batches_of_2"])
def test_tol_mode_inner_loop_and_replay(bc, orc, sweep, n, m):
    # DESIGN R7 / S:382: tolerance-mode inner loop on the GPU; its per-(outer, node)
    # counts replayed by the oracle reproduce the GPU iterates to 1e-9, and agree
    # with the oracle's own tolerance-mode counts (boundary flips are allowed but rare).
    # n = 4000: the single pass with row batches of 2 and 3 row groups, nodes dropping out
    P = dg.generate(3, m, n, 6, "logistic", seed=21)
    cs = dg.block_partition(n, 2 if sweep == 1 else 1)   # the single-pass sweep: one block per node
    K = 8
    prm = dict(kappa=6, max_outer=K, inner_fixed=0, eps_inner=1e-6, max_inner=60, refit=0,
               eps_p=0.0, eps_d=0.0, eps_b=0.0)
    solver = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "logistic", bc.Params(sweep=sweep, **prm), cs)
    solver.iterate(K)
    counts = solver.get(bc.FIELD_INNER_COUNTS, np.int32).reshape(K, 3)
    pb = orc.Problem([a.numpy() for a in P.A], [b.numpy() for b in P.b], orc.LOGISTIC, 1, np.array(cs))
    own = orc.run(pb, orc.Params(**prm))
    rep = orc.run(pb, orc.Params(**prm), schedule=counts)
    assert counts.min() >= 1 and counts.max() <= 60
    assert _rel(solver.z, rep["z"]) <= 1e-9
    assert np.mean(counts == own["inner_counts"]) >= 0.8


def test_fused_single_block_fp64_fp32(bc, orc):
    # the single-pass CTA-pair sweep (k_fused4) on single-block nodes, FP64 and FP32 storage
    for dtype, tol in ((torch.float64, 1e-9), (torch.float32, 1e-4)):
        solver, rep, zs, xs, ref, _ = run_pair(bc, orc, 3, 777, 304, 9, "logistic", 1, 6, 5, sweep=2, dtype=dtype)
        assert solver.sweep_kind()[0] == 4
        for k in range(6):
            assert _rel(zs[k], ref["z_trace"][k]) <= tol, (dtype, k)
        assert solver.support().tolist() == ref["support"].tolist()


# Woodbury fat-block path (DESIGN R27): blocks with m_i < n_j factor the m_i x m_i
# matrix K = (c/rho_l) I + A A^T instead of the n_j x n_j F; x_ij is materialized only
# where read.  Same oracle (which always solves the n_j x n_j system), same 1e-9 bar.
FAT_CASES = [
    # name, N, m_i, n, kappa, loss, M, K_outer, K_in[, C]
    ("ls_fat", 2, 80, 300, 8, "ls", 1, 15, 5),
    ("logistic_fat_blocks2", 3, 90, 400, 10, "logistic", 2, 12, 5),
    ("hinge_fat_blocks3", 2, 150, 600, 8, "hinge", 3, 10, 4),
    ("softmax_fat_c3", 2, 60, 200, 6, "softmax", 1, 8, 4, 3),
    ("logistic_mixed_fat_tall", 2, 200, 401, 8, "logistic", 2, 10, 4),
    ("ls_fat_ragged_blocks4", 2, 77, 1030, 12, "ls", 4, 10, 3),
]


@pytest.mark.parametrize("case", FAT_CASES, ids=[c[0] for c in FAT_CASES])
def test_woodbury_fat_blocks_match_oracle(bc, orc, case):
    _, N, m, n, kappa, loss, M, K, K_in = case[:9]
    C = case[9] if len(case) > 9 else 1
    assert m < max(np.diff(dg.block_partition(n, M)))    # at least one block takes the fat path
    solver, rep, zs, xs, ref, _ = run_pair(bc, orc, N, m, n, kappa, loss, M, K, K_in, C=C, sweep=1)
    assert solver.sweep_kind()[1] >= 1
    _check_fp64(solver, rep, zs, xs, ref, K)


def test_woodbury_fp32_and_schedule(bc, orc):
    solver, rep, zs, xs, ref, _ = run_pair(bc, orc, 3, 90, 400, 10, "logistic", 2, 10, 5, dtype=torch.float32)
    for k in range(10):
        assert _rel(zs[k], ref["z_trace"][k]) <= 1e-4, k
    assert solver.support().tolist() == ref["support"].tolist()
    # schedule with zero-sweep nodes: x of an unswept node must stay as it was
    P = dg.generate(3, 70, 240, 6, "logistic", seed=5)
    cs = dg.block_partition(240, 2)
    K = 5
    sched = np.array([[1, 4, 2], [3, 0, 1], [0, 1, 1], [2, 2, 0], [4, 0, 3]], dtype=np.int32)
    prm = dict(kappa=6, max_outer=K, inner_fixed=3, refit=0, eps_p=0.0, eps_d=0.0, eps_b=0.0)
    solver = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "logistic", bc.Params(**prm), cs)
    solver.set_schedule(sched)
    solver.iterate(K)
    ref = orc.run(orc.Problem([a.numpy() for a in P.A], [b.numpy() for b in P.b], orc.LOGISTIC, 1, np.array(cs)),
                  orc.Params(**prm), schedule=sched)
    assert _rel(solver.z, ref["z"]) <= 1e-9


def test_woodbury_tol_mode(bc, orc):
    P = dg.generate(3, 100, 360, 6, "logistic", seed=22)
    cs = dg.block_partition(360, 2)
    K = 6
    prm = dict(kappa=6, max_outer=K, inner_fixed=0, eps_inner=1e-6, max_inner=60, refit=0,
               eps_p=0.0, eps_d=0.0, eps_b=0.0)
    solver = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "logistic", bc.Params(sweep=1, **prm), cs)
    solver.iterate(K)
    counts = solver.get(bc.FIELD_INNER_COUNTS, np.int32).reshape(K, 3)
    pb = orc.Problem([a.numpy() for a in P.A], [b.numpy() for b in P.b], orc.LOGISTIC, 1, np.array(cs))
    own = orc.run(pb, orc.Params(**prm))
    rep = orc.run(pb, orc.Params(**prm), schedule=counts)
    assert _rel(solver.z, rep["z"]) <= 1e-9
    assert np.mean(counts == own["inner_counts"]) >= 0.8


def test_woodbury_fat_refuses_fused_sweep(bc):
    P = dg.generate(2, 80, 300, 8, "ls", seed=1)
    with pytest.raises(Exception):
        bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "ls", bc.Params(kappa=8, sweep=2),
                   dg.block_partition(300, 1))


def test_full_h_layout_matches_oracle(bc, orc):
    # BICADMM_HPACK=0: the unpacked n_j x n_j H (GEMV) instead of the packed lower tiles
    import os
    os.environ["BICADMM_HPACK"] = "0"
    try:
        for case in (CASES[3], FAT_CASES[1]):
            _, N, m, n, kappa, loss, M, K, K_in = case[:9]
            solver, rep, zs, xs, ref, _ = run_pair(bc, orc, N, m, n, kappa, loss, M, K, K_in, sweep=1)
            _check_fp64(solver, rep, zs, xs, ref, K)
    finally:
        del os.environ["BICADMM_HPACK"]


@pytest.mark.parametrize("sweep", [1, 2], ids=["two_pass", "fused"])
def test_graph_replay_bit_identical_to_eager(bc, sweep):
    # one outer iteration is captured as a CUDA graph and replayed (default); the eager
    # launches (BICADMM_GRAPH=0) must give bit-identical iterates and the same launch count
    import os
    P = dg.generate(3, 400, 128, 6, "logistic", seed=9)
    cs = dg.block_partition(128, 1)
    out = {}
    for g in ("1", "0"):
        os.environ["BICADMM_GRAPH"] = g
        try:
            s = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "logistic",
                           bc.Params(kappa=6, max_outer=8, inner_fixed=4, eps_p=0.0, eps_d=0.0, eps_b=0.0,
                                     sweep=sweep), cs)
            l0 = s.launches()
            s.iterate(6)
            out[g] = (s.z, s.trace(), s.launches() - l0)
            s.close()
        finally:
            del os.environ["BICADMM_GRAPH"]
    assert np.array_equal(out["1"][0], out["0"][0])
    assert np.array_equal(out["1"][1], out["0"][1])
    assert out["1"][2] == out["0"][2]


@pytest.mark.parametrize("M", [1, 2])
def test_block_ready_events_order_setup_after_late_copies(bc, M):
    # bicadmm_block.ready_event: node k's A and b are copied on another stream behind a ~0.1 s
    # device sleep; setup must wait on each block's event before its Gram. Destinations start
    # zeroed, so a Gram that ran early would factor c I and change every iterate.
    P = dg.generate(3, 500, 96, 6, "logistic", seed=21)
    cs = dg.block_partition(96, M)
    prm = bc.Params(kappa=6, max_outer=6, inner_fixed=4, eps_p=0.0, eps_d=0.0, eps_b=0.0)
    s = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "logistic", prm, cs)
    s.iterate(5)
    ref = (s.z, s.trace())
    s.close()
    hostA = [a.contiguous().pin_memory() for a in P.A]
    hostb = [b.contiguous().pin_memory() for b in P.b]
    dA = [torch.zeros_like(a, device="cuda") for a in P.A]
    db = [torch.zeros_like(b, device="cuda") for b in P.b]
    torch.cuda.synchronize()
    cp = torch.cuda.Stream()
    evs = []
    with torch.cuda.stream(cp):
        for k in range(3):
            torch.cuda._sleep(50_000_000)
            dA[k].copy_(hostA[k], non_blocking=True)
            db[k].copy_(hostb[k], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cp)
            evs.append(ev)
    blocks = [(k, j, dA[k][:, cs[j]:cs[j + 1]], evs[k]) for k in range(3) for j in range(M)]
    s = bc.BiCADMM(None, db, "logistic", prm, cs, blocks=blocks)
    s.iterate(5)
    assert np.array_equal(s.z, ref[0])
    assert np.array_equal(s.trace(), ref[1])
    s.close()


@pytest.mark.parametrize("groups", ["1", "2", "3", "4", "6"])
def test_fused4_row_groups(bc, orc, groups):
    # the CTA-pair sweep with its 12 main warps split into row groups (partials per group);
    # several nodes so that node boundaries fall inside clusters
    import os
    os.environ["BICADMM_F4_GROUPS"] = groups
    try:
        solver, rep, zs, xs, ref, _ = run_pair(bc, orc, 5, 611, 496, 9, "logistic", 1, 6, 5, sweep=2)
        assert solver.sweep_kind() == (4, 0)
        for k in range(6):
            assert _rel(zs[k], ref["z_trace"][k]) <= 1e-9, (groups, k)
        assert solver.support().tolist() == ref["support"].tolist()
    finally:
        del os.environ["BICADMM_F4_GROUPS"]


def test_fused4_ragged_width(bc, orc):
    # n_j = 306 (FP64: 2448-byte rows, not a multiple of 64 bytes) on the CTA-pair kernel
    solver, rep, zs, xs, ref, _ = run_pair(bc, orc, 3, 700, 306, 9, "logistic", 1, 6, 5, sweep=2)
    assert solver.sweep_kind() == (4, 0)
    for k in range(6):
        assert _rel(zs[k], ref["z_trace"][k]) <= 1e-9, k
    assert solver.support().tolist() == ref["support"].tolist()


@pytest.mark.parametrize("n", [702, 1502])
def test_fused4_fp32_half_row_rounded_copy(bc, orc, n):
    # FP32 n_j = 2 (mod 4) (as the C5 shard width 6,250): row pitch lda = n_j + 2 (16-byte rows),
    # the second half-row (an odd number of float pairs) is copied rounded up to 16 bytes
    # into the row padding, which holds NaN here: a read of it would poison every iterate
    N, m, K = 3, n + 300, 5   # tall blocks (the single pass takes m_i >= n_j)
    P = dg.generate(N, m, n, 9, "hinge", seed=31)
    cs = dg.block_partition(n, 1)
    prm = dict(kappa=9, max_outer=K, inner_fixed=4, refit=0, eps_p=0.0, eps_d=0.0, eps_b=0.0)
    blocks = []
    for k in range(N):
        t = torch.full((m, n + 2), float("nan"), dtype=torch.float32, device="cuda")
        t[:, :n] = P.A[k].to("cuda", torch.float32)
        blocks.append((k, 0, t[:, :n]))
    b = [x.to("cuda", torch.float32) for x in P.b]
    s = bc.BiCADMM(None, b, "hinge", bc.Params(sweep=2, **prm), cs, blocks=blocks)
    assert s.sweep_kind() == (4, 0)
    zs = []
    for _ in range(K):
        s.iterate(1)
        zs.append(s.z)
    ref = orc.run(orc.Problem([a.float().double().numpy() for a in P.A], [x.float().double().numpy() for x in P.b],
                              orc.HINGE, 1, np.array(cs)), orc.Params(**prm), trace_z=True)
    for k in range(K):
        assert _rel(zs[k], ref["z_trace"][k]) <= 1e-4, k
    s.finalize()
    assert s.support().tolist() == ref["support"].tolist()
    s.close()


@pytest.mark.parametrize("loss", ["ls", "hinge"])
def test_fused4_widest_rows_e17(bc, loss):
    # n_j = 12,500 FP64 (the C3 shard's block width: 50 KB half-rows, a 4-slot ring, 17
    # elements per lane, axpy delay 1): the auto-chosen single-pass kernel against the
    # independent two-pass kernels, iterate by iterate (1e-9)
    P = dg.generate(1, 12_600, 12_500, 20, loss, seed=17, device="cuda")   # tall: m_i >= n_j
    cs = dg.block_partition(12_500, 1)
    prm = dict(kappa=20, max_outer=4, inner_fixed=3, eps_p=0.0, eps_d=0.0, eps_b=0.0, refit=0)
    out = {}
    for sweep in (0, 1):
        s = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], loss, bc.Params(sweep=sweep, **prm), cs)
        if sweep == 0:
            assert s.sweep_kind() == (4, 0)
        zs = []
        for _ in range(4):
            s.iterate(1)
            zs.append(s.z)
        out[sweep] = (np.array(zs), s.get(bc.FIELD_X_LOCAL))
        s.close()
    for k in range(4):
        assert _rel(out[0][0][k], out[1][0][k]) <= 1e-9, k
    assert _rel(out[0][1], out[1][1]) <= 1e-9


@pytest.mark.parametrize("dt,n_max", [("f64", 13_432), ("f32", 13_824)])
def test_fused4_maximum_width_and_beyond(bc, dt, n_max):
    # the widest single-pass rows: FP64 13,432 columns (52.5 KB half-rows, the last width with a
    # 4-slot ring), FP32 13,824 (fused4_max_cols: 9 two-element vectors per lane); the fused
    # sweep against the two-pass kernels; 4 columns more and setup refuses the forced single
    # pass (BICADMM_ERR_INVALID) and the auto choice is two-pass
    dtype = torch.float64 if dt == "f64" else torch.float32
    P = dg.generate(1, n_max + 100, n_max, 20, "logistic", seed=19, device="cuda", dtype=dtype)
    cs = dg.block_partition(n_max, 1)
    prm = dict(kappa=20, max_outer=3, inner_fixed=3, eps_p=0.0, eps_d=0.0, eps_b=0.0, refit=0)
    out = {}
    for sweep in (2, 1):
        s = bc.BiCADMM(P.A, P.b, "logistic", bc.Params(sweep=sweep, **prm), cs)
        assert s.sweep_kind()[0] == (4 if sweep == 2 else 0)
        s.iterate(3)
        out[sweep] = (s.z, s.get(bc.FIELD_X_LOCAL))
        s.close()
    assert _rel(out[2][0], out[1][0]) <= 1e-9
    assert _rel(out[2][1], out[1][1]) <= 1e-9
    del P
    n2 = n_max + 4
    P2 = dg.generate(1, n2 + 8, n2, 10, "logistic", seed=19, device="cuda", dtype=dtype)
    cs2 = dg.block_partition(n2, 1)
    s = bc.BiCADMM(P2.A, P2.b, "logistic", bc.Params(kappa=10, inner_fixed=1), cs2)
    assert s.sweep_kind()[0] == 0
    s.close()
    with pytest.raises(bc.BicadmmError) as e:
        bc.BiCADMM(P2.A, P2.b, "logistic", bc.Params(kappa=10, inner_fixed=1, sweep=2), cs2)
    assert e.value.rc == bc.ERR_INVALID


def test_auto_sweep_choice(bc):
    # sweep = 0: the CTA-pair single-pass kernel for rows >= 5.5 KB (C = 1, single-block
    # nodes), two-pass otherwise
    for n, want in ((704, 4), (700, 0)):
        P = dg.generate(2, 4000, n, 10, "logistic", seed=2)   # tall blocks (m_i > n_j)
        s = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "logistic", bc.Params(kappa=10),
                       dg.block_partition(n, 1))
        assert s.sweep_kind() == (want, 0), (n, s.sweep_kind())
        s.close()


@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-9), (torch.float32, 1e-4)], ids=["f64", "f32"])
def test_logistic_refit_matches_oracle(bc, orc, dtype, tol):
    # DESIGN R29: damped Newton refit on the support, GPU vs oracle (run to the same
    # iterate, then the same refit; objective and x_final at the bar)
    P = dg.generate(3, 500, 120, 8, "logistic", seed=12)
    cs = dg.block_partition(120, 2)
    prm = dict(kappa=8, max_outer=25, inner_fixed=5, refit=1, eps_p=0.0, eps_d=0.0, eps_b=0.0)
    s = bc.BiCADMM([a.to("cuda", dtype) for a in P.A], [b.to("cuda", dtype) for b in P.b], "logistic",
                   bc.Params(**prm), cs)
    s.iterate(25)
    rep = s.finalize()
    Aref = [a.to(dtype).double().numpy() for a in P.A]
    bref = [b.to(dtype).double().numpy() for b in P.b]
    ref = orc.run(orc.Problem(Aref, bref, orc.LOGISTIC, 1, np.array(cs)), orc.Params(**prm))
    assert s.support().tolist() == ref["support"].tolist()
    xf = s.get(bc.FIELD_X_FINAL)
    assert _rel(xf, ref["x_final"]) <= tol
    assert abs(rep.objective - ref["objective"]) <= tol * abs(ref["objective"])
    # the refit lowers the objective relative to z on the support
    z_on_T = np.zeros_like(xf)
    T = ref["support"]
    z_on_T[T] = ref["z"][T]
    assert ref["objective"] <= orc.objective(orc.Problem(Aref, bref, orc.LOGISTIC, 1, np.array(cs)), 100.0, z_on_T)


@pytest.mark.parametrize("C", [3, 10])
def test_softmax_refit_matches_oracle(bc, orc, C):
    # DESIGN R29 for softmax: entry-support Newton refit, GPU vs oracle at 1e-9
    P = dg.generate(2, 400, 60, 12, "softmax", C=C, seed=31)
    cs = dg.block_partition(60, 2)
    prm = dict(kappa=12, max_outer=15, inner_fixed=4, refit=1, eps_p=0.0, eps_d=0.0, eps_b=0.0)
    s = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "softmax", bc.Params(**prm), cs, C=P.C)
    s.iterate(15)
    rep = s.finalize()
    ref = orc.run(orc.Problem([a.numpy() for a in P.A], [b.numpy() for b in P.b], orc.SOFTMAX, P.C, np.array(cs)),
                  orc.Params(**prm))
    assert s.support().tolist() == ref["support"].tolist()
    assert _rel(s.get(bc.FIELD_X_FINAL), ref["x_final"]) <= 1e-9
    assert abs(rep.objective - ref["objective"]) <= 1e-9 * abs(ref["objective"])


def test_device_loop_solve_matches_host_loop(bc):
    # bicadmm_solve runs the fixed-schedule outer loop as a CUDA-graph while node with
    # device-side termination; it must reproduce the host-driven loop bit for bit
    # (iterations, trace, z, support, objective)
    import os
    P = dg.generate(2, 100, 50, 5, "ls", seed=3)
    cs = dg.block_partition(50, 1)
    out = {}
    for g in ("1", "0"):
        os.environ["BICADMM_GRAPH"] = g
        try:
            s = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "ls",
                           bc.Params(kappa=5, max_outer=2000, inner_fixed=10, refit=1), cs)
            rep = s.solve()
            out[g] = (rep.outer_iters, rep.converged, s.trace(), s.z, s.support(), rep.objective,
                      s.get(bc.FIELD_INNER_COUNTS, np.int32))
            s.close()
        finally:
            del os.environ["BICADMM_GRAPH"]
    a, b = out["1"], out["0"]
    assert a[0] == b[0] and a[1] == b[1] == 1
    assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3]) and np.array_equal(a[4], b[4])
    assert a[5] == b[5]
    assert np.array_equal(a[6], b[6])


SELF_CASES = [
    # name, N, m_i, n, kappa, loss, M, C, refit
    ("logistic_M1", 3, 700, 256, 8, "logistic", 1, 1, 0),
    ("ls_M3_refit", 2, 500, 300, 10, "ls", 3, 1, 1),
    ("softmax_M2", 2, 400, 120, 9, "softmax", 2, 4, 0),
    ("hinge_M2", 2, 600, 200, 8, "hinge", 2, 1, 0),
]


@pytest.mark.parametrize("split", ["1", "2"], ids=["world_sums", "split_block_sums"])
@pytest.mark.parametrize("case", SELF_CASES, ids=[c[0] for c in SELF_CASES])
def test_nccl_one_rank_path_matches_local(bc, case, split):
    # BICADMM_NCCL_SELF: a real one-rank NCCL communicator, so the multi-rank code path runs on one
    # GPU -- eager launches (no graphs), the per-outer AllReduces of sum_i(x_i + u_i), the node
    # residual partials and the objective; with "2" also the per-sweep group AllReduce of the
    # node block sums S_i (Algorithm 2) that block-major placements use.  A one-rank
    # AllReduce is a copy, so the iterates must equal the local (comm = None) run: bit for bit
    # without split sums, and to 1e-13 with them (S_i is then summed by k_psum, not the prox kernel).
    import os
    name, N, m, n, kappa, loss, M, C, refit = case
    P = dg.generate(N, m, n, kappa, loss, seed=31, C=C)
    cs = dg.block_partition(n, M)
    out = {}
    for mode in ("local", "nccl"):
        comm = None
        if mode == "nccl":
            os.environ["BICADMM_NCCL_SELF"] = split
        try:
            if mode == "nccl":
                comm = bc.bicadmm_comm_init(1, 0, torch.cuda.current_device(), None, 0)
            s = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], loss,
                           bc.Params(kappa=kappa, max_outer=40, inner_fixed=0, max_inner=20, eps_inner=1e-9,
                                     eps_p=1e-7, eps_d=1e-7, eps_b=1e-7, refit=refit), cs, C=P.C, comm=comm)
            s.iterate(3)
            z3 = s.z
            rep = s.solve()
            rep = s.finalize()
            out[mode] = dict(z3=z3, z=s.z, trace=s.trace(), obj=rep.objective, sup=s.support(),
                             xf=s.get(bc.FIELD_X_FINAL), outer=rep.outer_iters, inner=rep.inner_sweeps)
            s.close()
        finally:
            os.environ.pop("BICADMM_NCCL_SELF", None)
            bc.bicadmm_comm_destroy(comm)
    a, b = out["local"], out["nccl"]
    if split == "1":
        assert np.array_equal(a["z3"], b["z3"])
        assert np.array_equal(a["z"], b["z"])
        assert np.array_equal(a["trace"], b["trace"])
        assert a["obj"] == b["obj"]
    else:
        assert _rel(b["z3"], a["z3"]) <= 1e-13
        assert a["outer"] == b["outer"]
        assert _rel(b["z"], a["z"]) <= 1e-11
        assert abs(a["obj"] - b["obj"]) <= 1e-11 * abs(a["obj"])
    assert np.array_equal(a["sup"], b["sup"])
    assert _rel(b["xf"], a["xf"]) <= 1e-11


def test_nccl_one_rank_single_pass_in_the_outer_graph(bc, capfd):
    # the multi-rank node-major path with the CTA-pair single pass (what a weak-scaling
    # configs[1] run takes on every rank): a real one-rank NCCL communicator, the fused sweep,
    # the per-outer AllReduces captured in the replayed outer-iteration graph; the iterates
    # equal the local run's bit for bit (a one-rank AllReduce is a copy)
    import os
    P = dg.generate(3, 900, 800, 8, "logistic", seed=17)   # tall single-block nodes, 6.4 KB rows
    cs = dg.block_partition(800, 1)
    out = {}
    for mode in ("local", "nccl"):
        comm = None
        os.environ["BICADMM_GRAPH_DEBUG"] = "1"
        if mode == "nccl":
            os.environ["BICADMM_NCCL_SELF"] = "1"
        try:
            if mode == "nccl":
                comm = bc.bicadmm_comm_init(1, 0, torch.cuda.current_device(), None, 0)
            s = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "logistic",
                           bc.Params(kappa=8, max_outer=40, inner_fixed=4, refit=0, eps_p=0, eps_d=0, eps_b=0),
                           cs, comm=comm)
            assert s.sweep_kind() == (4, 0), (mode, s.sweep_kind())
            zs = []
            for _ in range(6):
                s.iterate(1)
                zs.append(s.z)
            out[mode] = (np.array(zs), s.trace())
            s.close()
        finally:
            os.environ.pop("BICADMM_NCCL_SELF", None)
            os.environ.pop("BICADMM_GRAPH_DEBUG", None)
            bc.bicadmm_comm_destroy(comm)
        err = capfd.readouterr().err
        assert "captured outer-iteration graph" in err, (mode, err[-500:])
    (za, ta), (zb, tb) = out["local"], out["nccl"]
    assert np.array_equal(za, zb) and np.array_equal(ta, tb)


@pytest.mark.parametrize("split", ["1", "2"], ids=["world_sums", "split_block_sums"])
def test_nccl_collectives_captured_in_the_outer_graph(bc, split, capfd):
    # fixed inner schedule: from the second outer iteration on, one outer iteration (sweeps,
    # the NCCL AllReduces, the global step, the scalar read-back) is replayed as a CUDA graph
    # with the collectives captured in it; the iterates equal the local run's
    import os
    P = dg.generate(3, 300, 120, 8, "logistic", seed=7)
    cs = dg.block_partition(120, 2)
    out = {}
    for mode in ("local", "nccl"):
        comm = None
        os.environ["BICADMM_GRAPH_DEBUG"] = "1"
        if mode == "nccl":
            os.environ["BICADMM_NCCL_SELF"] = split
        try:
            if mode == "nccl":
                comm = bc.bicadmm_comm_init(1, 0, torch.cuda.current_device(), None, 0)
            s = bc.BiCADMM([a.cuda() for a in P.A], [b.cuda() for b in P.b], "logistic",
                           bc.Params(kappa=8, max_outer=40, inner_fixed=4, refit=0, eps_p=0, eps_d=0, eps_b=0, sweep=1),
                           cs, comm=comm)   # the same two-pass kernels on both sides (small nodes would take kind 5 locally)
            zs = []
            for _ in range(6):
                s.iterate(1)
                zs.append(s.z)
            out[mode] = (np.array(zs), s.trace())
            s.close()
        finally:
            os.environ.pop("BICADMM_NCCL_SELF", None)
            os.environ.pop("BICADMM_GRAPH_DEBUG", None)
            bc.bicadmm_comm_destroy(comm)
        err = capfd.readouterr().err
        assert "captured outer-iteration graph" in err, (mode, err[-500:])
    (za, ta), (zb, tb) = out["local"], out["nccl"]
    if split == "1":
        assert np.array_equal(za, zb) and np.array_equal(ta, tb)
    else:
        for k in range(6):
            assert _rel(zb[k], za[k]) <= 1e-13, k


@pytest.mark.parametrize("loss,C,bad", [("logistic", 1, 0.5), ("hinge", 1, 0.0), ("softmax", 3, 3.0),
                                        ("softmax", 3, 1.5), ("softmax", 3, -1.0), ("ls", 1, float("nan"))])
def test_domain_error_from_the_c_abi(bc, loss, C, bad):
    # BICADMM_ERR_DOMAIN (bicadmm.h) comes from bicadmm_setup itself (a device pass over
    # the labels), not from the Python wrapper: raw ctypes structs, no BiCADMM class
    import ctypes as ct
    P = dg.generate(2, 64, 32, 3, loss, seed=5, C=C)
    A = [a.cuda().contiguous() for a in P.A]
    b = [x.cuda().contiguous() for x in P.b]
    for fail_node in (None, 1):
        if fail_node is not None:
            b[fail_node][17] = bad
        cs = np.array([0, 32], dtype=np.int64)
        m = np.array([64, 64], dtype=np.int64)
        blocks = (bc.bicadmm_block * 2)(*[bc.bicadmm_block(i, 0, A[i].data_ptr(), 32, None) for i in range(2)])
        bptr = (ct.c_void_p * 2)(*[x.data_ptr() for x in b])
        prob = bc.bicadmm_problem(2, 1, C, bc.LOSSES[loss], bc.F64, 2, 32, m.ctypes.data_as(ct.POINTER(ct.c_int64)),
                                  cs.ctypes.data_as(ct.POINTER(ct.c_int64)), blocks, bptr)
        prm = bc.Params(kappa=3).struct()
        nbytes = ct.c_size_t(0)
        assert bc.lib().bicadmm_workspace_size(ct.byref(prob), ct.byref(prm), ct.byref(nbytes)) == 0
        ws = torch.empty(nbytes.value + 256, dtype=torch.uint8, device="cuda")
        base = ws.data_ptr() + (-ws.data_ptr()) % 256
        h = ct.c_void_p()
        rc = bc.lib().bicadmm_setup(ct.byref(prob), ct.byref(prm), None, ct.c_void_p(base), nbytes.value,
                                    ct.c_void_p(torch.cuda.current_stream().cuda_stream), ct.byref(h))
        if fail_node is None:
            assert rc == bc.OK
            bc.lib().bicadmm_destroy(h)
        else:
            assert rc == bc.ERR_DOMAIN
            assert not h.value


SMALL_CASES = [
    # name, N, m_i, n, kappa, loss, M, K, K_in, dtype
    ("c1_ls", 2, 100, 50, 5, "ls", 1, 30, 10, "f64"),
    ("logistic_blocks2", 3, 200, 96, 6, "logistic", 2, 12, 5, "f64"),
    ("hinge_blocks3", 2, 150, 90, 6, "hinge", 3, 12, 4, "f64"),
    ("logistic_fp32", 2, 180, 64, 5, "logistic", 1, 12, 5, "f32"),
]


@pytest.mark.parametrize("case", SMALL_CASES, ids=[c[0] for c in SMALL_CASES])
def test_small_nodes_whole_inner_loop_in_one_cta(bc, orc, case):
    # sweep kind 5 (auto, single rank, C == 1, nodes that fit one CTA's shared memory): the K
    # sweeps of an outer iteration in one launch; iterates against the oracle
    _, N, m, n, kappa, loss, M, K, K_in, dt = case
    dtype = torch.float64 if dt == "f64" else torch.float32
    solver, rep, zs, xs, ref, _ = run_pair(bc, orc, N, m, n, kappa, loss, M, K, K_in, dtype=dtype, sweep=0)
    assert solver.sweep_kind() == (5, 0)
    tol = 1e-9 if dt == "f64" else 1e-4
    for k in range(K):
        assert _rel(zs[k], ref["z_trace"][k]) <= tol, (k, _rel(zs[k], ref["z_trace"][k]))
        assert _rel(xs[k], ref["x_trace"][k].ravel()) <= tol, k
    assert solver.support().tolist() == ref["support"].tolist()
    assert abs(rep.objective - ref["objective"]) <= tol * abs(ref["objective"])
