"""The multi-rank code path on one GPU, against the oracle.

G ranks run as G handles of this process, each on its own host thread and CUDA
stream, joined by the library's in-process emulated communicator
(bicadmm_emu_group_create / bicadmm_comm_init_emu, include/bicadmm.h): every AllReduce
of the method -- Algorithm 2's per-sweep block sum over the node group
and the outer Collect over all ranks -- is a fixed-order device sum over the
members' buffers.  No kernel waits on another, so the ranks need not run concurrently.

Placements are the block-major shapes of BASELINE.json configs[2] (C3: one node, GPU g
holds feature block g), configs[3] (C4: softmax, 8 blocks over G = 2, 4, 8) and configs[4]
(C5: 8 nodes x 8 blocks, GPU g holds block g of every node), plus a node x block grid.
Bar (north star, DESIGN R22): every rank's iterates z^k, its local x_ij^k, t, v and the
residuals within 1e-9 of the single-process oracle run, identical support, objective
within 1e-9, and the replicated state (z, trace) bit-identical across ranks.
"""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2405_16267_b200 import datagen as dg  # noqa: E402
from paper_2405_16267_b200 import placement as pl  # noqa: E402


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


def run_emulated(bc, P, cs, loss, prm, G, mode, K, dtype=torch.float64, schedule=None, plans=None):
    """Run K outer iterations on G emulated ranks; returns per-rank dicts."""
    N, M, C = P.N, len(cs) - 1, P.C
    plans = plans or pl.plan(G, N, M, mode)
    dev = torch.cuda.current_device()
    A = [a.to("cuda", dtype) for a in P.A]
    b = [x.to("cuda", dtype) for x in P.b]
    torch.cuda.synchronize()
    group = bc.bicadmm_emu_group_create(G)
    comms = [bc.bicadmm_comm_init_emu(group, r, dev, plans[r].node_group) for r in range(G)]
    out = [None] * G
    errs = [None] * G

    def worker(r):
        try:
            torch.cuda.set_device(dev)
            st = torch.cuda.Stream()
            me = plans[r]
            blocks = [(i, j, A[i][:, cs[j]:cs[j + 1]]) for (i, j) in me.blocks]
            b_all = [b[i] if i in me.nodes else None for i in range(N)]
            with torch.cuda.stream(st):
                s = bc.BiCADMM(None, b_all, loss, bc.Params(**prm), cs, blocks=blocks, comm=comms[r], stream=st,
                               C=C)
                if schedule is not None:
                    s.set_schedule(schedule)
                zs, xs = [], []
                for _ in range(K):
                    s.iterate(1)
                    zs.append(s.z)
                    xs.append(s.get(bc.FIELD_X_LOCAL))
                rep = s.finalize()
                out[r] = dict(z=np.array(zs), x=xs, trace=s.trace(), sup=s.support(), obj=rep.objective,
                              xf=s.get(bc.FIELD_X_FINAL), counts=s.get(bc.FIELD_INNER_COUNTS, np.int32),
                              blocks=list(me.blocks), launches=s.launches())
                s.close()
        except Exception as e:  # noqa: BLE001 -- re-raised in the main thread
            errs[r] = e

    th = [threading.Thread(target=worker, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    alive = any(t.is_alive() for t in th)
    for c in comms:
        bc.bicadmm_comm_destroy(c)
    if not alive:
        bc.bicadmm_emu_group_destroy(group)
    assert not alive, "emulated ranks did not finish"
    for e in errs:
        if e is not None:
            raise e
    return out


def oracle_run(orc, P, cs, loss, prm, dtype=torch.float64, schedule=None):
    lid = {"ls": orc.LS, "logistic": orc.LOGISTIC, "hinge": orc.HINGE, "softmax": orc.SOFTMAX}[loss]
    Aref = [a.to(dtype).double().numpy() for a in P.A]
    bref = [x.to(dtype).double().numpy() for x in P.b]
    return orc.run(orc.Problem(Aref, bref, lid, P.C, np.array(cs)), orc.Params(**prm), trace_z=True, trace_x=True,
                   schedule=schedule)


def check_against_oracle(out, ref, cs, C, K, tol=1e-9):
    z0, tr0 = out[0]["z"], out[0]["trace"]
    for r, o in enumerate(out):
        # replicated state: identical bits on every rank (deterministic fixed-order sums)
        assert np.array_equal(o["z"], z0), r
        assert np.array_equal(o["trace"], tr0), r
        assert o["sup"].tolist() == ref["support"].tolist(), r
        assert abs(o["obj"] - ref["objective"]) <= tol * abs(ref["objective"]), (r, o["obj"], ref["objective"])
        assert o["launches"] > 0
    tr_o = ref["trace"]
    for k in range(K):
        assert _rel(z0[k], ref["z_trace"][k]) <= tol, (k, _rel(z0[k], ref["z_trace"][k]))
        t_o, v_o = tr_o[k, 3], tr_o[k, 4]
        assert abs(tr0[k, 3] - t_o) <= tol * abs(t_o)
        assert abs(tr0[k, 4] - v_o) <= tol * max(abs(v_o), abs(t_o))
        for c in (0, 1):
            assert abs(tr0[k, c] - tr_o[k, c]) <= tol * max(abs(tr_o[k, c]), abs(tr_o[0, c]))
        assert abs(tr0[k, 2] - tr_o[k, 2]) <= tol * max(abs(tr_o[k, 2]), abs(t_o))
        # each rank's local x_ij (blocks[] order) against the oracle's x_i restricted to block j,
        # relative to ||x_i|| (a block's slice of a sparse iterate may be tiny)
        for o in out:
            xs, off = o["x"][k], 0
            for (i, j) in o["blocks"]:
                w = (cs[j + 1] - cs[j]) * C
                want = ref["x_trace"][k][i][cs[j] * C:cs[j + 1] * C]
                scale = max(np.linalg.norm(ref["x_trace"][k][i]), 1e-300)
                assert np.linalg.norm(xs[off:off + w] - want) <= tol * scale, (k, i, j)
                off += w


EMU_CASES = [
    # name, N, m_i, n, kappa, loss, M, C, G, mode, K_outer, K_in
    ("C3_ls_blockmajor_G8", 1, 1500, 384, 12, "ls", 8, 1, 8, "block", 8, 4),
    ("C4_softmax_G2", 1, 900, 192, 12, "softmax", 8, 10, 2, "block", 5, 3),
    ("C4_softmax_G4", 1, 900, 192, 12, "softmax", 8, 10, 4, "block", 5, 3),
    ("C4_softmax_G8", 1, 900, 192, 12, "softmax", 8, 10, 8, "block", 5, 3),
    ("C5_hinge_blockmajor_G8", 8, 300, 256, 10, "hinge", 8, 1, 8, "block", 6, 3),
    ("grid_logistic_2x2", 2, 500, 160, 8, "logistic", 4, 1, 4, "auto", 8, 4),
    ("nodemajor_logistic_G4", 4, 400, 128, 6, "logistic", 1, 1, 4, "node", 8, 4),
]


@pytest.mark.parametrize("case", EMU_CASES, ids=[c[0] for c in EMU_CASES])
def test_emulated_ranks_match_oracle(bc, orc, case):
    _, N, m, n, kappa, loss, M, C, G, mode, K, K_in = case
    P = dg.generate(N, m, n, kappa, loss, seed=41, C=C)
    cs = dg.block_partition(n, M)
    prm = dict(kappa=kappa, max_outer=K, inner_fixed=K_in, refit=0, eps_p=0.0, eps_d=0.0, eps_b=0.0)
    out = run_emulated(bc, P, cs, loss, prm, G, mode, K)
    ref = oracle_run(orc, P, cs, loss, prm)
    check_against_oracle(out, ref, cs, P.C, K)


def test_emulated_tol_mode_replayed_by_oracle(bc, orc):
    # tolerance-mode inner loop on block-major ranks: subsets of nodes sweep (grouped
    # AllReduce of the active nodes' S_i, AllReduce of the ||dx||^2 partials); the oracle
    # replays the per-(outer, node) counts, which all ranks must agree on
    N, m, n, kappa, M, G, K = 3, 400, 96, 6, 2, 2, 6
    P = dg.generate(N, m, n, kappa, "logistic", seed=43)
    cs = dg.block_partition(n, M)
    prm = dict(kappa=kappa, max_outer=K, inner_fixed=0, eps_inner=1e-6, max_inner=40, refit=0,
               eps_p=0.0, eps_d=0.0, eps_b=0.0)
    out = run_emulated(bc, P, cs, "logistic", prm, G, "block", K)
    counts = out[0]["counts"].reshape(K, N)
    for o in out:
        assert np.array_equal(o["counts"].reshape(K, N), counts)
    assert counts.min() >= 1 and len(np.unique(counts)) > 1
    ref = oracle_run(orc, P, cs, "logistic", prm, schedule=counts)
    check_against_oracle(out, ref, cs, 1, K)


def test_emulated_fp32_blockmajor(bc, orc):
    # FP32 storage on block-major ranks: within 1e-4 of the oracle on the FP32-rounded data
    N, m, n, kappa, M, G, K = 2, 600, 128, 8, 4, 4, 6
    P = dg.generate(N, m, n, kappa, "logistic", seed=47)
    cs = dg.block_partition(n, M)
    prm = dict(kappa=kappa, max_outer=K, inner_fixed=4, refit=0, eps_p=0.0, eps_d=0.0, eps_b=0.0)
    out = run_emulated(bc, P, cs, "logistic", prm, G, "block", K, dtype=torch.float32)
    ref = oracle_run(orc, P, cs, "logistic", prm, dtype=torch.float32)
    for k in range(K):
        assert _rel(out[0]["z"][k], ref["z_trace"][k]) <= 1e-4
    for o in out:
        assert np.array_equal(o["z"], out[0]["z"])
        assert o["sup"].tolist() == ref["support"].tolist()


def test_emulated_ls_refit_blockmajor(bc, orc):
    # LS ridge refit on the support (DESIGN R19) across ranks: the CG mat-vecs all-reduce the
    # block sums over the group and the n-vector over the world
    N, m, n, kappa, M, G, K = 2, 300, 96, 6, 4, 4, 20
    P = dg.generate(N, m, n, kappa, "ls", seed=49)
    cs = dg.block_partition(n, M)
    prm = dict(kappa=kappa, max_outer=K, inner_fixed=6, refit=1, eps_p=0.0, eps_d=0.0, eps_b=0.0)
    out = run_emulated(bc, P, cs, "ls", prm, G, "block", K)
    ref = oracle_run(orc, P, cs, "ls", prm)
    for o in out:
        assert o["sup"].tolist() == ref["support"].tolist()
        assert _rel(o["xf"], ref["x_final"]) <= 1e-9
        assert abs(o["obj"] - ref["objective"]) <= 1e-9 * abs(ref["objective"])


def test_emulated_bad_placement_fails_on_every_rank(bc):
    # block (0, 1) on no rank and (0, 0) on two: bicadmm_setup's collective placement check
    # returns BICADMM_ERR_PLACEMENT on all ranks instead of hanging in a collective
    P = dg.generate(1, 200, 64, 4, "ls", seed=3)
    cs = dg.block_partition(64, 2)
    plans = pl.plan(2, 1, 2, "block")
    plans[1].blocks = [(0, 0)]
    prm = dict(kappa=4, max_outer=2, inner_fixed=2, refit=0)
    with pytest.raises(bc.BicadmmError) as e:
        run_emulated(bc, P, cs, "ls", prm, 2, "block", 1, plans=plans)
    assert e.value.rc == bc.ERR_PLACEMENT


NEWTON_REFIT_CASES = [
    # name, N, m_i, n, kappa, loss, M, C, G, mode
    ("logistic_blockmajor_G2", 2, 400, 96, 8, "logistic", 2, 1, 2, "block"),
    ("logistic_blockmajor_G4", 2, 400, 96, 8, "logistic", 4, 1, 4, "block"),
    ("logistic_nodemajor_G2", 2, 400, 96, 8, "logistic", 1, 1, 2, "node"),
    ("logistic_grid_2x2", 2, 400, 96, 8, "logistic", 2, 1, 4, "auto"),
    ("softmax_blockmajor_G2", 1, 500, 48, 12, "softmax", 2, 3, 2, "block"),
]


@pytest.mark.parametrize("case", NEWTON_REFIT_CASES, ids=[c[0] for c in NEWTON_REFIT_CASES])
def test_emulated_newton_refit(bc, orc, case):
    # logistic / softmax damped-Newton refit on the support (DESIGN R29) across ranks: support
    # columns summed over the node group, node sums (objective, gradient, Hessian) over all
    # ranks; every rank takes the same Newton steps and reaches the oracle's refit
    _, N, m, n, kappa, loss, M, C, G, mode = case
    P = dg.generate(N, m, n, kappa, loss, seed=53, C=C)
    cs = dg.block_partition(n, M)
    prm = dict(kappa=kappa, max_outer=15, inner_fixed=4, refit=1, eps_p=0.0, eps_d=0.0, eps_b=0.0)
    out = run_emulated(bc, P, cs, loss, prm, G, mode, 15)
    ref = oracle_run(orc, P, cs, loss, prm)
    for o in out:
        assert o["sup"].tolist() == ref["support"].tolist()
        assert np.array_equal(o["xf"], out[0]["xf"])
        assert _rel(o["xf"], ref["x_final"]) <= 1e-9, _rel(o["xf"], ref["x_final"])
        assert abs(o["obj"] - ref["objective"]) <= 1e-9 * abs(ref["objective"])


@pytest.mark.parametrize("G,dt", [(2, "f64"), (4, "f64"), (2, "f32")])
def test_emulated_nodemajor_single_pass(bc, orc, G, dt):
    # node-major weak scaling (configs[1]'s multi-GPU shape): every rank holds whole nodes and
    # runs the CTA-pair single pass (rows >= 5.5 KB); Collect and the residual partials cross
    # the ranks once per outer iteration.  Against the oracle at 1e-9, bit-identical z on all ranks.
    N, m, n, K = 2 * G, 780, 720, 5
    P = dg.generate(N, m, n, 9, "logistic", seed=23)
    cs = dg.block_partition(n, 1)
    prm = dict(kappa=9, max_outer=K, inner_fixed=3, refit=0, eps_p=0.0, eps_d=0.0, eps_b=0.0, sweep=2)
    dtype = torch.float64 if dt == "f64" else torch.float32
    out = run_emulated(bc, P, cs, "logistic", prm, G, "node", K, dtype=dtype)
    oprm = {k: v for k, v in prm.items() if k != "sweep"}
    ref = oracle_run(orc, P, cs, "logistic", oprm, dtype=dtype)
    check_against_oracle(out, ref, cs, 1, K, tol=1e-9 if dt == "f64" else 1e-4)
