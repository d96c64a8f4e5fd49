"""Multi-rank host logic on CPU (world_size 2, gloo).

1. placement.plan covers every (node, block) exactly once with consistent groups.
2. The exchange design of capi.cu -- per-sweep AllReduce of the node block sums
   over the node group (Algorithm 2), per-outer AllReduce of sum_i(x_i+u_i)
   and of the per-node ||x_ij - z_j||^2 partials over all ranks ("Collect"),
   everything else replicated -- is mirrored here with the oracle's step functions
   and gloo collectives, and must reproduce the single-process oracle run.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_16267_b200 import datagen as dg
from paper_2405_16267_b200 import placement as pl


@pytest.mark.parametrize("world,N,M,mode", [(2, 2, 2, "auto"), (2, 1, 8, "auto"), (2, 4, 1, "auto"),
                                            (8, 1, 8, "block"), (8, 8, 8, "node"), (4, 8, 8, "auto"),
                                            (8, 4, 8, "auto"), (2, 3, 2, "block")])
def test_placement_plans(world, N, M, mode):
    plans = pl.plan(world, N, M, mode)
    pl.check(plans, N, M)
    assert len(plans) == world
    gn, gb = pl.grid_shape(world, N, M, mode)
    assert gn * gb == world


def test_placement_errors():
    with pytest.raises(ValueError):
        pl.plan(4, 2, 1, "auto")
    with pytest.raises(ValueError):
        pl.plan(4, 2, 8, "node")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc
        N, m, n, M, kappa, K, K_in = 2, 40, 24, 2, 4, 6, 3
        P = dg.generate(N, m, n, kappa, "logistic", seed=4)
        cs = dg.block_partition(n, M)
        prm = dict(rho_c=4.0, alpha=0.5, rho_l=4.0, gamma=100.0)
        plans = pl.plan(world, N, M, mode)
        me = plans[rank]
        # group of ranks sharing my node group
        groups = {}
        for p in plans:
            groups.setdefault(p.node_group, []).append(p.rank)
        gh = {c: dist.new_group(r) for c, r in sorted(groups.items())}
        mygroup = gh[me.node_group]
        gsize = len(groups[me.node_group])
        A = [a.numpy() for a in P.A]
        b = [x.numpy() for x in P.b]
        c = 1.0 / (N * prm["gamma"]) + prm["rho_c"]
        L = {(i, j): orc.block_factor(A[i][:, cs[j]:cs[j + 1]], prm["rho_l"], c) for (i, j) in me.blocks}
        x = {ij: np.zeros(cs[ij[1] + 1] - cs[ij[1]]) for ij in me.blocks}
        u = {ij: np.zeros_like(v) for ij, v in x.items()}
        p = {ij: np.zeros(m) for ij in me.blocks}
        nu = {i: np.zeros(m) for i in me.nodes}
        ob = {i: np.zeros(m) for i in me.nodes}
        ab = {i: np.zeros(m) for i in me.nodes}
        z, s, v, t = np.zeros(n), np.zeros(n), 0.0, 0.0
        rho_b = prm["alpha"] * prm["rho_c"]
        for k in range(K):
            for _ in range(K_in):
                for (i, j) in me.blocks:
                    q = p[(i, j)] + ob[i] - ab[i] - nu[i]
                    rhs = prm["rho_l"] * orc.gemv_t(A[i][:, cs[j]:cs[j + 1]], q) + \
                        prm["rho_c"] * (z[cs[j]:cs[j + 1]] - u[(i, j)])
                    x[(i, j)] = orc.chol_solve(L[(i, j)], rhs)
                    p[(i, j)] = orc.gemv(A[i][:, cs[j]:cs[j + 1]], x[(i, j)])
                for i in me.nodes:
                    S = sum(p[(ii, j)] for (ii, j) in me.blocks if ii == i)
                    if gsize > 1:                       # per-sweep AllReduce over the node group
                        St = torch.from_numpy(np.ascontiguousarray(S))
                        dist.all_reduce(St, group=mygroup)
                        S = St.numpy()
                    ab[i] = S / M
                    for r in range(m):
                        ob[i][r] = orc.prox_omega(orc.LOGISTIC, M, prm["rho_l"], b[i][r], [ab[i][r] + nu[i][r]])[0]
                    nu[i] = nu[i] + ab[i] - ob[i]
            wsum = np.zeros(n)
            for (i, j) in me.blocks:
                wsum[cs[j]:cs[j + 1]] += x[(i, j)] + u[(i, j)]
            wt = torch.from_numpy(wsum)
            dist.all_reduce(wt)                         # per-outer AllReduce over all ranks
            z, t, _ = orc.zt_update(wt.numpy() / N, s, v, N, prm["rho_c"], rho_b)
            s, _ = orc.s_update(z, t, v, kappa)
            v += float(z @ s - t)
            for (i, j) in me.blocks:
                u[(i, j)] += x[(i, j)] - z[cs[j]:cs[j + 1]]
        out_q.put((rank, z, t, v))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["block", "node"])
def test_distributed_exchange_matches_single_process(orc, mode):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    P = dg.generate(2, 40, 24, 4, "logistic", seed=4)
    cs = dg.block_partition(24, 2)
    ref = orc.run(orc.Problem([a.numpy() for a in P.A], [b.numpy() for b in P.b], orc.LOGISTIC, 1, np.array(cs)),
                  orc.Params(kappa=4, max_outer=6, inner_fixed=3, refit=0, eps_p=0, eps_d=0, eps_b=0))
    zs = {r: z for (r, z, _, _) in res}
    # replicated state is identical on every rank
    assert np.array_equal(zs[0], zs[1])
    assert np.linalg.norm(zs[0] - ref["z"]) <= 1e-12 * np.linalg.norm(ref["z"])
    for (_, _, t, v) in res:
        assert abs(t - ref["t"]) <= 1e-12 * abs(ref["t"])
