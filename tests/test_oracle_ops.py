"""Pins for the oracle's single operations (CPU only).

Each test pins an oracle function to something other than itself: a value printed
in SPEC.md / derived in SURVEY.md (tests/golden/spec_examples.json, each with its
citation), a closed form, a brute-force grid, an independent solver (SPEC's PGD,
scipy.optimize on the *objective* rather than the oracle's stationarity equation),
or numpy's library routines for plain linear algebra.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
from scipy import optimize

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
LOSS = {"ls": 0, "logistic": 1, "softmax": 2, "hinge": 3}


# ---------------------------------------------------------------- losses / objective
@pytest.mark.parametrize("ex", GOLD["loss_value"], ids=lambda e: e["cite"])
def test_loss_value_spec(orc, ex):
    assert orc.loss_value(LOSS[ex["loss"]], ex["w"], ex["b"]) == pytest.approx(ex["expect"], abs=1e-15)


def test_loss_value_errors(orc):
    with pytest.raises(orc.OracleError):
        orc.loss_value(orc.LOGISTIC, [0.0], [0.5])          # S:60 domain
    with pytest.raises(orc.OracleError):
        orc.loss_value(orc.LS, [0.0, 1.0], [0.5])            # S:60 dimension


def test_loss_convexity_and_nonnegativity(orc):
    # S:85-86 invariants
    rng = np.random.default_rng(0)
    for loss in (orc.LS, orc.LOGISTIC, orc.HINGE):
        for _ in range(200):
            b = 1.0 if rng.random() < 0.5 else -1.0
            w1, w2, th = rng.normal(scale=3), rng.normal(scale=3), rng.random()
            f = lambda w: orc.phi(loss, [w], b)
            assert f(th * w1 + (1 - th) * w2) <= th * f(w1) + (1 - th) * f(w2) + 1e-12
            assert f(w1) >= 0.0


def test_softmax_phi_matches_logsumexp(orc):
    rng = np.random.default_rng(1)
    for _ in range(50):
        w = rng.normal(size=10) * 5
        y = int(rng.integers(10))
        ref = math.log(sum(math.exp(v) for v in w)) - w[y]
        assert orc.phi(orc.SOFTMAX, w, y, C=10) == pytest.approx(ref, rel=1e-13, abs=1e-13)


def test_objective_spec(orc):
    ex = GOLD["objective"][0]
    pb = orc.Problem([np.array(ex["A"], float)], [np.array(ex["b"], float)], orc.LS, 1, np.array([0, 2]))
    assert orc.objective(pb, ex["gamma"], ex["x"]) == pytest.approx(ex["expect"], abs=1e-14)


def test_objective_random_independent_sum(orc):
    # equals per-node loss sums plus the ridge term computed independently (numpy)
    rng = np.random.default_rng(2)
    A = [rng.normal(size=(7, 6)), rng.normal(size=(5, 6))]
    b = [rng.normal(size=7), rng.normal(size=5)]
    x = rng.normal(size=6)
    pb = orc.Problem(A, b, orc.LS, 1, np.array([0, 6]))
    ref = sum(float(np.sum((a @ x - bb) ** 2)) for a, bb in zip(A, b)) + float(x @ x) / (2 * 3.0)
    assert orc.objective(pb, 3.0, x) == pytest.approx(ref, rel=1e-13)
    # S:87 invariant under shard reordering
    pb2 = orc.Problem(A[::-1], b[::-1], orc.LS, 1, np.array([0, 6]))
    assert orc.objective(pb2, 3.0, x) == pytest.approx(ref, rel=1e-13)


@pytest.mark.parametrize("ex", GOLD["kappa_from_sparsity"], ids=lambda e: e["cite"])
def test_kappa_from_sparsity(orc, ex):
    assert orc.kappa_from_sparsity(ex["n"], ex["s_l"]) == ex["expect"]


def test_kappa_from_sparsity_domain(orc):
    with pytest.raises(orc.OracleError):
        orc.kappa_from_sparsity(10, 1.0)


# ---------------------------------------------------------------- Theorem 1 geometry
@pytest.mark.parametrize("ex", GOLD["l0_witness"], ids=lambda e: e["cite"])
def test_l0_witness_spec(orc, ex):
    s, t = orc.l0_witness(ex["x"], ex["kappa"])
    assert s.tolist() == ex["s"] and t == ex["t"]


def test_l0_witness_infeasible(orc):
    with pytest.raises(orc.OracleError):
        orc.l0_witness([1, 1, 1], 2)


@pytest.mark.parametrize("ex", GOLD["check_theorem1"], ids=lambda e: e["cite"])
def test_check_theorem1_spec(orc, ex):
    assert orc.check_theorem1(ex["x"], ex["s"], ex["t"], ex["kappa"], 0.0) == ex["expect"]


def test_theorem1_property_suite(orc):
    # SPEC AC5: witnesses pass at tol 0; accepted tuples are kappa-sparse.
    rng = np.random.default_rng(3)
    for _ in range(1000):
        n = int(rng.integers(1, 12))
        kappa = int(rng.integers(0, n + 1))
        x = np.zeros(n)
        sup = rng.choice(n, size=int(rng.integers(0, kappa + 1)), replace=False)
        x[sup] = rng.normal(size=sup.size)
        s, t = orc.l0_witness(x, kappa)
        assert orc.check_theorem1(x, s, t, kappa, 0.0)
    accepted = 0
    for _ in range(1000):
        n = int(rng.integers(1, 8))
        kappa = int(rng.integers(0, n + 1))
        x = np.where(rng.random(n) < 0.5, 0.0, rng.normal(size=n))
        s = np.clip(np.round(rng.normal(size=n) * 2) / 2, -1, 1)
        t = float(np.sum(np.abs(x)))
        if orc.check_theorem1(x, s, t, kappa, 1e-9):
            accepted += 1
            assert np.count_nonzero(x) <= kappa
    assert accepted > 50


@pytest.mark.parametrize("ex", GOLD["proj_l1_epigraph"], ids=lambda e: e["cite"])
def test_proj_l1_epigraph_spec(orc, ex):
    z, t = orc.proj_l1_epigraph(ex["z"], ex["t"])
    assert np.allclose(z, ex["z_out"], atol=1e-15) and t == pytest.approx(ex["t_out"], abs=1e-15)


def test_proj_l1_epigraph_grid_and_nonexpansive(orc):
    # SPEC AC6: 2-D grid search within 2e-2; idempotent and nonexpansive at 1e-10.
    rng = np.random.default_rng(4)
    g = np.arange(-3, 3.0001, 0.01)
    Z, T = np.meshgrid(g, g, indexing="ij")
    feas = np.abs(Z) <= T
    for _ in range(50):
        z0, t0 = rng.uniform(-2.5, 2.5), rng.uniform(-2.5, 2.5)
        d = np.where(feas, (Z - z0) ** 2 + (T - t0) ** 2, np.inf)
        k = np.unravel_index(np.argmin(d), d.shape)
        zp, tp = orc.proj_l1_epigraph([z0], t0)
        assert abs(zp[0] - Z[k]) <= 2e-2 and abs(tp - T[k]) <= 2e-2
    for _ in range(1000):
        n = int(rng.integers(1, 6))
        a, b = rng.normal(size=n) * 2, rng.normal(size=n) * 2
        ta, tb = rng.normal() * 2, rng.normal() * 2
        pa, sa = orc.proj_l1_epigraph(a, ta)
        pb, sb = orc.proj_l1_epigraph(b, tb)
        pa2, sa2 = orc.proj_l1_epigraph(pa, sa)
        assert np.allclose(pa2, pa, atol=1e-10) and abs(sa2 - sa) <= 1e-10
        lhs = math.sqrt(np.sum((pa - pb) ** 2) + (sa - sb) ** 2)
        rhs = math.sqrt(np.sum((a - b) ** 2) + (ta - tb) ** 2)
        assert lhs <= rhs + 1e-10


# ---------------------------------------------------------------- per-sample prox (22)
@pytest.mark.parametrize("ex", GOLD["omega_bar"], ids=lambda e: e["cite"] + "-" + e["loss"] + str(e["p"]))
def test_omega_bar_pins(orc, ex):
    w = orc.prox_omega(LOSS[ex["loss"]], ex["M"], ex["rho_l"], ex["b"], [ex["p"]])[0]
    assert w == pytest.approx(ex["expect"], abs=2e-15)


def _prox_objective(loss, M, rho_l, b, p, w):
    # the definition (22), written from P:191-192, not the oracle's stationarity equation
    mw = M * w
    if loss == "ls":
        f = (mw - b) ** 2
    elif loss == "logistic":
        f = np.logaddexp(0.0, -b * mw)
    else:
        f = np.maximum(0.0, 1.0 - b * mw)
    return f + 0.5 * M * rho_l * (w - p) ** 2


@pytest.mark.parametrize("loss", ["ls", "logistic", "hinge"])
def test_omega_bar_minimises_definition(orc, loss):
    rng = np.random.default_rng(5)
    for _ in range(200):
        M = int(rng.integers(1, 9))
        rho_l = float(rng.choice([0.5, 1.0, 4.0, 16.0]))
        b = float(rng.normal()) if loss == "ls" else float(rng.choice([-1.0, 1.0]))
        p = float(rng.normal() * 2)
        w = orc.prox_omega(LOSS[loss], M, rho_l, b, [p])[0]
        ref = optimize.minimize_scalar(lambda v: _prox_objective(loss, M, rho_l, b, p, v),
                                       bounds=(p - 10, p + 10), method="bounded",
                                       options=dict(xatol=1e-13, maxiter=2000)).x
        assert abs(w - ref) <= 1e-6
        f = _prox_objective(loss, M, rho_l, b, p, w)
        for dv in (1e-7, -1e-7):
            assert f <= _prox_objective(loss, M, rho_l, b, p, w + dv) + 1e-14


def test_softmax_c2_reduces_to_logistic(orc):
    # C=2 softmax prox on omega: the sum is preserved and omega_1 - omega_0 is the
    # logistic prox of p_1 - p_0 with rho_l/2 (label +1 iff class 1).  Independent
    # oracle code paths (dense Newton vs bisection).
    rng = np.random.default_rng(6)
    for _ in range(200):
        M, rho_l = int(rng.integers(1, 9)), float(rng.choice([1.0, 4.0, 8.0]))
        p = rng.normal(size=2) * 2
        y = int(rng.integers(2))
        w = orc.prox_omega(orc.SOFTMAX, M, rho_l, y, p, C=2)
        d = orc.prox_omega(orc.LOGISTIC, M, rho_l / 2, 1.0 if y == 1 else -1.0, [p[1] - p[0]])[0]
        assert w.sum() == pytest.approx(p.sum(), abs=1e-13)
        assert (w[1] - w[0]) == pytest.approx(d, abs=1e-12)


def test_softmax_c10_minimises_definition(orc):
    rng = np.random.default_rng(7)
    for _ in range(30):
        M, rho_l, C = int(rng.integers(1, 9)), float(rng.choice([1.0, 4.0])), 10
        p = rng.normal(size=C) * 2
        y = int(rng.integers(C))

        def obj(w):
            mw = M * w
            return np.logaddexp.reduce(mw) - mw[y] + 0.5 * M * rho_l * np.sum((w - p) ** 2)
        w = orc.prox_omega(orc.SOFTMAX, M, rho_l, y, p, C=C)
        ref = optimize.minimize(obj, p, method="BFGS", options=dict(gtol=1e-12)).x
        assert np.max(np.abs(w - ref)) <= 1e-6
        assert obj(w) <= obj(ref) + 1e-12


def test_prox_domain_error(orc):
    with pytest.raises(orc.OracleError):
        orc.prox_omega(orc.HINGE, 1, 1.0, 0.5, [0.0])


# ---------------------------------------------------------------- (z,t)-update (7b)
def _zt_objective(wbar, s, v, N, rho_c, rho_b, z, t):
    return 0.5 * N * rho_c * np.sum((z - wbar) ** 2) + 0.5 * rho_b * (s @ z - t + v) ** 2


def test_zt_spec_example(orc):
    ex = GOLD["zt_update"][0]
    z, t, _ = orc.zt_update(ex["wbar"], ex["s"], ex["v"], ex["N"], ex["rho_c"], ex["rho_b"])
    assert np.allclose(z, ex["z"], atol=1e-15) and t == pytest.approx(ex["t"], abs=1e-15)


def test_zt_grid_search_2d(orc):
    # brute-force grid over (z1, z2, t) in [-3,3]^3; here on a 1e-2 grid in z
    # with the exact optimal t for each z, confirming the minimiser within 2e-2.
    g = np.arange(-3, 3.0001, 0.01)
    Z1, Z2 = np.meshgrid(g, g, indexing="ij")
    rng = np.random.default_rng(8)
    for _ in range(10):
        wbar, s = rng.uniform(-2, 2, size=2), rng.uniform(-1, 1, size=2)
        s = s / max(1.0, np.abs(s).sum())
        v = float(rng.normal() * 0.5)
        N, rho_c, rho_b = 1, 1.0, float(rng.choice([0.5, 1.0, 2.0]))
        l1 = np.abs(Z1) + np.abs(Z2)
        sz = s[0] * Z1 + s[1] * Z2
        T = np.maximum(l1, sz + v)
        F = 0.5 * N * rho_c * ((Z1 - wbar[0]) ** 2 + (Z2 - wbar[1]) ** 2) + 0.5 * rho_b * (sz - T + v) ** 2
        k = np.unravel_index(np.argmin(F), F.shape)
        z, t, _ = orc.zt_update(wbar, s, v, N, rho_c, rho_b)
        assert abs(z[0] - Z1[k]) <= 2e-2 and abs(z[1] - Z2[k]) <= 2e-2


def test_zt_matches_spec_pgd(orc):
    # Two independent methods for the same argmin: exact sort-and-scan vs SPEC's PGD.
    rng = np.random.default_rng(9)
    for trial in range(30):
        n = int(rng.integers(2, 40))
        wbar = rng.normal(size=n)
        s = np.zeros(n)
        idx = rng.choice(n, size=min(n, 3), replace=False)
        s[idx] = rng.uniform(-1, 1, size=idx.size)
        v = float(rng.normal())
        N, rho_c = int(rng.integers(1, 5)), float(rng.choice([1.0, 4.0]))
        rho_b = rho_c * float(rng.choice([0.25, 0.5, 1.0]))
        z, t, tau = orc.zt_update(wbar, s, v, N, rho_c, rho_b)
        zp, tp = orc.zt_pgd(wbar, s, v, N, rho_c, rho_b)
        assert np.max(np.abs(z - zp)) <= 1e-7 and abs(t - tp) <= 1e-7
        assert np.abs(z).sum() <= t + 1e-12
        assert _zt_objective(wbar, s, v, N, rho_c, rho_b, z, t) <= \
            _zt_objective(wbar, s, v, N, rho_c, rho_b, zp, tp) + 1e-12


def test_zt_rho_b_to_zero_gives_wbar(orc):
    rng = np.random.default_rng(10)
    wbar, s = rng.normal(size=20), rng.uniform(-1, 1, size=20) / 20
    z, t, _ = orc.zt_update(wbar, s, 0.3, 2, 1.0, 1e-14)
    assert np.allclose(z, wbar, atol=1e-12)


def test_zt_closed_form_sequence(orc):
    # wbar frozen at (2,1), N = rho_c = rho_b = 1, kappa = 1,
    # s0 = (1,0), v0 = 0  =>  z^k = (2, 2^-k), t^k = 2 + 2^-k, v^k = -(1 - 2^-k).
    seq = GOLD["zt_sequence"]["z2"]
    wbar, s, v = np.array([2.0, 1.0]), np.array([1.0, 0.0]), 0.0
    for k, z2 in enumerate(seq, start=1):
        z, t, tau = orc.zt_update(wbar, s, v, 1, 1.0, 1.0)
        assert z[0] == 2.0 and z[1] == pytest.approx(z2, abs=1e-15)
        assert t == pytest.approx(2 + 2.0 ** -k, abs=1e-15)
        assert tau == pytest.approx(1 - 2.0 ** -k, abs=1e-15)
        s, _ = orc.s_update(z, t, v, 1)
        g = float(z @ s - t)
        v += g
        assert abs(g) == pytest.approx(2.0 ** -k, abs=1e-15)
        assert v == pytest.approx(-(1 - 2.0 ** -k), abs=1e-15)


def test_zt_case1_tau_zero(orc):
    # psi(0) = ||w||_1 - s'w <= v  =>  z = wbar, t = s'wbar + v (App. A.1 case 1)
    wbar, s = np.array([1.0, -2.0, 0.5]), np.array([1.0, -1.0, 0.0])
    z, t, tau = orc.zt_update(wbar, s, 1.0, 3, 2.0, 1.0)
    assert tau == 0.0 and np.array_equal(z, wbar) and t == pytest.approx(3.0 + 1.0)


# ---------------------------------------------------------------- s-update (13)
@pytest.mark.parametrize("ex", GOLD["s_update"], ids=lambda e: e["cite"])
def test_s_update_spec(orc, ex):
    s, _ = orc.s_update(ex["z"], ex["t"], ex["v"], ex["kappa"])
    assert np.allclose(s, ex["s"], atol=1e-15)


def test_s_update_beats_random_probes(orc):
    # SPEC AC6: objective (z's - t + v)^2 <= that of 10^4 random feasible s.
    rng = np.random.default_rng(11)
    for _ in range(100):
        n = int(rng.integers(1, 10))
        kappa = int(rng.integers(0, n + 1))
        z, t, v = rng.normal(size=n), float(rng.normal() * 2), float(rng.normal())
        s, mcap = orc.s_update(z, t, v, kappa)
        assert np.abs(s).max(initial=0) <= 1 and np.abs(s).sum() <= kappa + 1e-12
        f = (z @ s - t + v) ** 2
        P = rng.uniform(-1, 1, size=(10_000, n))
        P *= np.minimum(1.0, kappa / np.maximum(np.abs(P).sum(1, keepdims=True), 1e-300))
        assert f <= np.min((P @ z - t + v) ** 2) + 1e-12
        # optimal value (clamp(theta, +-Mcap) - theta)^2
        th = t - v
        assert f == pytest.approx((np.clip(th, -mcap, mcap) - th) ** 2, abs=1e-12)


def test_s_update_ties_lowest_index(orc):
    s, mcap = orc.s_update([1.0, -1.0, 1.0, 0.5], 10.0, 0.0, 2)
    assert s.tolist() == [1.0, -1.0, 0.0, 0.0] and mcap == 2.0


# ---------------------------------------------------------------- linear algebra
def test_gemv_and_gemv_t_vs_numpy(orc):
    rng = np.random.default_rng(12)
    for C in (1, 3, 10):
        A = rng.normal(size=(37, 29))
        x = rng.normal(size=29 * C)
        q = rng.normal(size=37 * C)
        assert np.allclose(orc.gemv(A, x, C), (A @ x.reshape(29, C)).ravel(), rtol=1e-13, atol=1e-13)
        assert np.allclose(orc.gemv_t(A, q, C), (A.T @ q.reshape(37, C)).ravel(), rtol=1e-13, atol=1e-13)


def test_block_factor_and_solve(orc):
    rng = np.random.default_rng(13)
    A = rng.normal(size=(60, 23))
    rho_l, c = 4.0, 4.0025
    L = orc.block_factor(A, rho_l, c)
    F = rho_l * A.T @ A + c * np.eye(23)
    assert np.allclose(np.triu(L, 1), 0.0)
    assert np.allclose(L @ L.T, F, rtol=1e-13, atol=1e-12)
    rhs = rng.normal(size=23 * 2)
    x = orc.chol_solve(L, rhs, C=2)
    assert np.allclose(F @ x.reshape(23, 2), rhs.reshape(23, 2), atol=1e-12)


def test_device_x_update_special_cases(orc):
    # A = I, 1/(N gamma) -> 0, rho_c = rho_l = 1: x = (a + q)/2
    n = 5
    rng = np.random.default_rng(14)
    a, q = rng.normal(size=n), rng.normal(size=n)
    L = orc.block_factor(np.eye(n), 1.0, 1.0)
    x = orc.chol_solve(L, 1.0 * (np.eye(n).T @ q) + 1.0 * a)
    assert np.allclose(x, (a + q) / 2, atol=1e-15)
    # rho_l = 0 -> x = rho_c (z - u) / c
    A = rng.normal(size=(8, n))
    L = orc.block_factor(A, 0.0, 2.5)
    zu = rng.normal(size=n)
    assert np.allclose(orc.chol_solve(L, 2.0 * zu), 2.0 * zu / 2.5, atol=1e-15)


def test_best_subset_spec(orc):
    ex = GOLD["best_subset"][0]
    pb = orc.Problem([np.array(ex["A"], float)], [np.array(ex["b"], float)], orc.LS, 1, np.array([0, 2]))
    sup, x, obj = orc.best_subset(pb, ex["gamma"], ex["kappa"])
    assert sup.tolist() == ex["support"] and obj == pytest.approx(ex["objective_approx"], abs=1e-5)


def test_best_subset_brute_force_numpy(orc):
    # independent enumeration with numpy lstsq-free normal equations on tiny data
    rng = np.random.default_rng(15)
    A = [rng.normal(size=(15, 7)), rng.normal(size=(12, 7))]
    b = [rng.normal(size=15), rng.normal(size=12)]
    gamma = 0.5
    pb = orc.Problem(A, b, orc.LS, 1, np.array([0, 7]))
    sup, x, obj = orc.best_subset(pb, gamma, 3)
    Aall, ball = np.vstack(A), np.concatenate(b)
    best = (float(ball @ ball), ())
    for k in range(1, 4):
        for T in itertools.combinations(range(7), k):
            AT = Aall[:, T]
            xt = np.linalg.solve(2 * AT.T @ AT + np.eye(k) / gamma, 2 * AT.T @ ball)
            f = float(np.sum((AT @ xt - ball) ** 2) + xt @ xt / (2 * gamma))
            if f < best[0]:
                best = (f, T)
    assert tuple(sup.tolist()) == best[1] and obj == pytest.approx(best[0], rel=1e-11)


def test_ridge_dense_gradient(orc):
    # gradient at the solution vanishes (computed with numpy)
    rng = np.random.default_rng(16)
    A = [rng.normal(size=(20, 6)), rng.normal(size=(15, 6))]
    b = [rng.normal(size=20), rng.normal(size=15)]
    pb = orc.Problem(A, b, orc.LS, 1, np.array([0, 6]))
    x = orc.ridge_dense(pb, 2.0)
    grad = sum(2 * a.T @ (a @ x - bb) for a, bb in zip(A, b)) + x / 2.0
    assert np.max(np.abs(grad)) <= 1e-10


def test_prox_direct_ls_spec(orc):
    # A = 0, b = 0  =>  x = rho_c (z - u) / c
    rng = np.random.default_rng(17)
    z, u = rng.normal(size=4), rng.normal(size=4)
    x = orc.prox_direct_ls(np.zeros((3, 4)), np.zeros(3), 2.0, 2.5, z, u)
    assert np.allclose(x, 2.0 * (z - u) / 2.5, atol=1e-15)
    # gradient of the Eq. (8) objective at x vanishes
    A, b = rng.normal(size=(8, 5)), rng.normal(size=8)
    z, u = rng.normal(size=5), rng.normal(size=5)
    N, gamma, rho_c = 2, 3.0, 1.5
    c = 1 / (N * gamma) + rho_c
    x = orc.prox_direct_ls(A, b, rho_c, c, z, u)
    grad = 2 * A.T @ (A @ x - b) + x / (N * gamma) + rho_c * (x - z + u)
    assert np.max(np.abs(grad)) <= 1e-10


def _logistic_refit_problem(seed, N=2, m=80, n=14):
    rng = np.random.default_rng(seed)
    A = [rng.normal(size=(m, n)) / np.sqrt(m) for _ in range(N)]
    xt = np.zeros(n)
    xt[[1, 4, 9]] = [1.5, -2.0, 1.0]
    b = [np.where(a @ xt + 0.3 * rng.normal(size=m) >= 0, 1.0, -1.0) for a in A]
    return A, b


@pytest.mark.parametrize("gamma", [100.0, 0.5])
def test_refit_logistic_matches_scipy(orc, gamma):
    # DESIGN R29: the refit minimises objective (1) restricted to T; pinned against an
    # independent minimiser (scipy BFGS on the objective written with numpy) and KKT
    A, b = _logistic_refit_problem(5)
    T = np.array([1, 4, 7, 9])
    pb = orc.Problem(A, b, orc.LOGISTIC, 1, np.array([0, 14]))

    def f(x):
        return sum(np.logaddexp(0.0, -bb * (a[:, T] @ x)).sum() for a, bb in zip(A, b)) + x @ x / (2 * gamma)

    def g(x):
        return sum(a[:, T].T @ (-bb / (1.0 + np.exp(bb * (a[:, T] @ x)))) for a, bb in zip(A, b)) + x / gamma

    ref = optimize.minimize(f, np.zeros(T.size), jac=g, method="BFGS", options={"gtol": 1e-13, "maxiter": 10000})
    x = orc.refit_logistic(pb, gamma, T, np.zeros(T.size))
    assert np.max(np.abs(g(x))) <= 1e-11
    assert np.max(np.abs(x - ref.x)) <= 1e-7 * max(1.0, np.max(np.abs(ref.x)))
    # a far start (saturated margins) still converges to the same point: the line search
    x2 = orc.refit_logistic(pb, gamma, T, np.array([40.0, -40.0, 40.0, -40.0]))
    assert np.max(np.abs(x2 - x)) <= 1e-10 * max(1.0, np.max(np.abs(x)))


def test_run_logistic_refit_is_refit_of_z(orc):
    # orc_run with refit: x_final = refit_logistic started at z on the support
    A, b = _logistic_refit_problem(6, N=3, m=60, n=14)
    pb = orc.Problem(A, b, orc.LOGISTIC, 1, np.array([0, 14]))
    r = orc.run(pb, orc.Params(kappa=3, max_outer=60, inner_fixed=5, refit=1))
    T = r["support"]
    x = orc.refit_logistic(pb, 100.0, T, r["z"][T])
    assert np.allclose(r["x_final"][T], x, rtol=0, atol=1e-12)
    assert np.count_nonzero(r["x_final"]) <= 3


@pytest.mark.parametrize("gamma", [100.0, 0.5])
def test_refit_softmax_matches_scipy(orc, gamma):
    # DESIGN R29 for softmax: entry support of vec(X), pinned against scipy BFGS on the
    # objective written with numpy (logsumexp - w_y) and against KKT
    rng = np.random.default_rng(9)
    C, n, m = 4, 10, 90
    A = [rng.normal(size=(m, n)) / np.sqrt(m) for _ in range(2)]
    Xt = np.zeros((n, C))
    Xt[2, 1], Xt[5, 3], Xt[7, 0] = 2.0, -1.5, 1.0
    y = [np.argmax(a @ Xt + 0.3 * rng.normal(size=(m, C)), axis=1).astype(float) for a in A]
    T = np.array([2 * C + 1, 5 * C + 3, 7 * C + 0, 7 * C + 2, 9 * C + 1])
    L, Cc = T // C, T % C
    pb = orc.Problem(A, y, orc.SOFTMAX, C, np.array([0, n]))

    def W(a, x):
        w = np.zeros((a.shape[0], C))
        for k in range(T.size):
            w[:, Cc[k]] += a[:, L[k]] * x[k]
        return w

    def f(x):
        s = 0.0
        for a, yy in zip(A, y):
            w = W(a, x)
            s += (np.logaddexp.reduce(w, axis=1) - w[np.arange(len(yy)), yy.astype(int)]).sum()
        return s + x @ x / (2 * gamma)

    def g(x):
        out = x / gamma
        for a, yy in zip(A, y):
            w = W(a, x)
            p = np.exp(w - w.max(axis=1, keepdims=True))
            p /= p.sum(axis=1, keepdims=True)
            p[np.arange(len(yy)), yy.astype(int)] -= 1.0
            out = out + np.array([a[:, L[k]] @ p[:, Cc[k]] for k in range(T.size)])
        return out

    ref = optimize.minimize(f, np.zeros(T.size), jac=g, method="BFGS", options={"gtol": 1e-13, "maxiter": 10000})
    x = orc.refit_softmax(pb, gamma, T, np.zeros(T.size))
    assert np.max(np.abs(g(x))) <= 1e-11
    assert np.max(np.abs(x - ref.x)) <= 1e-7 * max(1.0, np.max(np.abs(ref.x)))


def test_run_softmax_refit_is_refit_of_z(orc):
    rng = np.random.default_rng(11)
    C, n, m = 3, 12, 70
    A = [rng.normal(size=(m, n)) / np.sqrt(m) for _ in range(2)]
    y = [rng.integers(0, C, size=m).astype(float) for _ in range(2)]
    pb = orc.Problem(A, y, orc.SOFTMAX, C, np.array([0, n]))
    r = orc.run(pb, orc.Params(kappa=4, max_outer=40, inner_fixed=4, refit=1))
    T = r["support"]
    x = orc.refit_softmax(pb, 100.0, T, r["z"][T])
    assert np.allclose(r["x_final"][T], x, rtol=0, atol=1e-12)
