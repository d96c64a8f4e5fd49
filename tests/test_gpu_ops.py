"""GPU parity of each hot-path step (bicadmm_ops.h entry points, i.e. the same
kernels the solver launches) against the FP64 oracle, element by element, on
seeded inputs spanning several tiles and a ragged tail.

Tolerances: FP64 storage -> 1e-12 relative (reduction-order rounding only);
FP32 storage of A -> compared with the oracle on the same FP32-rounded matrix
in FP64 (the kernels accumulate in FP64), so also ~1e-12."""
import ctypes as ct

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bc():
    from paper_2405_16267_b200 import build
    build.build()
    from paper_2405_16267_b200 import bicadmm
    bicadmm.lib()
    assert torch.cuda.is_available()
    return bicadmm


def _p(t):
    return ct.c_void_p(t.data_ptr())


def _s():
    return ct.c_void_p(torch.cuda.current_stream().cuda_stream)


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


SHAPES = [(1, 1), (7, 3), (300, 50), (1037, 513), (2050, 1026), (129, 4099)]


@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("m,nj", SHAPES)
def test_gemv(bc, orc, dt, m, nj):
    rng = np.random.default_rng(m * 7 + nj)
    lda = -(-nj // 4) * 4 + 4
    Ah = rng.normal(size=(m, lda))
    tdt = torch.float64 if dt == "f64" else torch.float32
    A = torch.tensor(Ah, dtype=tdt, device="cuda")
    x = torch.tensor(rng.normal(size=nj), dtype=torch.float64, device="cuda")
    y = torch.zeros(m, dtype=torch.float64, device="cuda")
    bc.check(bc.lib().bicadmm_op_gemv(bc.F64 if dt == "f64" else bc.F32, m, nj, _p(A), lda, _p(x), _p(y), _s()))
    torch.cuda.synchronize()
    Aref = A.double().cpu().numpy()[:, :nj]
    ref = orc.gemv(Aref, x.cpu().numpy())
    assert _rel(y.cpu().numpy(), ref) <= 1e-12


@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("m,nj", SHAPES)
def test_gemv_t(bc, orc, dt, m, nj):
    rng = np.random.default_rng(m * 3 + nj)
    lda = -(-nj // 4) * 4
    tdt = torch.float64 if dt == "f64" else torch.float32
    A = torch.tensor(rng.normal(size=(m, lda)), dtype=tdt, device="cuda")
    p = torch.tensor(rng.normal(size=m), dtype=torch.float64, device="cuda")
    d = torch.tensor(rng.normal(size=m), dtype=torch.float64, device="cuda")
    z = torch.tensor(rng.normal(size=nj), dtype=torch.float64, device="cuda")
    u = torch.tensor(rng.normal(size=nj), dtype=torch.float64, device="cuda")
    r = torch.zeros(nj, dtype=torch.float64, device="cuda")
    dtc = bc.F64 if dt == "f64" else bc.F32
    wsb = bc.lib().bicadmm_op_gemv_t_ws(dtc, m, nj)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    bc.check(bc.lib().bicadmm_op_gemv_t(dtc, m, nj, _p(A), lda, _p(p), _p(d), _p(z), _p(u), 4.0, 2.5, _p(r),
                                        _p(ws), wsb, _s()))
    torch.cuda.synchronize()
    Aref = A.double().cpu().numpy()[:, :nj]
    q = p.cpu().numpy() + d.cpu().numpy()
    ref = 4.0 * orc.gemv_t(Aref, q) + 2.5 * (z.cpu().numpy() - u.cpu().numpy())
    assert _rel(r.cpu().numpy(), ref) <= 1e-12


@pytest.mark.parametrize("loss", ["ls", "logistic", "hinge"])
@pytest.mark.parametrize("M", [1, 3, 8])
def test_prox(bc, orc, loss, M):
    rng = np.random.default_rng(M)
    m = 3001
    b = rng.normal(size=m) if loss == "ls" else np.where(rng.random(m) < 0.5, -1.0, 1.0)
    S = rng.normal(size=m) * 3
    nu = rng.normal(size=m)
    rho_l = 4.0
    tb = torch.tensor(b, device="cuda")
    tS = torch.tensor(S, device="cuda")
    tnu = torch.tensor(nu, device="cuda")
    td = torch.zeros(m, dtype=torch.float64, device="cuda")
    tom = torch.zeros(m, dtype=torch.float64, device="cuda")
    lid = bc.LOSSES[loss]
    bc.check(bc.lib().bicadmm_op_prox(lid, bc.F64, 1, m, M, rho_l, _p(tb), _p(tS), _p(tnu), _p(td), _p(tom), _s()))
    torch.cuda.synchronize()
    abar = S / M
    om = np.array([orc.prox_omega(lid, M, rho_l, b[r], [abar[r] + nu[r]])[0] for r in range(m)])
    nu_new = nu + abar - om
    delta = om - abar - nu_new
    assert np.max(np.abs(tom.cpu().numpy() - om) / np.maximum(1, np.abs(om))) <= 1e-14
    assert np.max(np.abs(tnu.cpu().numpy() - nu_new)) <= 1e-13
    assert np.max(np.abs(td.cpu().numpy() - delta)) <= 1e-13


@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("m,nj", [(40, 3), (300, 64), (1000, 130), (700, 257)])
def test_block_factor(bc, orc, dt, m, nj):
    rng = np.random.default_rng(nj)
    lda = -(-nj // 4) * 4
    tdt = torch.float64 if dt == "f64" else torch.float32
    Ah = rng.normal(size=(m, lda)) / np.sqrt(m)
    A = torch.tensor(Ah, dtype=tdt, device="cuda")
    rho_l, c = 4.0, 4.0025
    ldh = lda
    H = torch.zeros(nj, ldh, dtype=tdt, device="cuda")
    dtc = bc.F64 if dt == "f64" else bc.F32
    wsb = bc.lib().bicadmm_op_block_factor_ws(nj)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    bc.check(bc.lib().bicadmm_op_block_factor(dtc, m, nj, _p(A), lda, rho_l, c, _p(H), ldh, _p(ws), wsb, _s()))
    torch.cuda.synchronize()
    Aref = A.double().cpu().numpy()[:, :nj]
    L = orc.block_factor(Aref, rho_l, c)
    F = L @ L.T
    Hn = H.double().cpu().numpy()[:, :nj]
    tol = 1e-13 if dt == "f64" else 2e-7
    assert np.max(np.abs(Hn @ F - np.eye(nj))) <= tol * 10
    rhs = rng.normal(size=nj)
    assert _rel(Hn @ rhs, orc.chol_solve(L, rhs)) <= tol
    assert np.array_equal(Hn, Hn.T)


@pytest.mark.parametrize("m,nj", [(33, 5), (517, 70), (2000, 129)])
def test_gram(bc, m, nj):
    rng = np.random.default_rng(m)
    A = torch.tensor(rng.normal(size=(m, -(-nj // 4) * 4)), device="cuda")
    G = torch.zeros(nj, nj, dtype=torch.float64, device="cuda")
    bc.check(bc.lib().bicadmm_op_gram(bc.F64, m, nj, _p(A), A.stride(0), 2.0, 0.5, _p(G), nj, _s()))
    torch.cuda.synchronize()
    An = A.cpu().numpy()[:, :nj]
    ref = 2.0 * An.T @ An + 0.5 * np.eye(nj)
    assert np.max(np.abs(G.cpu().numpy() - ref)) <= 1e-12 * np.max(np.abs(ref))


@pytest.mark.parametrize("m,nj,dt", [(33, 5, "f64"), (517, 70, "f64"), (2000, 129, "f64"), (40000, 300, "f64"),
                                     (3000, 200, "f32"), (70001, 64, "f64")])
def test_gram_tc(bc, m, nj, dt):
    # tcgen05 kind::i8 Ozaki-scheme Gram (lower triangle) vs the FP64 definition; columns of
    # very different magnitudes (per-column scaling), ragged sizes, several 32768-row chunks
    rng = np.random.default_rng(m + nj)
    An = rng.normal(size=(m, -(-nj // 4) * 4)) * np.exp(rng.uniform(-6, 6, size=-(-nj // 4) * 4))
    tdt = torch.float64 if dt == "f64" else torch.float32
    A = torch.tensor(An, device="cuda", dtype=tdt)
    An = A.double().cpu().numpy()[:, :nj]
    G = torch.full((nj, nj), 7.0, dtype=torch.float64, device="cuda")
    code = bc.F64 if dt == "f64" else bc.F32
    wsb = bc.lib().bicadmm_op_gram_tc_ws(code, m, nj)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    bc.check(bc.lib().bicadmm_op_gram_tc(code, m, nj, _p(A), A.stride(0), 2.0, 0.5, _p(G), nj, _p(ws), wsb, _s()))
    torch.cuda.synchronize()
    Gn = G.cpu().numpy()
    ref = 2.0 * An.T @ An + 0.5 * np.eye(nj)
    lo = np.tril_indices(nj)
    d = np.sqrt(np.abs(np.diag(ref)))
    err = np.abs(Gn - ref)[lo] / np.outer(d, d)[lo]     # relative to sqrt(G_ii G_jj)
    assert np.max(err) <= 3e-14   # S = 7 round-to-nearest digits: measured <= 5e-15
    assert np.all(Gn[np.triu_indices(nj, 1)] == 7.0)     # upper triangle untouched


GEMM_TC_CASES = [
    # name, M, N, K, layout, flags, beta
    ("rect_rowmajor", 300, 200, 500, "nn", 0, 0.0),
    ("rect_beta_ragged", 131, 77, 33, "nt", 0, -0.5),
    ("syrk_lower", 260, 260, 190, "nt", 1, 1.0),
    ("tri_hi_B", 200, 250, 250, "trB_hi", 2 << 8, 0.0),      # X = F21 W11^T (B_op(k,j)=0 for k > j)
    ("tri_lo_B", 200, 250, 250, "trB_lo", 2 << 4, 0.0),      # X = L21 W11 (B_op(k,j)=0 for k < j)
    ("tri_hi_A", 260, 140, 260, "trA_hi", 1 << 8, 0.0),      # W21 = -W22 X (A_op(i,k)=0 for k > i)
    ("tri_gram_mirror", 333, 333, 333, "wtw", 1 | 2 | (3 << 4), 0.0),   # H = W^T W
    ("long_k_chunks", 64, 96, 70000, "nn", 0, 0.0),
]


@pytest.mark.parametrize("case", GEMM_TC_CASES, ids=[c[0] for c in GEMM_TC_CASES])
def test_gemm_tc(bc, case):
    # the a0 factor's large products on the tcgen05 Ozaki engine vs the FP64 definition, with
    # the zero structures whose tiles it skips; error relative to ||A_op(i,:)|| ||B_op(:,j)||
    name, M, N, K, layout, flags, beta = case
    rng = np.random.default_rng(M + N + K)
    lo_scale = np.exp(rng.uniform(-4, 4, size=max(M, N, K)))
    A = rng.normal(size=(M, K)) * lo_scale[:M, None]
    B = rng.normal(size=(K, N)) * lo_scale[None, :N]
    same = 0
    if layout == "trB_hi":
        B = np.tril(rng.normal(size=(N, K))).T          # B_op(k,j) = W[j][k], W lower
    elif layout == "trB_lo":
        B = np.tril(rng.normal(size=(K, N)))            # B_op(k,j) = W[k][j], W lower
    elif layout == "trA_hi":
        A = np.tril(rng.normal(size=(M, K)))            # A_op(i,k) = W[i][k], W lower
    elif layout == "wtw":
        W = np.tril(rng.normal(size=(K, M)) * lo_scale[None, :M])
        A, B, same = W.T, W, 1
    C0 = rng.normal(size=(M, N))
    ref = A @ B + beta * C0
    # device operands in the layouts the factor uses
    if layout == "nt":                                  # B_op(k,j) = Bs[j][k] (row-major N x K)
        Bs = torch.tensor(np.ascontiguousarray(B.T), device="cuda")
        b_sl, b_sr = Bs.stride(0), 1
    elif layout == "trB_hi":
        Bs = torch.tensor(np.ascontiguousarray(B.T), device="cuda")
        b_sl, b_sr = Bs.stride(0), 1
    else:                                               # row-major K x N
        Bs = torch.tensor(np.ascontiguousarray(B), device="cuda")
        b_sl, b_sr = 1, Bs.stride(0)
    if layout == "wtw":                                 # A_op(i,k) = W[k][i]
        As = torch.tensor(np.ascontiguousarray(W), device="cuda")
        a_sl, a_sr = 1, As.stride(0)
    else:
        As = torch.tensor(np.ascontiguousarray(A), device="cuda")
        a_sl, a_sr = As.stride(0), 1
    C = torch.tensor(C0, device="cuda")
    if flags & 1:
        C.copy_(torch.tensor(np.where(np.tril(np.ones((M, N))) > 0, C0, 7.0), device="cuda"))
    L = bc.lib()
    wsb = L.bicadmm_op_gemm_tc_ws(M, N, K, same)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    bc.check(L.bicadmm_op_gemm_tc(bc.F64, M, N, K, _p(As), a_sl, a_sr, _p(Bs), b_sl, b_sr, same, 1.0, beta, 0.0,
                                  _p(C), C.stride(0), flags, _p(ws), wsb, _s()))
    torch.cuda.synchronize()
    Cn = C.cpu().numpy()
    scale = np.outer(np.linalg.norm(A, axis=1), np.linalg.norm(B, axis=0)) + abs(beta) * np.abs(C0)
    err = np.abs(Cn - ref) / np.maximum(scale, 1e-300)
    if flags & 1:
        lo = np.tril_indices(M)
        assert np.max(err[lo]) <= 3e-14
        if flags & 2:
            assert np.array_equal(Cn, Cn.T)
        else:
            assert np.all(Cn[np.triu_indices(M, 1)] == 7.0)
    else:
        assert np.max(err) <= 3e-14


ZT_CASES = []
_rng = np.random.default_rng(42)
for _k in range(12):
    _n = int(_rng.choice([2, 50, 1000, 4097, 30011]))
    _w = _rng.normal(size=_n)
    _sv = np.zeros(_n)
    _idx = _rng.choice(_n, size=min(_n, 5), replace=False)
    _sv[_idx] = _rng.uniform(-1, 1, size=_idx.size) if _k % 3 else np.sign(_w[_idx])
    _v = float(_rng.normal() * (0.1 if _k % 4 else 10))
    ZT_CASES.append((_w, _sv, _v, int(_rng.integers(1, 9)), float(_rng.choice([1.0, 4.0])), float(_rng.choice([0.5, 1.0]))))
ZT_CASES.append((np.array([2.0, 1.0]), np.array([1.0, 0.0]), 0.0, 1, 1.0, 1.0))
ZT_CASES.append((np.array([1.0, -2.0, 0.5]), np.array([1.0, -1.0, 0.0]), 1.0, 3, 2.0, 0.5))  # case 1
ZT_CASES.append((np.zeros(7), np.zeros(7), -1.0, 2, 1.0, 0.5))                              # all zero


@pytest.mark.parametrize("case", range(len(ZT_CASES)))
def test_zt(bc, orc, case):
    w, s, v, N, rho_c, alpha = ZT_CASES[case]
    rho_b = alpha * rho_c
    n = w.size
    wsum = torch.tensor(w * N, device="cuda")       # the kernel divides by N
    ts = torch.tensor(s, device="cuda")
    wbar = torch.zeros(n, dtype=torch.float64, device="cuda")
    z = torch.tensor(np.full(n, 0.25), device="cuda")
    zp = torch.zeros(n, dtype=torch.float64, device="cuda")
    out = (ct.c_double * 4)()
    bc.check(bc.lib().bicadmm_op_zt(n, N, rho_c, rho_b, _p(wsum), _p(ts), v, _p(wbar), _p(z), _p(zp), out, _s()))
    wb = (w * N) / N
    zr, tr, taur = orc.zt_update(wb, s, v, N, rho_c, rho_b)
    zg = z.cpu().numpy()
    assert np.max(np.abs(zg - zr)) <= 1e-12 * max(1.0, np.max(np.abs(zr)))
    assert abs(out[0] - tr) <= 1e-12 * max(1.0, abs(tr))
    assert abs(out[1] - taur) <= 1e-12 * max(1.0, abs(taur))
    assert np.all(zp.cpu().numpy() == 0.25)
    assert out[2] == pytest.approx(np.sum((zg - 0.25) ** 2), rel=1e-12, abs=1e-300)


S_CASES = []
_rng = np.random.default_rng(7)
for _k in range(10):
    _n = int(_rng.choice([1, 3, 100, 5000, 40000]))
    _z = _rng.normal(size=_n)
    if _k % 3 == 0:
        _z = np.round(_z * 2) / 2          # many ties
    if _k % 4 == 1:
        _z[_rng.random(_n) < 0.7] = 0.0    # many zeros
    S_CASES.append((_z, float(_rng.normal() * 3), float(_rng.normal()), int(_rng.integers(0, _n + 2))))
S_CASES.append((np.array([3.0, 1.0, -2.0]), 10.0, 0.0, 2))
S_CASES.append((np.array([3.0, 1.0, -2.0]), 2.5, 0.0, 2))
S_CASES.append((np.array([1.0, -1.0, 1.0, 0.5]), 10.0, 0.0, 2))  # ties -> lower index


@pytest.mark.parametrize("case", range(len(S_CASES)))
def test_s_update_and_support(bc, orc, case):
    z, t, v, kappa = S_CASES[case]
    n = z.size
    tz = torch.tensor(z, device="cuda")
    s = torch.full((n,), 7.0, dtype=torch.float64, device="cuda")
    out = (ct.c_double * 3)()
    bc.check(bc.lib().bicadmm_op_s_update(n, kappa, _p(tz), t, v, _p(s), out, _s()))
    sr, mcap = orc.s_update(z, t, v, kappa)
    sg = s.cpu().numpy()
    assert np.array_equal(sg != 0, sr != 0)             # identical selection T (integer decision)
    assert np.max(np.abs(sg - sr)) <= 1e-14             # scale differs only by Mcap's summation order
    assert out[0] == pytest.approx(mcap, rel=1e-13, abs=0)
    g = float(z @ sr - t)
    assert out[1] == pytest.approx(g, rel=1e-12, abs=1e-12 * max(1, abs(t)))
    # support: top-kappa of |z| among nonzeros, ties to the lower index, ascending
    sup = torch.zeros(max(kappa, 1), dtype=torch.int64, device="cuda")
    cnt = (ct.c_int64 * 1)()
    bc.check(bc.lib().bicadmm_op_support(n, kappa, _p(tz), _p(sup), cnt, _s()))
    order = sorted(range(n), key=lambda l: (-abs(z[l]), l))
    ref = sorted(l for l in order[:min(kappa, n)] if z[l] != 0.0)
    assert cnt[0] == len(ref)
    assert sup.cpu().numpy()[:cnt[0]].tolist() == ref
