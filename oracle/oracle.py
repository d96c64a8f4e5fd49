"""ctypes + numpy wrapper around liborc.so, the FP64 CPU ORACLE for Bi-cADMM.

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` leg may import this module.
The product path (``paper_2405_16267_b200``) never imports it, and this module
never imports the product path (it shares only the seeded input generator
``paper_2405_16267_b200.datagen``, which holds none of the method's arithmetic,
and only through the callers).

Every wrapped function cites the passage of arXiv 2405.16267 (``P:n`` = PAPER.md
line n, ``S:n`` = SPEC.md line n) it implements; see oracle/orc.c.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liborc.so")

LS, LOGISTIC, SOFTMAX, HINGE = 0, 1, 2, 3
LOSS_IDS = {"ls": LS, "logistic": LOGISTIC, "softmax": SOFTMAX, "hinge": HINGE}
TRACE_COLS = 6  # p_r, d_r, b_r, t, v, tau

_i32, _i64, _f64 = ct.c_int32, ct.c_int64, ct.c_double
_pd = ct.POINTER(ct.c_double)
_pi64 = ct.POINTER(ct.c_int64)
_pi32 = ct.POINTER(ct.c_int32)


class _Problem(ct.Structure):
    _fields_ = [("N", _i32), ("M", _i32), ("C", _i32), ("loss", _i32), ("n", _i64),
                ("m", _pi64), ("A", ct.POINTER(_pd)), ("b", ct.POINTER(_pd)),
                ("col_start", _pi64)]


class _Params(ct.Structure):
    _fields_ = [("kappa", _i64), ("rho_c", _f64), ("alpha", _f64), ("rho_l", _f64),
                ("gamma", _f64), ("eps_p", _f64), ("eps_d", _f64), ("eps_b", _f64),
                ("max_outer", _i32), ("inner_fixed", _i32), ("eps_inner", _f64),
                ("max_inner", _i32), ("refit", _i32)]


class _Result(ct.Structure):
    _fields_ = [("z", _pd), ("s", _pd), ("t", _pd), ("v", _pd), ("x", _pd), ("u", _pd),
                ("trace", _pd), ("inner_counts", _pi32), ("z_trace", _pd), ("x_trace", _pd),
                ("support", _pi64), ("support_len", _pi64), ("x_final", _pd),
                ("objective", _pd), ("iters", _pi32), ("converged", _pi32), ("timings", _pd), ("nu", _pd),
                ("step_s", _pd)]


def build(force: bool = False) -> str:
    """Compile oracle/orc.c -> oracle/liborc.so (gcc, -O2, strict IEEE, OpenMP)."""
    src = os.path.join(HERE, "orc.c")
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(src),
                                                  os.path.getmtime(os.path.join(HERE, "orc.h")))):
        return LIB_PATH
    cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
           "-fPIC", "-shared", "-o", LIB_PATH + ".tmp", src, "-lm"]
    subprocess.run(cmd, check=True, cwd=HERE)
    os.replace(LIB_PATH + ".tmp", LIB_PATH)
    return LIB_PATH


_lib = None


def lib() -> ct.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ct.CDLL(LIB_PATH)
        L.orc_phi.restype = _f64
        L.orc_phi.argtypes = [ct.c_int, ct.c_int, _pd, _f64]
        L.orc_loss_value.argtypes = [ct.c_int, ct.c_int, _i64, _pd, _pd, _pd]
        L.orc_objective.argtypes = [ct.POINTER(_Problem), _f64, _pd, _pd]
        L.orc_kappa_from_sparsity.restype = _i64
        L.orc_kappa_from_sparsity.argtypes = [_i64, _f64]
        L.orc_l0_witness.argtypes = [_i64, _pd, _i64, _pd, _pd]
        L.orc_check_theorem1.argtypes = [_i64, _pd, _pd, _f64, _f64, _f64]
        L.orc_proj_l1_epigraph.argtypes = [_i64, _pd, _f64, _pd, _pd]
        L.orc_prox_omega.argtypes = [ct.c_int, ct.c_int, ct.c_int, _f64, _f64, _pd, _pd]
        L.orc_zt_update.argtypes = [_i64, ct.c_int, _f64, _f64, _pd, _pd, _f64, _pd, _pd, _pd]
        L.orc_s_update.argtypes = [_i64, _i64, _pd, _f64, _f64, _pd, _pd]
        L.orc_zt_pgd.argtypes = [_i64, ct.c_int, _f64, _f64, _pd, _pd, _f64, _f64, ct.c_int, _pd, _pd]
        L.orc_gemv.argtypes = [_i64, _i64, _pd, _i64, ct.c_int, _pd, _pd]
        L.orc_gemv_t.argtypes = [_i64, _i64, _pd, _i64, ct.c_int, _pd, _pd]
        L.orc_block_factor.argtypes = [_i64, _i64, _pd, _i64, _f64, _f64, _pd]
        L.orc_chol_solve.argtypes = [_i64, _pd, ct.c_int, _pd, _pd]
        L.orc_run.argtypes = [ct.POINTER(_Problem), ct.POINTER(_Params), _pi32, ct.POINTER(_Result)]
        L.orc_prox_direct_ls.argtypes = [_i64, _i64, _pd, _pd, _f64, _f64, _pd, _pd, _pd]
        L.orc_ridge_dense.argtypes = [ct.POINTER(_Problem), _f64, _pd]
        L.orc_refit_ls.argtypes = [ct.POINTER(_Problem), _f64, _i64, _pi64, _pd]
        L.orc_refit_logistic.argtypes = [ct.POINTER(_Problem), _f64, _i64, _pi64, _pd]
        L.orc_refit_softmax.argtypes = [ct.POINTER(_Problem), _f64, _i64, _pi64, _pd]
        L.orc_best_subset.argtypes = [ct.POINTER(_Problem), _f64, _i64, _pi64, _pi64, _pd, _pd]
        _lib = L
    return _lib


def _d(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_pd)


def _f64c(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class _Check(RuntimeError):
    pass


def _rc(rc: int) -> None:
    if rc != 0:
        raise _Check({-1: "invalid", -2: "dim", -3: "domain", -4: "infeasible", -5: "nomem"}.get(rc, str(rc)))


OracleError = _Check


# ----------------------------------------------------------------------------- problem
@dataclass
class Problem:
    """Node shards A_i (m_i x n, row-major FP64), labels b_i, loss, classes C and the
    contiguous feature-block boundaries col_start (DESIGN R16)."""
    A: list
    b: list
    loss: int
    C: int
    col_start: np.ndarray
    _keep: list = field(default_factory=list, repr=False)

    @property
    def N(self):
        return len(self.A)

    @property
    def n(self):
        return self.A[0].shape[1]

    @property
    def M(self):
        return len(self.col_start) - 1

    def struct(self) -> _Problem:
        A = [_f64c(a) for a in self.A]
        b = [_f64c(x) for x in self.b]
        m = np.array([a.shape[0] for a in A], dtype=np.int64)
        cs = np.ascontiguousarray(self.col_start, dtype=np.int64)
        Ap = (_pd * len(A))(*[_d(a) for a in A])
        bp = (_pd * len(b))(*[_d(x) for x in b])
        self._keep = [A, b, m, cs, Ap, bp]
        return _Problem(len(A), len(cs) - 1, self.C, self.loss, A[0].shape[1],
                        m.ctypes.data_as(_pi64), Ap, bp, cs.ctypes.data_as(_pi64))


@dataclass
class Params:
    kappa: int
    rho_c: float = 4.0
    alpha: float = 0.5
    rho_l: float = 4.0
    gamma: float = 100.0
    eps_p: float = 1e-4
    eps_d: float = 1e-4
    eps_b: float = 1e-4
    max_outer: int = 1000
    inner_fixed: int = 10
    eps_inner: float = 1e-6
    max_inner: int = 200
    refit: int = 1

    def struct(self) -> _Params:
        return _Params(self.kappa, self.rho_c, self.alpha, self.rho_l, self.gamma, self.eps_p,
                       self.eps_d, self.eps_b, self.max_outer, self.inner_fixed, self.eps_inner,
                       self.max_inner, self.refit)


def run(problem: Problem, params: Params, schedule=None, trace_z: bool = False, trace_x: bool = False) -> dict:
    """Algorithm 1 with Algorithm 2 as the x-step, Eq. (7) order."""
    L = lib()
    N, n, C, K = problem.N, problem.n, problem.C, params.max_outer
    ln = n * C
    out = dict(z=np.zeros(ln), s=np.zeros(ln), t=np.zeros(1), v=np.zeros(1),
               x=np.zeros((N, ln)), u=np.zeros((N, ln)), trace=np.zeros((K, TRACE_COLS)),
               inner_counts=np.zeros((K, N), dtype=np.int32),
               support=np.zeros(max(params.kappa, 1), dtype=np.int64),
               support_len=np.zeros(1, dtype=np.int64), x_final=np.zeros(ln),
               objective=np.zeros(1), iters=np.zeros(1, dtype=np.int32),
               converged=np.zeros(1, dtype=np.int32), timings=np.zeros(4), step_s=np.zeros(K),
               nu=np.zeros(max(1, int(sum(a.shape[0] for a in problem.A)) * C)))
    zt = np.zeros((K, ln)) if trace_z else None
    xt = np.zeros((K, N, ln)) if trace_x else None
    res = _Result(_d(out["z"]), _d(out["s"]), _d(out["t"]), _d(out["v"]), _d(out["x"]), _d(out["u"]),
                  _d(out["trace"]), out["inner_counts"].ctypes.data_as(_pi32),
                  _d(zt) if zt is not None else None, _d(xt) if xt is not None else None,
                  out["support"].ctypes.data_as(_pi64), out["support_len"].ctypes.data_as(_pi64),
                  _d(out["x_final"]), _d(out["objective"]), out["iters"].ctypes.data_as(_pi32),
                  out["converged"].ctypes.data_as(_pi32), _d(out["timings"]), _d(out["nu"]), _d(out["step_s"]))
    sched = None
    if schedule is not None:
        schedule = np.ascontiguousarray(schedule, dtype=np.int32)
        assert schedule.shape == (K, N)
        sched = schedule.ctypes.data_as(_pi32)
    ps, pp = problem.struct(), params.struct()
    _rc(L.orc_run(ct.byref(ps), ct.byref(pp), sched, ct.byref(res)))
    it = int(out["iters"][0])
    return dict(z=out["z"], s=out["s"], t=float(out["t"][0]), v=float(out["v"][0]), x=out["x"],
                u=out["u"], trace=out["trace"][:it], inner_counts=out["inner_counts"][:it],
                support=out["support"][:int(out["support_len"][0])], x_final=out["x_final"],
                objective=float(out["objective"][0]), iters=it, converged=bool(out["converged"][0]),
                timings=dict(zip(("setup_s", "inner_s", "outer_s", "total_s"), out["timings"].tolist())),
                step_s=out["step_s"][:it],
                nu=np.split(out["nu"][:int(sum(a.shape[0] for a in problem.A)) * C], np.cumsum([a.shape[0] * C for a in problem.A])[:-1]),
                z_trace=None if zt is None else zt[:it], x_trace=None if xt is None else xt[:it])


# ----------------------------------------------------------------------------- single ops
def phi(loss: int, w, b: float, C: int = 1) -> float:
    w = _f64c(np.atleast_1d(w))
    return lib().orc_phi(loss, C, _d(w), float(b))


def loss_value(loss: int, w, b, C: int = 1) -> float:
    w, b = _f64c(w), _f64c(b)
    out = np.zeros(1)
    m = b.shape[0]
    if w.size != m * C:
        raise OracleError("dim")
    _rc(lib().orc_loss_value(loss, C, m, _d(w), _d(b), _d(out)))
    return float(out[0])


def objective(problem: Problem, gamma: float, x) -> float:
    x = _f64c(x)
    out = np.zeros(1)
    ps = problem.struct()
    _rc(lib().orc_objective(ct.byref(ps), gamma, _d(x), _d(out)))
    return float(out[0])


def kappa_from_sparsity(n: int, s_l: float) -> int:
    k = lib().orc_kappa_from_sparsity(n, s_l)
    if k < 0:
        raise OracleError("domain")
    return int(k)


def l0_witness(x, kappa: int):
    x = _f64c(x)
    s, t = np.zeros_like(x), np.zeros(1)
    _rc(lib().orc_l0_witness(x.size, _d(x), kappa, _d(s), _d(t)))
    return s, float(t[0])


def check_theorem1(x, s, t: float, kappa: float, tol: float) -> bool:
    x, s = _f64c(x), _f64c(s)
    return bool(lib().orc_check_theorem1(x.size, _d(x), _d(s), t, float(kappa), tol))


def proj_l1_epigraph(z, t: float):
    z = _f64c(z)
    zo, to = np.zeros_like(z), np.zeros(1)
    lib().orc_proj_l1_epigraph(z.size, _d(z), t, _d(zo), _d(to))
    return zo, float(to[0])


def prox_omega(loss: int, M: int, rho_l: float, b: float, p, C: int = 1) -> np.ndarray:
    p = _f64c(np.atleast_1d(p))
    out = np.zeros(C)
    _rc(lib().orc_prox_omega(loss, C, M, rho_l, float(b), _d(p), _d(out)))
    return out


def zt_update(wbar, s, v: float, N: int, rho_c: float, rho_b: float):
    wbar, s = _f64c(wbar), _f64c(s)
    z, t, tau = np.zeros_like(wbar), np.zeros(1), np.zeros(1)
    lib().orc_zt_update(wbar.size, N, rho_c, rho_b, _d(wbar), _d(s), v, _d(z), _d(t), _d(tau))
    return z, float(t[0]), float(tau[0])


def zt_pgd(wbar, s, v: float, N: int, rho_c: float, rho_b: float, step_tol=1e-12, max_steps=200000):
    wbar, s = _f64c(wbar), _f64c(s)
    z, t = np.zeros_like(wbar), np.zeros(1)
    lib().orc_zt_pgd(wbar.size, N, rho_c, rho_b, _d(wbar), _d(s), v, step_tol, max_steps, _d(z), _d(t))
    return z, float(t[0])


def s_update(z, t: float, v: float, kappa: int):
    z = _f64c(z)
    s, mcap = np.zeros_like(z), np.zeros(1)
    lib().orc_s_update(z.size, kappa, _d(z), t, v, _d(s), _d(mcap))
    return s, float(mcap[0])


def gemv(A, x, C: int = 1) -> np.ndarray:
    A, x = _f64c(A), _f64c(x)
    m, nj = A.shape
    y = np.zeros(m * C)
    lib().orc_gemv(m, nj, _d(A), nj, C, _d(x), _d(y))
    return y


def gemv_t(A, q, C: int = 1) -> np.ndarray:
    A, q = _f64c(A), _f64c(q)
    m, nj = A.shape
    y = np.zeros(nj * C)
    lib().orc_gemv_t(m, nj, _d(A), nj, C, _d(q), _d(y))
    return y


def block_factor(A, rho_l: float, c: float) -> np.ndarray:
    A = _f64c(A)
    m, nj = A.shape
    L = np.zeros((nj, nj))
    _rc(lib().orc_block_factor(m, nj, _d(A), nj, rho_l, c, _d(L)))
    return L


def chol_solve(L, rhs, C: int = 1) -> np.ndarray:
    L, rhs = _f64c(L), _f64c(rhs)
    x = np.zeros_like(rhs)
    lib().orc_chol_solve(L.shape[0], _d(L), C, _d(rhs), _d(x))
    return x


def prox_direct_ls(A, b, rho_c: float, c: float, z, u) -> np.ndarray:
    A, b, z, u = _f64c(A), _f64c(b), _f64c(z), _f64c(u)
    x = np.zeros(A.shape[1])
    _rc(lib().orc_prox_direct_ls(A.shape[0], A.shape[1], _d(A), _d(b), rho_c, c, _d(z), _d(u), _d(x)))
    return x


def ridge_dense(problem: Problem, gamma: float) -> np.ndarray:
    x = np.zeros(problem.n)
    ps = problem.struct()
    _rc(lib().orc_ridge_dense(ct.byref(ps), gamma, _d(x)))
    return x


def refit_ls(problem: Problem, gamma: float, T) -> np.ndarray:
    T = np.ascontiguousarray(T, dtype=np.int64)
    x = np.zeros(T.size)
    ps = problem.struct()
    _rc(lib().orc_refit_ls(ct.byref(ps), gamma, T.size, T.ctypes.data_as(_pi64), _d(x)))
    return x


def refit_logistic(problem: Problem, gamma: float, T, x0) -> np.ndarray:
    """Logistic refit on support T (DESIGN R29), damped Newton from x0."""
    T = np.ascontiguousarray(T, dtype=np.int64)
    x = np.ascontiguousarray(x0, dtype=np.float64).copy()
    ps = problem.struct()
    _rc(lib().orc_refit_logistic(ct.byref(ps), gamma, T.size, T.ctypes.data_as(_pi64), _d(x)))
    return x


def refit_softmax(problem: Problem, gamma: float, T, x0) -> np.ndarray:
    """Softmax refit on the entry support T of vec(X) (DESIGN R29), damped Newton from x0."""
    T = np.ascontiguousarray(T, dtype=np.int64)
    x = np.ascontiguousarray(x0, dtype=np.float64).copy()
    ps = problem.struct()
    _rc(lib().orc_refit_softmax(ct.byref(ps), gamma, T.size, T.ctypes.data_as(_pi64), _d(x)))
    return x


def best_subset(problem: Problem, gamma: float, kappa: int):
    sup, sl = np.zeros(max(kappa, 1), dtype=np.int64), np.zeros(1, dtype=np.int64)
    x, obj = np.zeros(problem.n), np.zeros(1)
    ps = problem.struct()
    _rc(lib().orc_best_subset(ct.byref(ps), gamma, kappa, sup.ctypes.data_as(_pi64),
                              sl.ctypes.data_as(_pi64), _d(x), _d(obj)))
    return sup[:int(sl[0])].copy(), x, float(obj[0])
