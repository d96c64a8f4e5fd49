"""Thin ctypes binding of libbicadmm.so (include/bicadmm.h, include/bicadmm_ops.h).

Argument marshalling only: every step of the Bi-cADMM path runs in the CUDA
kernels of the library.  There is no CPU fallback: ``lib()`` raises if the
extension is missing or cannot be loaded.  torch supplies device memory (the
caller's matrices and the workspace tensor) and the CUDA stream.

The ABI functions keep their C names (``bicadmm_setup`` ...).  ``BiCADMM`` is a
convenience wrapper that builds the problem/params structs from torch tensors.
"""
from __future__ import annotations

import ctypes as ct
import os
from dataclasses import dataclass

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libbicadmm.so")

OK, ERR_INVALID, ERR_DIM, ERR_DOMAIN, ERR_PLACEMENT, ERR_OOM, ERR_CUDA, ERR_NCCL, ERR_STATE = 0, -1, -2, -3, -4, -5, -6, -7, -8
LS, LOGISTIC, SOFTMAX, HINGE = 0, 1, 2, 3
LOSSES = {"ls": LS, "logistic": LOGISTIC, "softmax": SOFTMAX, "hinge": HINGE}
F64, F32 = 0, 1
(FIELD_Z, FIELD_S, FIELD_SCALARS, FIELD_X_LOCAL, FIELD_U_LOCAL, FIELD_SUPPORT, FIELD_X_FINAL,
 FIELD_TRACE, FIELD_WBAR, FIELD_NU, FIELD_INNER_COUNTS, FIELD_LAUNCHES, FIELD_PHASE_MS, FIELD_PHASE_COUNT,
 FIELD_SWEEP_KIND, FIELD_P_LOCAL, FIELD_R_LOCAL) = range(17)
NPHASE = 8
PHASES = ("gemv_t_partial", "gemv_t_reduce", "h_apply", "gemv", "allreduce", "prox", "global_step", "fused_sweep")
SWEEP_AUTO, SWEEP_TWO_PASS, SWEEP_FUSED = 0, 1, 2

_i32, _i64, _f64, _vp = ct.c_int32, ct.c_int64, ct.c_double, ct.c_void_p


class bicadmm_block(ct.Structure):
    _fields_ = [("node", _i32), ("block", _i32), ("A", _vp), ("lda", _i64), ("ready_event", _vp)]


class bicadmm_problem(ct.Structure):
    _fields_ = [("N", _i32), ("M", _i32), ("C", _i32), ("loss", _i32), ("dtype", _i32), ("n_blocks", _i32),
                ("n", _i64), ("m", ct.POINTER(_i64)), ("col_start", ct.POINTER(_i64)),
                ("blocks", ct.POINTER(bicadmm_block)), ("b", ct.POINTER(_vp))]


class bicadmm_params(ct.Structure):
    _fields_ = [("kappa", _i64), ("rho_c", _f64), ("alpha", _f64), ("rho_l", _f64), ("lambda_", _f64),
                ("eps_p", _f64), ("eps_d", _f64), ("eps_b", _f64), ("max_outer", _i32), ("inner_fixed", _i32),
                ("eps_inner", _f64), ("max_inner", _i32), ("refit", _i32), ("sweep", _i32)]


class bicadmm_step_info(ct.Structure):
    _fields_ = [("outer_iters", _i32), ("inner_sweeps", _i32), ("p_r", _f64), ("d_r", _f64), ("b_r", _f64),
                ("t", _f64), ("v", _f64), ("tau", _f64), ("converged", _i32)]


class bicadmm_report(ct.Structure):
    _fields_ = [("converged", _i32), ("outer_iters", _i32), ("inner_sweeps", _i64), ("support_len", _i64),
                ("objective", _f64), ("p_r", _f64), ("d_r", _f64), ("b_r", _f64), ("ms_setup", _f64),
                ("ms_solve", _f64)]


# Every symbol the headers declare (tests check the .so exports all of them).
ABI_SYMBOLS = [
    "bicadmm_version", "bicadmm_rc_string", "bicadmm_uid_size", "bicadmm_get_unique_id", "bicadmm_comm_init",
    "bicadmm_comm_destroy", "bicadmm_emu_group_create", "bicadmm_comm_init_emu", "bicadmm_emu_group_destroy",
    "bicadmm_workspace_size", "bicadmm_setup", "bicadmm_iterate", "bicadmm_solve",
    "bicadmm_finalize", "bicadmm_set_schedule", "bicadmm_get", "bicadmm_last_error", "bicadmm_destroy",
    "bicadmm_set_profiling",
    "bicadmm_op_gemv", "bicadmm_op_gemv_t_ws", "bicadmm_op_gemv_t", "bicadmm_op_prox", "bicadmm_op_block_factor_ws",
    "bicadmm_op_block_factor", "bicadmm_op_gram", "bicadmm_op_gram_tc_ws", "bicadmm_op_gram_tc",
    "bicadmm_op_gemm_tc_ws", "bicadmm_op_gemm_tc", "bicadmm_op_zt", "bicadmm_op_s_update", "bicadmm_op_support",
    "bicadmm_launch_count",
]


class BicadmmError(RuntimeError):
    def __init__(self, rc: int, msg: str = ""):
        self.rc = rc
        super().__init__(f"bicadmm rc={rc} ({_rc_name(rc)}){': ' + msg if msg else ''}")


def _rc_name(rc):
    return {0: "ok", -1: "invalid", -2: "dim", -3: "domain", -4: "placement", -5: "oom", -6: "cuda",
            -7: "nccl", -8: "state"}.get(rc, "?")


_lib = None


def lib() -> ct.CDLL:
    """Load libbicadmm.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("BICADMM_LIB_PATH") or LIB_PATH   # A/B timing of alternative builds only
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with __graft_entry__.build() "
                           "(python -m paper_2405_16267_b200.build); there is no CPU fallback")
    L = ct.CDLL(path)
    P = ct.POINTER
    sig = {
        "bicadmm_version": (ct.c_int, []),
        "bicadmm_rc_string": (ct.c_char_p, [ct.c_int]),
        "bicadmm_uid_size": (ct.c_int, []),
        "bicadmm_get_unique_id": (ct.c_int, [_vp]),
        "bicadmm_comm_init": (ct.c_int, [ct.c_int, ct.c_int, ct.c_int, _vp, ct.c_int, P(_vp)]),
        "bicadmm_comm_destroy": (ct.c_int, [_vp]),
        "bicadmm_emu_group_create": (ct.c_int, [ct.c_int, P(_vp)]),
        "bicadmm_comm_init_emu": (ct.c_int, [_vp, ct.c_int, ct.c_int, ct.c_int, P(_vp)]),
        "bicadmm_emu_group_destroy": (ct.c_int, [_vp]),
        "bicadmm_workspace_size": (ct.c_int, [P(bicadmm_problem), P(bicadmm_params), P(ct.c_size_t)]),
        "bicadmm_setup": (ct.c_int, [P(bicadmm_problem), P(bicadmm_params), _vp, _vp, ct.c_size_t, _vp, P(_vp)]),
        "bicadmm_iterate": (ct.c_int, [_vp, ct.c_int, P(bicadmm_step_info)]),
        "bicadmm_solve": (ct.c_int, [_vp, P(bicadmm_report)]),
        "bicadmm_finalize": (ct.c_int, [_vp, P(bicadmm_report)]),
        "bicadmm_set_schedule": (ct.c_int, [_vp, P(_i32), ct.c_int]),
        "bicadmm_get": (ct.c_int, [_vp, ct.c_int, _vp, ct.c_size_t, ct.c_int, P(ct.c_size_t)]),
        "bicadmm_last_error": (ct.c_char_p, [_vp]),
        "bicadmm_set_profiling": (ct.c_int, [_vp, ct.c_int]),
        "bicadmm_destroy": (ct.c_int, [_vp]),
        "bicadmm_op_gemv": (ct.c_int, [ct.c_int, _i64, _i64, _vp, _i64, _vp, _vp, _vp]),
        "bicadmm_op_gemv_t_ws": (ct.c_size_t, [ct.c_int, _i64, _i64]),
        "bicadmm_op_gemv_t": (ct.c_int, [ct.c_int, _i64, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _f64, _f64, _vp, _vp,
                                         ct.c_size_t, _vp]),
        "bicadmm_op_prox": (ct.c_int, [ct.c_int, ct.c_int, ct.c_int, _i64, ct.c_int, _f64, _vp, _vp, _vp, _vp, _vp, _vp]),
        "bicadmm_op_block_factor_ws": (ct.c_size_t, [_i64]),
        "bicadmm_op_block_factor": (ct.c_int, [ct.c_int, _i64, _i64, _vp, _i64, _f64, _f64, _vp, _i64, _vp,
                                               ct.c_size_t, _vp]),
        "bicadmm_op_gram": (ct.c_int, [ct.c_int, _i64, _i64, _vp, _i64, _f64, _f64, _vp, _i64, _vp]),
        "bicadmm_op_gram_tc_ws": (ct.c_size_t, [ct.c_int, _i64, _i64]),
        "bicadmm_op_gemm_tc_ws": (ct.c_size_t, [_i64, _i64, _i64, ct.c_int]),
        "bicadmm_op_gemm_tc": (ct.c_int, [ct.c_int, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _i64, ct.c_int,
                                          _f64, _f64, _f64, _vp, _i64, ct.c_int, _vp, ct.c_size_t, _vp]),
        "bicadmm_op_gram_tc": (ct.c_int, [ct.c_int, _i64, _i64, _vp, _i64, _f64, _f64, _vp, _i64, _vp, ct.c_size_t, _vp]),
        "bicadmm_op_zt": (ct.c_int, [_i64, ct.c_int, _f64, _f64, _vp, _vp, _f64, _vp, _vp, _vp, P(_f64), _vp]),
        "bicadmm_op_s_update": (ct.c_int, [_i64, _i64, _vp, _f64, _f64, _vp, P(_f64), _vp]),
        "bicadmm_op_support": (ct.c_int, [_i64, _i64, _vp, _vp, P(_i64), _vp]),
        "bicadmm_launch_count": (_i64, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    _lib = L
    return L


def check(rc: int, handle=None) -> None:
    if rc != OK:
        msg = ""
        if handle:
            msg = (lib().bicadmm_last_error(handle) or b"").decode()
        raise BicadmmError(rc, msg)


# ------------------------------------------------------------------------ ABI (same names)
def bicadmm_version():
    return lib().bicadmm_version()


def bicadmm_workspace_size(problem, params) -> int:
    n = ct.c_size_t(0)
    check(lib().bicadmm_workspace_size(ct.byref(problem), ct.byref(params), ct.byref(n)))
    return n.value


def bicadmm_setup(problem, params, comm, workspace_ptr, workspace_bytes, stream_ptr):
    h = _vp()
    check(lib().bicadmm_setup(ct.byref(problem), ct.byref(params), comm, workspace_ptr, workspace_bytes,
                              stream_ptr, ct.byref(h)))
    return h


def bicadmm_iterate(handle, n_outer: int) -> bicadmm_step_info:
    info = bicadmm_step_info()
    check(lib().bicadmm_iterate(handle, n_outer, ct.byref(info)), handle)
    return info


def bicadmm_solve(handle) -> bicadmm_report:
    rep = bicadmm_report()
    check(lib().bicadmm_solve(handle, ct.byref(rep)), handle)
    return rep


def bicadmm_finalize(handle) -> bicadmm_report:
    rep = bicadmm_report()
    check(lib().bicadmm_finalize(handle, ct.byref(rep)), handle)
    return rep


def bicadmm_set_schedule(handle, counts: np.ndarray) -> None:
    counts = np.ascontiguousarray(counts, dtype=np.int32)
    check(lib().bicadmm_set_schedule(handle, counts.ctypes.data_as(ct.POINTER(_i32)), counts.shape[0]), handle)


def bicadmm_get(handle, field: int, dtype=np.float64) -> np.ndarray:
    n = ct.c_size_t(0)
    check(lib().bicadmm_get(handle, field, None, 0, 0, ct.byref(n)), handle)
    out = np.zeros(n.value // np.dtype(dtype).itemsize, dtype=dtype)
    if n.value:
        check(lib().bicadmm_get(handle, field, out.ctypes.data, n.value, 0, None), handle)
    return out


def bicadmm_destroy(handle) -> None:
    if handle:
        lib().bicadmm_destroy(handle)


def bicadmm_get_unique_id() -> bytes:
    L = lib()
    buf = ct.create_string_buffer(L.bicadmm_uid_size())
    check(L.bicadmm_get_unique_id(buf))
    return buf.raw


def bicadmm_comm_init(world: int, rank: int, device: int, uid: bytes | None, group_color: int):
    c = _vp()
    buf = ct.create_string_buffer(uid, len(uid)) if uid else None
    check(lib().bicadmm_comm_init(world, rank, device, buf, group_color, ct.byref(c)))
    return c


def bicadmm_comm_destroy(comm) -> None:
    if comm:
        lib().bicadmm_comm_destroy(comm)


def bicadmm_emu_group_create(world: int):
    g = _vp()
    check(lib().bicadmm_emu_group_create(world, ct.byref(g)))
    return g


def bicadmm_comm_init_emu(group, rank: int, device: int, group_color: int):
    c = _vp()
    check(lib().bicadmm_comm_init_emu(group, rank, device, group_color, ct.byref(c)))
    return c


def bicadmm_emu_group_destroy(group) -> None:
    if group:
        lib().bicadmm_emu_group_destroy(group)


# ------------------------------------------------------------------------ convenience wrapper
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
    refit: int = 0
    sweep: int = 0

    def struct(self) -> bicadmm_params:
        return bicadmm_params(self.kappa, self.rho_c, self.alpha, self.rho_l, 1.0 / self.gamma, self.eps_p,
                              self.eps_d, self.eps_b, self.max_outer, self.inner_fixed, self.eps_inner,
                              self.max_inner, self.refit, self.sweep)


def _stream_ptr(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ct.c_void_p(s.cuda_stream)


def _aligned_matrix(A, torch):
    """Return (tensor, lda) with 16-byte aligned rows (lda % 4 == 0); copies only if needed."""
    m, n = A.shape
    if A.stride(1) == 1 and A.stride(0) % 4 == 0 and A.data_ptr() % 16 == 0:
        return A, A.stride(0)
    lda = -(-n // 4) * 4
    P = torch.zeros(m, lda, dtype=A.dtype, device=A.device)
    P[:, :n] = A
    return P, lda


class BiCADMM:
    """bicadmm_setup(A, b, loss, kappa, rho, lambda) on torch CUDA tensors.

    A: list over nodes of (m_i x n) tensors (all blocks local: single rank), or pass
    ``blocks=[(i, j, A_ij_view)]`` for an explicit placement (multi-rank).
    """

    def __init__(self, A, b, loss, params: Params, col_start, C: int = 1, blocks=None, comm=None,
                 stream=None, dtype=None):
        import torch
        self.torch = torch
        self.loss = LOSSES[loss] if isinstance(loss, str) else int(loss)
        self.params = params
        self.C = C
        self.col_start = np.ascontiguousarray(col_start, dtype=np.int64)
        self.M = len(self.col_start) - 1
        self.N = len(b)
        self.stream = stream
        first = A[0] if A is not None else blocks[0][2]
        self.n = int(self.col_start[-1])
        tdt = dtype or first.dtype
        self.dtype = F64 if tdt == torch.float64 else F32
        self._keep = []
        blk = []
        if blocks is None:
            for i, Ai in enumerate(A):
                Ap, lda = _aligned_matrix(Ai, torch)
                self._keep.append(Ap)
                for j in range(self.M):
                    c0 = int(self.col_start[j])
                    blk.append(bicadmm_block(i, j, Ap.data_ptr() + c0 * Ap.element_size(), lda))
            self.m = np.array([a.shape[0] for a in A], dtype=np.int64)
        else:
            ms = {}
            for ent in blocks:
                # (i, j, A_ij) or (i, j, A_ij, ready): ready a torch.cuda.Event recorded after A_ij
                # and b_i were written (bicadmm_block.ready_event; setup waits on it per block)
                i, j, Aij = ent[:3]
                ev = ent[3] if len(ent) > 3 else None
                assert Aij.stride(1) == 1
                blk.append(bicadmm_block(i, j, Aij.data_ptr(), Aij.stride(0),
                                         ev.cuda_event if ev is not None else None))
                ms[i] = Aij.shape[0]
                self._keep.append(Aij)
            self.m = np.array([ms.get(i, b[i].shape[0] if b[i] is not None else 1) for i in range(self.N)],
                              dtype=np.int64)
        self.blocks = (bicadmm_block * len(blk))(*blk)
        bl = []
        for i in range(self.N):
            if b[i] is None:
                bl.append(None)
                continue
            bi = b[i].contiguous()   # label domain checked by bicadmm_setup (BICADMM_ERR_DOMAIN)
            self._keep.append(bi)
            bl.append(bi.data_ptr())
        self.bptr = (_vp * self.N)(*bl)
        self.problem = bicadmm_problem(self.N, self.M, C, self.loss, self.dtype, len(blk), self.n,
                                       self.m.ctypes.data_as(ct.POINTER(_i64)),
                                       self.col_start.ctypes.data_as(ct.POINTER(_i64)), self.blocks, self.bptr)
        self.pstruct = params.struct()
        self.ws_bytes = bicadmm_workspace_size(self.problem, self.pstruct)
        dev = first.device
        self.workspace = torch.empty(self.ws_bytes + 256, dtype=torch.uint8, device=dev)
        base = self.workspace.data_ptr()
        off = (-base) % 256
        self.handle = bicadmm_setup(self.problem, self.pstruct, comm, ct.c_void_p(base + off),
                                    self.ws_bytes, _stream_ptr(stream))

    # ---- driver
    def iterate(self, n_outer: int = 1) -> bicadmm_step_info:
        return bicadmm_iterate(self.handle, n_outer)

    def solve(self) -> bicadmm_report:
        return bicadmm_solve(self.handle)

    def finalize(self) -> bicadmm_report:
        return bicadmm_finalize(self.handle)

    def set_schedule(self, counts) -> None:
        bicadmm_set_schedule(self.handle, counts)

    def get(self, field: int, dtype=np.float64) -> np.ndarray:
        return bicadmm_get(self.handle, field, dtype)

    @property
    def z(self):
        return self.get(FIELD_Z)

    @property
    def s(self):
        return self.get(FIELD_S)

    def scalars(self) -> dict:
        v = self.get(FIELD_SCALARS)
        return dict(zip(("t", "v", "tau", "p_r", "d_r", "b_r"), v.tolist()))

    def trace(self) -> np.ndarray:
        return self.get(FIELD_TRACE).reshape(-1, 6)

    def support(self) -> np.ndarray:
        return self.get(FIELD_SUPPORT, np.int64)

    def set_profiling(self, on: bool) -> None:
        check(lib().bicadmm_set_profiling(self.handle, 1 if on else 0), self.handle)

    def phases(self) -> dict:
        ms = self.get(FIELD_PHASE_MS)
        cnt = self.get(FIELD_PHASE_COUNT, np.int64)
        return {name: (float(ms[k]), int(cnt[k])) for k, name in enumerate(PHASES)}

    def sweep_kind(self) -> tuple:
        """(inner-sweep implementation: 0 two-pass, 1-4 single-pass kernels; local fat blocks)."""
        k = self.get(FIELD_SWEEP_KIND, np.int32)
        return int(k[0]), int(k[1])

    def launches(self) -> int:
        return int(self.get(FIELD_LAUNCHES, np.int64)[0])

    def close(self) -> None:
        if getattr(self, "handle", None):
            bicadmm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
