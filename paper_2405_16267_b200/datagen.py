"""Seeded synthetic inputs shaped like the paper's workloads.

This module holds NO Bi-cADMM arithmetic: it only draws the data of P:268
(dense N(0,1) features with unit-l2-norm columns per node, a kappa-sparse ground
truth, Gaussian noise, labels).  It is the one module shared by the oracle tests
and the CUDA path, so both sides see the same input bits.

Recipe:
  * A_i ~ iid N(0,1), m_i x n, then every column of every A_i scaled to unit l2 norm.
  * x_true: kappa nonzeros at uniformly random positions of the n*C entries,
    values +-U[0.5, 2].
  * e ~ N(0, sigma^2), sigma = 0.01.
  * LS: b = A x_true + e.  Logistic / hinge: b = sign(A x_true + e), 0 -> +1.
    Softmax: y_r = argmax_c (A X_true + E)_{r,c}, X_true n x C.
Generation runs on ``device`` with a seeded ``torch.Generator`` (CPU: mt19937,
CUDA: Philox), node by node.  The same (seed, device) always gives the same bits.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

LOSSES = ("ls", "logistic", "softmax", "hinge")


@dataclass
class SynthProblem:
    A: list            # [N] tensors m_i x n (row-major, contiguous, lda = n)
    b: list            # [N] tensors m_i (LS real, +-1, or class ids as float)
    x_true: torch.Tensor  # n*C (row-major n x C)
    loss: str
    C: int
    kappa: int
    seed: int

    @property
    def N(self) -> int:
        return len(self.A)

    @property
    def n(self) -> int:
        return self.A[0].shape[1]


def block_partition(n: int, M: int, align: int = 4) -> list:
    """Contiguous feature blocks: width ceil(n/M) rounded up to a
    multiple of ``align`` columns so each block starts 16-byte aligned (DESIGN R16);
    the last block takes the remainder."""
    w = -(-n // M)
    w = -(-w // align) * align
    starts = [min(j * w, n) for j in range(M)] + [n]
    if any(starts[j + 1] <= starts[j] for j in range(M)):
        # degenerate tiny n: fall back to the plain ceil(n/M) split
        w = -(-n // M)
        starts = [min(j * w, n) for j in range(M)] + [n]
    return starts


def generate(N: int, m_i, n: int, kappa: int, loss: str = "ls", C: int = 1, seed: int = 0,
             noise_std: float = 0.01, device="cpu", dtype=torch.float64) -> SynthProblem:
    if loss not in LOSSES:
        raise ValueError(f"unknown loss {loss!r}")
    if loss == "softmax" and C < 2:
        raise ValueError("softmax needs C >= 2")
    if loss != "softmax":
        C = 1
    ms = [int(m_i)] * N if isinstance(m_i, int) else [int(v) for v in m_i]
    dev = torch.device(device)
    g = torch.Generator(device=dev)
    g.manual_seed(int(seed))
    # ground truth: kappa nonzeros among n*C entries, values +-U[0.5, 2]
    perm = torch.randperm(n * C, generator=g, device=dev)[:kappa]
    mag = 0.5 + 1.5 * torch.rand(kappa, generator=g, device=dev, dtype=torch.float64)
    sign = torch.where(torch.rand(kappa, generator=g, device=dev) < 0.5, -1.0, 1.0).to(torch.float64)
    x_true = torch.zeros(n * C, device=dev, dtype=torch.float64)
    x_true[perm] = mag * sign
    Xt = x_true.view(n, C)
    A_list, b_list = [], []
    for i in range(N):
        A = torch.randn(ms[i], n, generator=g, device=dev, dtype=torch.float64)
        A.div_(torch.linalg.vector_norm(A, dim=0, keepdim=True).clamp_min(1e-300))
        y = A @ Xt + noise_std * torch.randn(ms[i], C, generator=g, device=dev, dtype=torch.float64)
        if loss == "ls":
            b = y[:, 0].clone()
        elif loss in ("logistic", "hinge"):
            b = torch.where(y[:, 0] >= 0, 1.0, -1.0).to(torch.float64)
        else:
            b = torch.argmax(y, dim=1).to(torch.float64)
        A_list.append(A.to(dtype).contiguous())
        b_list.append(b.to(dtype).contiguous())
        del y
    return SynthProblem(A_list, b_list, x_true, loss, C, int(kappa), int(seed))


def _block_seed(seed: int, i: int, j: int) -> int:
    return (int(seed) * 1_000_003 + 7919 * (i + 1) + 104_729 * (j + 1)) % (2 ** 62)


def generate_blocks(N: int, m_i: int, n: int, kappa: int, loss: str, col_start, blocks, C: int = 1,
                    seed: int = 0, noise_std: float = 0.01, device="cuda", dtype=torch.float64,
                    sum_products=None, row_chunk: int = 65_536):
    """Same recipe as ``generate``, drawn feature block by feature block so that a rank
    holding only some blocks A_ij never materialises a whole node matrix (block-major
    placements: configs[2]-[4] at G > 1, where A is 80-800 GB in total).

    blocks: the local (i, j) pairs.  Every A_ij comes from its own seeded generator
    (independent of the placement), is drawn in row chunks straight into a ``dtype``
    tensor, and has its columns scaled to unit l2 norm (a per-column operation, so the
    block split changes nothing in the recipe).  x_true is drawn from ``seed`` alone
    (identical on every rank).  The labels need the full product A_i x_true =
    sum_j A_ij x_true_j: this function forms the local partial products and calls
    ``sum_products(list of m_i x C FP64 tensors, one per node)`` to sum them over the
    ranks holding the node's other blocks (a torch.distributed all-reduce in bench.py;
    None = all of the node's blocks are local).  Noise is drawn per node from its own
    seed, so every rank forms the same b_i.

    Returns (A: {(i, j): tensor m_i x n_j contiguous}, b: [N] with None for nodes that
    have no local block, x_true)."""
    if loss not in LOSSES:
        raise ValueError(f"unknown loss {loss!r}")
    if loss != "softmax":
        C = 1
    dev = torch.device(device)
    g = torch.Generator(device=dev)
    g.manual_seed(int(seed))
    perm = torch.randperm(n * C, generator=g, device=dev)[:kappa]
    mag = 0.5 + 1.5 * torch.rand(kappa, generator=g, device=dev, dtype=torch.float64)
    sign = torch.where(torch.rand(kappa, generator=g, device=dev) < 0.5, -1.0, 1.0).to(torch.float64)
    x_true = torch.zeros(n * C, device=dev, dtype=torch.float64)
    x_true[perm] = mag * sign
    Xt = x_true.view(n, C)
    nodes = sorted({i for i, _ in blocks})
    prod = {i: torch.zeros(m_i, C, device=dev, dtype=torch.float64) for i in nodes}
    A = {}
    for (i, j) in blocks:
        c0, c1 = int(col_start[j]), int(col_start[j + 1])
        nj = c1 - c0
        gb = torch.Generator(device=dev)
        gb.manual_seed(_block_seed(seed, i, j))
        Aij = torch.empty(m_i, nj, device=dev, dtype=dtype)
        sq = torch.zeros(nj, device=dev, dtype=torch.float64)
        rc = max(1024, min(row_chunk, (1 << 27) // max(nj * C, 1)))   # <= 1 GiB FP64 temporaries
        for r0 in range(0, m_i, rc):
            r1 = min(m_i, r0 + rc)
            ch = torch.randn(r1 - r0, nj, generator=gb, device=dev, dtype=torch.float64)
            sq += (ch * ch).sum(dim=0)
            Aij[r0:r1] = ch.to(dtype)
            del ch
        inv = 1.0 / sq.sqrt().clamp_min(1e-300)
        for r0 in range(0, m_i, rc):
            r1 = min(m_i, r0 + rc)
            ch = Aij[r0:r1].double() * inv
            Aij[r0:r1] = ch.to(dtype)
            prod[i][r0:r1] += ch @ Xt[c0:c1]
            del ch
        A[(i, j)] = Aij
    plist = [prod[i] for i in nodes]
    if sum_products is not None:
        sum_products(plist)
    b = [None] * N
    for k, i in enumerate(nodes):
        gn = torch.Generator(device=dev)
        gn.manual_seed(_block_seed(seed, i, -1))
        y = plist[k] + noise_std * torch.randn(m_i, C, generator=gn, device=dev, dtype=torch.float64)
        if loss == "ls":
            bi = y[:, 0].clone()
        elif loss in ("logistic", "hinge"):
            bi = torch.where(y[:, 0] >= 0, 1.0, -1.0).to(torch.float64)
        else:
            bi = torch.argmax(y, dim=1).to(torch.float64)
        b[i] = bi.to(dtype).contiguous()
    return A, b, x_true


# Named shapes of BASELINE.json configs; "replica" shrinks m
# (and n where the oracle needs it) for oracle-time parity.
CONFIGS = {
    "C1": dict(N=2, M=1, m_i=100, n=50, kappa=5, loss="ls", C=1),
    "C2": dict(N=4, M=1, m_i=25_000, n=10_000, kappa=100, loss="logistic", C=1),
    "C3": dict(N=1, M=8, m_i=1_000_000, n=100_000, kappa=1000, loss="ls", C=1),
    "C4": dict(N=1, M=8, m_i=500_000, n=20_000, kappa=500, loss="softmax", C=10),
    "C5": dict(N=8, M=8, m_i=250_000, n=50_000, kappa=1000, loss="hinge", C=1),
}
