"""Placement of (node, feature-block) pairs on ranks.

The paper's hierarchy puts node i's feature blocks A_ij on the GPUs
of node i.  On one NVSwitch box we map it onto a G_n x G_b grid of ranks:
rank (a, b) holds the blocks of node group a that fall in block group b.

* node-major (G_b = 1): a rank owns whole nodes; no per-sweep exchange; the
  outer "Collect" all-reduces sum_i (x_i + u_i) over all ranks.
* block-major (G_n = 1): rank b owns block group b of every node; Algorithm 2's
  per-sweep AllReduce of the m-vector block sums runs over all ranks.
* grid: both; the per-sweep AllReduce runs over the ranks of one node group
  (``group_color`` = a), the per-outer one over all ranks.

Pure host logic: no torch, no CUDA; unit-tested with world_size 2 under gloo.
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass
class RankPlan:
    rank: int
    node_group: int               # group_color for bicadmm_comm_init
    block_group: int
    nodes: list = field(default_factory=list)
    blocks: list = field(default_factory=list)   # [(node, block)]


def _split(n: int, parts: int) -> list:
    """Contiguous split of range(n) into `parts` near-equal ranges (first ones larger)."""
    q, r = divmod(n, parts)
    out, s = [], 0
    for p in range(parts):
        e = s + q + (1 if p < r else 0)
        out.append(list(range(s, e)))
        s = e
    return out


def grid_shape(world: int, N: int, M: int, mode: str = "auto") -> tuple:
    """(G_n, G_b) with G_n * G_b = world."""
    if mode == "node":
        if N < world:
            raise ValueError("node-major placement needs N >= world")
        return world, 1
    if mode == "block":
        if M < world:
            raise ValueError("block-major placement needs M >= world")
        return 1, world
    if mode != "auto":
        raise ValueError(mode)
    # prefer node-major (no per-sweep exchange); fall back to blocks
    for gn in range(world, 0, -1):
        if world % gn == 0 and gn <= N and world // gn <= M:
            return gn, world // gn
    raise ValueError(f"cannot place N={N} nodes x M={M} blocks on {world} ranks")


def plan(world: int, N: int, M: int, mode: str = "auto") -> list:
    gn, gb = grid_shape(world, N, M, mode)
    node_groups, block_groups = _split(N, gn), _split(M, gb)
    plans = []
    for r in range(world):
        a, b = divmod(r, gb)
        p = RankPlan(rank=r, node_group=a, block_group=b, nodes=list(node_groups[a]))
        p.blocks = [(i, j) for i in node_groups[a] for j in block_groups[b]]
        plans.append(p)
    return plans


def check(plans: list, N: int, M: int) -> None:
    """Every (i, j) exactly once; ranks sharing a node share its node group."""
    seen = {}
    for p in plans:
        for ij in p.blocks:
            if ij in seen:
                raise AssertionError(f"block {ij} on ranks {seen[ij]} and {p.rank}")
            seen[ij] = p.rank
    missing = [(i, j) for i in range(N) for j in range(M) if (i, j) not in seen]
    if missing:
        raise AssertionError(f"blocks not placed: {missing[:5]}")
    color = {}
    for p in plans:
        for i in p.nodes:
            if color.setdefault(i, p.node_group) != p.node_group:
                raise AssertionError(f"node {i} spans node groups")
