"""Multi-GPU plumbing for the triangle count (one process per GPU).

The oriented CSR is replicated on every rank (each rank builds it from the same
deterministic edge list -- no communication).  Rank r counts only the
oriented edges in its degree-weighted range [b[r], b[r+1]) (tc_count with
part_index=r, part_count=P: contiguous source ranges of the (deg,id) DAG with
~equal wedge work), then ONE allreduce (NCCL over NVLink on the GPU box, gloo
in the CPU tests) sums the u64 total and the per-vertex array.

`row_cost` / `partition_bounds` restate, on the host, the device partition
(count.cu RowCost + k_part_bounds) so the split can be checked without a GPU.
"""
from __future__ import annotations

import numpy as np


def degree_rank_dag(offsets: np.ndarray, nbrs: np.ndarray):
    """(deg,id)-oriented DAG in rank space from a symmetric CSR: returns
    (off, col, src) with rows = ranks and N+(r) ascending (graph.cuh layout)."""
    n = offsets.size - 1
    deg = np.diff(offsets).astype(np.int64)
    order = np.lexsort((np.arange(n), deg))          # rank -> id, by (deg, id)
    rank = np.empty(n, np.int64)
    rank[order] = np.arange(n)
    u = np.repeat(np.arange(n, dtype=np.int64), deg)
    v = nbrs.astype(np.int64)
    ru, rv = rank[u], rank[v]
    keep = ru < rv
    src, col = ru[keep], rv[keep]
    idx = np.lexsort((col, src))
    src, col = src[idx], col[idx]
    off = np.zeros(n + 1, np.int64)
    np.add.at(off, src + 1, 1)
    off = np.cumsum(off)
    return off, col, src, order


ITEM_COST = 700  # count.cu kItemCost: per-item overhead in candidate-probe units


def row_cost(off: np.ndarray) -> np.ndarray:
    """Per source row u of the oriented DAG with d = d+(u): C(d,2) candidate
    wedges + ITEM_COST per item (count.cu RowCost)."""
    d = np.diff(off.astype(np.int64))
    return d * np.maximum(d - 1, 0) // 2 + ITEM_COST * d


def partition_bounds(cost: np.ndarray, parts: int, off: np.ndarray) -> np.ndarray:
    """Oriented-edge bounds of a parts-way split: b[0]=0, b[P]=E, b[p] = off[r]
    for the first row r with exclusive-prefix(cost)[r] >= total*p/P
    (count.cu k_part_bounds; the double rounding mirrors the device)."""
    n = cost.size
    E = int(off[-1]) if off.size else 0
    prefix = np.concatenate([[0], np.cumsum(cost)[:-1]]) if n else np.zeros(0, np.int64)
    total = int(cost.sum())
    b = np.zeros(parts + 1, np.int64)
    b[parts] = E
    for p in range(1, parts):
        target = int(float(total) * p / parts)
        r = int(np.searchsorted(prefix, target, side="left"))
        b[p] = int(off[r]) if r < n else E
    return b


def count_part_host(off, col, src, e0: int, e1: int, n: int):
    """Triangles whose low->mid edge lies in [e0, e1) (pivot formulation), with
    per-vertex counts in RANK space -- a slow host check for small graphs."""
    total = 0
    t = np.zeros(n, np.int64)
    for e in range(e0, e1):
        u, v = int(src[e]), int(col[e])
        suffix = col[e + 1: off[u + 1]]
        nv = col[off[v]: off[v + 1]]
        common = np.intersect1d(suffix, nv, assume_unique=True)
        c = common.size
        if c:
            total += c
            t[u] += c
            t[v] += c
            t[common] += 1
    return total, t


def allreduce_counts(total, per_vertex=None, group=None):
    """Sum the per-rank partial counts (torch tensors, int64) in place."""
    import torch.distributed as dist
    dist.all_reduce(total, group=group)
    if per_vertex is not None:
        dist.all_reduce(per_vertex, group=group)


def max_over_ranks(x: float, device=None, group=None) -> float:
    """Device-timed step time: the job's time is the slowest rank's."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
