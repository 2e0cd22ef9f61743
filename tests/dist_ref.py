"""Host restatement of the multi-GPU work split (TEST INFRASTRUCTURE).

The device split (count.cu k_pivot_wedges + PivotCost + k_part_bounds) gives
part p the pivots -- the middle vertices of the (deg,id) order -- with rank in
[b[p], b[p+1]): contiguous rank ranges of ~equal join work.  This restates it
with numpy so the split can be checked on CPU (tests/test_multigpu_gloo.py)
and pinned to the device bounds (test_gpu_parity::test_partition_bounds_match_host).
"""
from __future__ import annotations

import numpy as np

ITEM_COST = 32     # count.cu kItemCost: per in-edge item, in candidate-probe units
SEG_COST = 4       # count.cu kSegRowCost: per member of N+(v), per CTA segment
DENSE_COST = 48    # count.cu TCB_DENSE_COST: one dense-core item (k_join_dense)
COLD_COST = 6      # count.cu TCB_COLD_COST: a cold (hash) probe
WARP_COST = 12      # count.cu TCB_WARP_COST: a warp-bin probe
WARP_MAX_DEG = 64  # graph.cuh kWarpMaxDeg
SMALL_COST = 7     # count.cu TCB_SMALL_COST: multiplier of a small-bin pivot's probes
SLAB_COST = 10      # count.cu TCB_SLAB_COST: a cold probe of a pivot whose table spills to the global slab
SMALL_ITEMS, SMALL_COLD, CTA_SMEM_SLOTS = 32, 256, 1024  # graph.cuh kSmallItems/kSmallCold, count.cu kCtaSmemSlots
CTA_SEG_ITEMS = 512
HOT_BITS = 1 << 16  # graph.cuh kHotBits
CORE_BITS = 2048    # graph.cuh kCoreBits; dense rows have >= core_bits / 32 core members


def core_bits_for(n: int) -> int:
    """build.cu finish_graph's default core size: kCoreBits / 2 for n <= 2^17."""
    return CORE_BITS // 2 if n <= (1 << 17) else CORE_BITS


def dense_core(off: np.ndarray, col: np.ndarray):
    """build.cu finish_graph: core ranks [cb, n) (cb - h0 a multiple of 32)
    and the core members cut out of every dense row (0 for sparse rows)."""
    n = off.size - 1
    h0 = n - HOT_BITS if n > HOT_BITS else 0
    cc = np.zeros(n, np.int64)
    bits = core_bits_for(n)
    if n < bits or n - bits < h0:
        return n, cc
    cb = h0 + ((n - bits - h0 + 31) & ~31)
    src = np.repeat(np.arange(n), np.diff(off))
    c = np.bincount(src[col >= cb], minlength=n).astype(np.int64)
    return cb, np.where(c >= bits // 32, c, 0)


def degree_rank_dag(offsets: np.ndarray, nbrs: np.ndarray):
    """(deg,id)-oriented DAG in rank space from a symmetric CSR: returns
    (off, col, src, order) with rows = ranks and N+(r) ascending (graph.cuh)."""
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


def pivot_cost(off: np.ndarray, col: np.ndarray, src: np.ndarray) -> np.ndarray:
    """Per pivot v (count.cu k_pivot_wedges + PivotCost): the probe cost of
    its in-edges' sparse suffixes (bitmap probes 1, cold hash probes
    COLD_COST, warp-bin probes WARP_COST; a dense row's core members are one
    DENSE_COST item) + ITEM_COST per in-edge + SEG_COST * d+(v) per CTA
    segment; 0 without work."""
    n = off.size - 1
    e = np.arange(col.size, dtype=np.int64)
    _, cc = dense_core(off, col)
    h0 = n - HOT_BITS if n > HOT_BITS else 0
    nhot = np.bincount(src[col >= h0], minlength=n).astype(np.int64)  # hot members per row
    end = off[src + 1]
    a = e + 1
    se = end - cc[src]                               # sparse part ends
    ce = np.minimum(end - nhot[src], se)             # cold part ends
    cold = np.maximum(ce - a, 0)
    hot = np.maximum(se - np.maximum(a, ce), 0)
    dplus = np.diff(off)
    din = np.bincount(col, minlength=n).astype(np.int64)
    pcold = dplus - nhot                             # pivot's members below the hot window
    warp = dplus <= WARP_MAX_DEG                     # graph.cuh PivotClass
    small = ~warp & (din <= SMALL_ITEMS) & (pcold <= SMALL_COLD)
    slab = ~warp & ~small & (2 * pcold > CTA_SMEM_SLOTS)
    v = col
    suffix = np.where(warp[v], WARP_COST * (cold + hot), hot + np.where(slab[v], SLAB_COST, COLD_COST) * cold)
    suffix = np.where(small[v], SMALL_COST * suffix, suffix)
    suffix = suffix + np.where((cc[src] > 0) & (a < end), DENSE_COST, 0)
    jv = np.zeros(n, np.int64)
    np.add.at(jv, col, suffix)
    din = np.bincount(col, minlength=n).astype(np.int64)
    dv = np.diff(off)
    segs = (din + CTA_SEG_ITEMS - 1) // CTA_SEG_ITEMS
    cost = jv + ITEM_COST * din + SEG_COST * dv * segs
    return np.where((dv > 0) & (din > 0), cost, 0)


def partition_bounds(cost: np.ndarray, parts: int, r0: int = 0) -> np.ndarray:
    """Pivot rank bounds: b[0]=0, b[P]=n, b[p] = r0 + first i with
    exclusive-prefix(cost[r0:])[i] >= total*p/P (double rounding as on the
    device); r0 = the number of isolated vertices (the lowest ranks)."""
    n = cost.size
    c = cost[r0:]
    prefix = np.concatenate([[0], np.cumsum(c)[:-1]]) if c.size else np.zeros(0, np.int64)
    total = int(c.sum())
    b = np.zeros(parts + 1, np.int64)
    b[parts] = n
    for p in range(1, parts):
        target = int(float(total) * p / parts)
        b[p] = r0 + int(np.searchsorted(prefix, target, side="left"))
    return b


def isolated(offsets: np.ndarray) -> int:
    return int(np.count_nonzero(np.diff(offsets) == 0))


def count_part_host(off, col, src, v_lo: int, v_hi: int, n: int):
    """Triangles whose middle vertex (pivot) has rank in [v_lo, v_hi), with
    per-vertex counts in RANK space -- a slow host check for small graphs."""
    total = 0
    t = np.zeros(n, np.int64)
    for e in np.nonzero((col >= v_lo) & (col < v_hi))[0]:
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
