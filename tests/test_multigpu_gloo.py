"""CPU: the N>1 path's host logic at world_size 2 over gloo.

Each rank takes its degree-weighted pivot rank range (dist_ref.partition_bounds,
the host restatement of the device split in count.cu) and counts the
triangles whose middle vertex lies in it; one allreduce must give the
oracle's total and per-vertex counts.  The GPU test
(test_gpu_parity::test_partition_bounds_match_host) pins the restatement to
the device's bounds.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _graph():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle_ctypes import Oracle
    o = Oracle()
    pairs = o.gen_rmat(10, 16)
    off, nb, E, _, _ = o.build_graph(pairs, 1 << 10)
    T, pv = o.count(off, nb, per_vertex=True)
    return off, nb, T, pv


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import dist_ref as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    off, nb, T, pv = _graph()
    roff, col, src, order = tdist.degree_rank_dag(off, nb)
    b = tdist.partition_bounds(tdist.pivot_cost(roff, col, src), world)
    tot, t_rank = tdist.count_part_host(roff, col, src, int(b[rank]), int(b[rank + 1]), off.size - 1)
    total = torch.tensor([tot], dtype=torch.int64)
    per_vertex = torch.from_numpy(t_rank[order.argsort()].astype(np.int64))  # rank -> id space
    dist.all_reduce(total)
    dist.all_reduce(per_vertex)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    if rank == 0:
        q.put((int(total.item()), per_vertex.numpy().copy(), t_max, b.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_gloo_partitioned_count(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    total, per_vertex, t_max, bounds = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    off, nb, T, pv = _graph()
    assert total == T
    assert np.array_equal(per_vertex.astype(np.uint64), pv)
    assert t_max == float(world)
    assert bounds[0] == 0 and bounds[-1] == off.size - 1 and bounds == sorted(bounds)


def test_partition_is_balanced_and_covering():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import dist_ref as tdist
    off, nb, T, pv = _graph()
    roff, col, src, order = tdist.degree_rank_dag(off, nb)
    cost = tdist.pivot_cost(roff, col, src)
    n = off.size - 1
    tot = 0
    for P in (1, 2, 3, 4, 8):
        b = tdist.partition_bounds(cost, P)
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0)
        parts = [int(cost[b[p]:b[p + 1]].sum()) for p in range(P)]
        assert sum(parts) == int(cost.sum())
        # each part within one maximal pivot cost of the ideal share
        assert max(parts) - cost.sum() / P <= cost.max() + 1
        # the parts partition the triangles
        tot = sum(tdist.count_part_host(roff, col, src, int(b[p]), int(b[p + 1]), n)[0] for p in range(P))
        assert tot == T
