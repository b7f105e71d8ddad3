"""World-size-2 ``gloo`` tests of the row-sharded multi-GPU data flow (CPU).

The N>1 product path shards users and items with
``alsncg_partition_rows`` (engine.cu partition_rows), runs each half-sweep on
the local rows, replicates them with a ragged all-gather (NCCL broadcast
group, engine.cu allgather_rows) and reduces quartic/loss partials over fixed
64-row tiles in global tile order.  Here gloo stands in for NCCL and the CPU
oracle for the kernels (test infrastructure only): the assembled factors and
tile sums must be bit-identical to the single-process results, and every rank
must compute the same shard bounds.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import socket

import numpy as np
import pytest

WORLD = 2
TILE = 64


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bounds(n_rows, ptr, world):
    from paper_1508_03110_b200 import _lib
    out = np.zeros(world + 1, np.int32)
    ptr = np.ascontiguousarray(ptr, dtype=np.int64)
    _lib.check(_lib.lib().alsncg_partition_rows(n_rows, ptr.ctypes.data, world, TILE, out.ctypes.data))
    return out


def _worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist

        import paper_1508_03110_b200 as P
        from oracle.pyoracle import Oracle, OracleRatings
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        R = P.generate(0)  # BASELINE config 0 (host-side generator)
        O = OracleRatings.from_csr(R.n_users(), R.n_items(), R.uptr, R.uidx, R.uval)
        n_u, n_m, n_f, lam = O.n_u, O.n_m, 10, 0.1
        ub, mb = _bounds(n_u, O.uptr, world), _bounds(n_m, O.iptr, world)
        # every rank computes the same bounds
        got = [torch.zeros(world + 1, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(got, torch.from_numpy(ub.copy()))
        same_u = all(np.array_equal(g.numpy(), ub) for g in got)
        dist.all_gather(got, torch.from_numpy(mb.copy()))
        same_m = all(np.array_equal(g.numpy(), mb) for g in got)
        orc = Oracle("port")
        x0 = orc.random_init(n_f, n_u, n_m, 7)
        # user half-sweep on local rows, ragged all-gather (disjoint rows: a sum is a gather)
        full_u, _ = orc.half_sweep(O, True, n_f, x0[n_f * n_u:], lam)
        mine = np.zeros_like(full_u)
        mine[ub[rank] * n_f: ub[rank + 1] * n_f] = full_u[ub[rank] * n_f: ub[rank + 1] * n_f]
        t = torch.from_numpy(mine.copy())
        dist.all_reduce(t)
        users = t.numpy()
        full_m, _ = orc.half_sweep(O, False, n_f, users, lam)
        mine = np.zeros_like(full_m)
        mine[mb[rank] * n_f: mb[rank + 1] * n_f] = full_m[mb[rank] * n_f: mb[rank + 1] * n_f]
        t = torch.from_numpy(mine.copy())
        dist.all_reduce(t)
        items = t.numpy()
        # squared residuals per 64-user tile, exactly rounded per tile; each
        # rank owns whole tiles, the tile list is concatenated in global order
        um = users.reshape(n_u, n_f)
        im = items.reshape(n_m, n_f)
        n_tiles = (n_u + TILE - 1) // TILE
        tiles = np.zeros(n_tiles)
        for tt in range(ub[rank] // TILE, (ub[rank + 1] + TILE - 1) // TILE):
            vals = []
            for u in range(tt * TILE, min(n_u, (tt + 1) * TILE)):
                for k in range(O.uptr[u], O.uptr[u + 1]):
                    e = O.uval[k] - float(um[u] @ im[O.uidx[k]])
                    vals.append(e * e)
            tiles[tt] = math.fsum(vals)
        tt = torch.from_numpy(tiles.copy())
        dist.all_reduce(tt)
        q.put((rank, same_u, same_m, ub.tolist(), mb.tolist(), users, items, tt.numpy()))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surface worker failures in the parent
        q.put((rank, "error", repr(e)))


def test_sharded_half_sweeps_and_tiles_match_single_process():
    import multiprocessing as mp

    import paper_1508_03110_b200 as P
    from oracle.pyoracle import Oracle, OracleRatings
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[1] != "error", r
    res.sort(key=lambda r: r[0])
    # single-process reference of the same decomposition
    R = P.generate(0)
    O = OracleRatings.from_csr(R.n_users(), R.n_items(), R.uptr, R.uidx, R.uval)
    n_u, n_m, n_f, lam = O.n_u, O.n_m, 10, 0.1
    orc = Oracle("port")
    x0 = orc.random_init(n_f, n_u, n_m, 7)
    users, _ = orc.half_sweep(O, True, n_f, x0[n_f * n_u:], lam)
    items, _ = orc.half_sweep(O, False, n_f, users, lam)
    for rank, same_u, same_m, ub, mb, u_r, m_r, tiles in res:
        assert same_u and same_m
        for b, n, ptr in ((ub, n_u, O.uptr), (mb, n_m, O.iptr)):
            assert b[0] == 0 and b[-1] == n and all(b[i] <= b[i + 1] for i in range(WORLD))
            assert all(v % TILE == 0 for v in b[1:-1])  # tiles never straddle ranks
            shard_nnz = [int(ptr[b[i + 1]] - ptr[b[i]]) for i in range(WORLD)]
            worst_row = int(np.diff(ptr).max())
            assert max(shard_nnz) - min(shard_nnz) <= 2 * TILE * worst_row  # nnz-balanced
        assert np.array_equal(u_r, users) and np.array_equal(m_r, items)
    assert np.array_equal(res[0][7], res[1][7])


def test_partition_rows_edge_cases():
    ptr = np.array([0, 5, 5, 5, 9], np.int64)  # 4 rows, two empty
    b = _bounds(4, ptr, 1)
    assert b.tolist() == [0, 4]
    b = _bounds(4, ptr, 3)  # more ranks than tiles: all rows land in one shard
    assert b[0] == 0 and b[-1] == 4 and sorted(b.tolist()) == b.tolist()
    b = _bounds(0, np.zeros(1, np.int64), 2)
    assert b.tolist() == [0, 0, 0]
    with pytest.raises(ValueError):  # EINVAL maps to std::invalid_argument
        _bounds(4, ptr, 0)
