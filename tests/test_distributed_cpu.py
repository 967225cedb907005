"""Multi-rank host logic of the slab decomposition on CPU (gloo, world_size 2 and 3).

What runs here is the library's own host logic -- heat1d_partition (slab of
each rank), heat1d_plan_exchange (the four halo messages, their offsets and
their ISSUE ORDER, which matters when both neighbours are the same rank, G=2)
and heat1d_get_unique_id (the NCCL id that rank 0 broadcasts) -- driven by
real torch.distributed point-to-point messages between processes.  The
per-slab T-step update between exchanges is a test-side numpy stand-in for
the interior/edge kernels (same expression order as Eq. 2 in the oracle).
The result must equal the single-process oracle bitwise (the
segmented algorithm computes the plain sweep).  -m "not gpu".
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nx, np_, T, nt, k, seed, out_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2307_01117_b200 as h1
        import synth
        # NCCL bootstrap plumbing: rank 0's 128-byte id reaches every rank intact
        obj = [h1.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        assert isinstance(obj[0], bytes) and len(obj[0]) == 128
        ids = [None] * world
        dist.all_gather_object(ids, obj[0])
        assert all(i == obj[0] for i in ids)

        first, count = h1.partition(nx, np_, world, rank)
        u0 = synth.uniform(seed, 0, nx * np_, -1.0, 1.0)
        r = float(k)
        P = T
        buf = torch.zeros(count + 2 * P, dtype=torch.float64)
        buf[P:P + count] = torch.from_numpy(u0[first:first + count])
        done = 0
        while done < nt:
            Tp = min(T, nt - done)
            pl = h1.plan_exchange(nx, np_, world, rank, Tp)
            assert pl.cells == Tp and pl.left == (rank - 1) % world and pl.right == (rank + 1) % world

            def view(off):
                return buf[P + off:P + off + Tp]
            # the plan's issue order: send(right edge), send(left edge), recv(left pad), recv(right pad)
            s1 = view(pl.send_right_off).clone()
            s2 = view(pl.send_left_off).clone()
            r1 = torch.empty(Tp, dtype=torch.float64)
            r2 = torch.empty(Tp, dtype=torch.float64)
            reqs = [dist.isend(s1, pl.right), dist.isend(s2, pl.left), dist.irecv(r1, pl.left),
                    dist.irecv(r2, pl.right)]
            for q in reqs:
                q.wait()
            view(pl.recv_left_off).copy_(r1)
            view(pl.recv_right_off).copy_(r2)
            # Tp steps on [-Tp, count+Tp): the light cone shrinks to [0, count)
            w = buf[P - Tp:P + count + Tp].numpy().copy()
            for _ in range(Tp):
                w = w[1:-1] + r * ((w[:-2] - 2.0 * w[1:-1]) + w[2:])
            buf[P:P + count] = torch.from_numpy(w)
            done += Tp
        parts = [None] * world
        dist.all_gather_object(parts, (first, buf[P:P + count].numpy().copy()))
        if rank == 0:
            out_q.put(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nx,np_,T,nt,k", [
    (2, 1000, 8, 8, 37, 0.4),     # G=2: left and right neighbour are the same rank
    (2, 7, 3, 5, 23, 0.5),        # uneven partitions, tail passes
    (3, 500, 4, 4, 30, 0.25),     # np not divisible by G: front-loaded partitions
    (3, 1, 5, 1, 9, 0.4),         # np < ... one-cell partitions, T = 1
])
def test_slab_exchange_plan_gloo(world, nx, np_, T, nt, k):
    import oracle
    import synth
    from paper_2307_01117_b200 import _build
    _build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(rk, world, port, nx, np_, T, nt, k, 31, q)) for rk in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts.sort(key=lambda t: t[0])
    got = np.concatenate([a for _, a in parts])
    u0 = synth.uniform(31, 0, nx * np_, -1.0, 1.0)
    want = oracle.run(u0, k, nt)
    np.testing.assert_array_equal(got, want)


def _worker_light_cone(rank, world, port, N, nt, k, seed, out_q):
    """The host-array multi-rank solve (heat1d_solve_host, nranks > 1): ONE exchange of
    nt-deep halos -- in the same issue order as the library's NCCL group -- then every rank
    finishes on its own (here with the oracle's light-cone window, O3)."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_2307_01117_b200 as h1
        import synth
        first, count = h1.partition(N, 1, world, rank)
        u = torch.from_numpy(synth.uniform(seed, first, count, -1.0, 1.0))
        # the library's own plan at depth nt (heat1d_plan_exchange; heat1d_solve_host issues it)
        pl = h1.plan_exchange(N, 1, world, rank, nt)
        assert pl.cells == nt and pl.recv_left_off == -nt and pl.recv_right_off == count
        s_last = u[pl.send_right_off:pl.send_right_off + nt].clone()
        s_first = u[pl.send_left_off:pl.send_left_off + nt].clone()
        r_left, r_right = torch.empty(nt, dtype=torch.float64), torch.empty(nt, dtype=torch.float64)
        reqs = [dist.isend(s_last, pl.right), dist.isend(s_first, pl.left), dist.irecv(r_left, pl.left),
                dist.irecv(r_right, pl.right)]
        for q in reqs:
            q.wait()
        w0 = np.concatenate([r_left.numpy(), u.numpy(), r_right.numpy()])
        mine = oracle.window(w0, nt, float(k))
        parts = [None] * world
        dist.all_gather_object(parts, (first, mine))
        if rank == 0:
            out_q.put(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N,nt", [(2, 5000, 300), (3, 4099, 200)])
def test_one_deep_halo_exchange_suffices_gloo(world, N, nt):
    """Light cone across ranks: after one exchange of nt-deep halos no rank needs anything
    else for the whole nt-step solve; the reassembled ring equals the oracle bitwise."""
    import oracle
    import synth
    from paper_2307_01117_b200 import _build
    _build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker_light_cone, args=(rk, world, port, N, nt, 0.4, 77, q)) for rk in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts.sort(key=lambda t: t[0])
    got = np.concatenate([a for _, a in parts])
    np.testing.assert_array_equal(got, oracle.run(synth.uniform(77, 0, N, -1.0, 1.0), 0.4, nt))
