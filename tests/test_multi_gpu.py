"""Multi-GPU parity: one process per GPU, the library's own NCCL communicator and peer
mappings, bitwise against the oracle.  -m gpu; SKIPS (does not pass) below 2 devices.

Each case spawns min(8, device_count) ranks.  The ranks bootstrap over a gloo group
(rank 0's ncclUniqueId from heat1d_get_unique_id is broadcast with it); everything else --
ncclCommInitRank, the warm-up exchange, the collective K6 vote, the CUDA-IPC mappings of
the P2P transport and of the K6 mailboxes, the exchanges of every pass, the collective
destroy -- is libheat1d's.  Rank 0 reassembles the ring and compares it with the oracle
(the segmented algorithm computes the plain sweep, reading c9).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def _devices():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), NCCL_DEBUG="WARN")
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2307_01117_b200 as h1
        import synth
        nx, np_, nt, k, kw = case["nx"], case["np"], case["nt"], case["k"], case["kw"]
        obj = [h1.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        first, count = h1.partition(nx, np_, world, rank)
        u0 = synth.uniform(case["seed"], first, count, -1.0, 1.0)
        outs = []
        with h1.Heat1D(nx, np_, nt, k, 1.0, 1.0, rank=rank, nranks=world, nccl_id=obj[0], device=rank,
                       **kw) as h:
            info = h.info()
            h.set_initial(u0)
            for step in case.get("runs", [nt]):
                h.run(step)
                outs.append(h.get())
        res = [None] * world
        dist.all_gather_object(res, (first, outs, info["resident"], info["transport"], info["T"]))
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


def _run(case):
    import torch.multiprocessing as mp
    world = min(case.get("world", 8), _devices())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return world, sorted(res, key=lambda t: t[0])


needs2 = pytest.mark.skipif(_devices() < 2, reason="needs >= 2 GPUs (this box has %d)" % _devices())

CASES = {
    # large slabs: K2 passes + depth-T halos every T steps, both transports, a tail pass
    "k2_p2p": dict(nx=1 << 20, np=8, nt=2 * 64 + 5, k=0.5, seed=5, kw=dict(resident=False, transport="p2p")),
    "k2_nccl": dict(nx=1 << 20, np=8, nt=2 * 64 + 5, k=0.4, seed=6, kw=dict(resident=False, transport="nccl")),
    # cumulative runs (a run boundary re-pushes the edges; a tail pass, then deeper passes)
    "k2_runs": dict(nx=1 << 20, np=8, nt=0, k=0.5, seed=7, runs=[70, 1, 64, 130],
                    kw=dict(resident=False, transport="p2p")),
    # on-chip slabs: K6 across ranks, halos through NVLink mailboxes
    "k6": dict(nx=131_072, np=8, nt=1000, k=0.25, seed=8, kw=dict(resident=True)),
    # slabs straddling K6 capacity (one rank fits, another not): the vote picks K2 for all
    # and every rank runs the same T and pad
    "straddle": dict(nx=700_000, np=5, nt=150, k=0.5, seed=9, world=2, kw=dict()),
}


@needs2
@pytest.mark.parametrize("name", sorted(CASES))
def test_multi_gpu_bitwise(name):
    import oracle
    import synth
    case = CASES[name]
    world, res = _run(case)
    N = case["nx"] * case["np"]
    u0 = synth.uniform(case["seed"], 0, N, -1.0, 1.0)
    Ts = {t[4] for t in res}
    assert len(Ts) == 1, "ranks disagree on T: %r" % Ts
    if name == "k6":
        assert all(t[2] == 1 for t in res), "every rank should run K6"
    if name == "straddle":
        assert all(t[2] == 0 for t in res), "the vote must put every rank on K2"
    want = u0
    for i, step in enumerate(case.get("runs", [case["nt"]])):
        want = oracle.run(want, case["k"], step)
        got = np.concatenate([t[1][i] for t in res])
        if not np.array_equal(got, want):
            bad = np.flatnonzero(got != want)
            raise AssertionError("%s (G=%d) run %d: %d cells differ, first %d" % (name, world, i, bad.size, bad[0]))
