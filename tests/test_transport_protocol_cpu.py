"""The cross-rank P2P halo protocol, modelled on CPU with one thread per rank (-m "not gpu").

On one GPU the multi-rank P2P path can only run as virtual slabs whose waits are all
satisfied by earlier launches (B200_PROFILING.md: ranks whose kernels wait on one another
must not share a GPU).  This test runs the protocol's host and device logic concurrently,
one thread per rank with random delays at every step, so that a rank really can be a pass
ahead of, or behind, its neighbours:

- host side, as heat1d.cpp run_passes (transport P2P): at the first pass of every run the
  exchange index skips one (xg += 1) and k_push_edges puts the T-deep edges of the current
  buffer into the neighbours' pads, releasing their flags with xg+1; each pass runs K3p
  with index xg, then xg += 1;
- device side, as kernels.cu k3_edges_put: wait until my flag for each pad is >= g+1,
  read the window (pads included), update the strip, write it to B and put it into the
  neighbour's pad of B, then release the neighbour's flag with g+2; the interior pass
  (K2) reads A only.

Every pad write carries the exchange index it belongs to, and every pad read asserts
that it sees exactly the index it waited for -- an overwrite by a fast neighbour, the
hazard that two pad buffers and the index skips are there to prevent, fails the test.
The result must equal the oracle bitwise after several runs with tail passes.
"""
from __future__ import annotations

import random
import threading
import time

import numpy as np
import pytest

import oracle
import synth


def eq2_block(w, r):
    """One Jacobi step on a window (interior cells only): b + r*((a - 2b) + c)."""
    a, b, c = w[:-2], w[1:-1], w[2:]
    return b + r * ((a - 2.0 * b) + c)


class Rank:
    def __init__(self, g, u, T):
        self.g = g
        self.n = u.size
        self.T = T
        self.buf = [np.zeros(self.n + 2 * T), np.zeros(self.n + 2 * T)]  # [pad T | n cells | pad T]
        self.buf[0][T:T + self.n] = u
        self.tag = [[-1, -1], [-1, -1]]   # [buffer][side] exchange index of the pad contents
        self.flag = [0, 0]                # [side] monotone: pads of index <= flag-1 are in place
        self.cur = 0
        self.xg = 0
        self.lock = threading.Lock()


def jitter(rng):
    if rng.random() < 0.3:
        time.sleep(rng.random() * 2e-4)


def put(dst, b, side, vals, gidx, rng):
    """Remote stores into dst's pad (side 0 = left pad, 1 = right pad) of buffer b, then the release."""
    T = dst.T
    jitter(rng)
    with dst.lock:
        if side == 0:
            dst.buf[b][T - vals.size:T] = vals
        else:
            dst.buf[b][T + dst.n:T + dst.n + vals.size] = vals
        dst.tag[b][side] = gidx
    jitter(rng)
    with dst.lock:
        dst.flag[side] = max(dst.flag[side], gidx + 1)


def wait_flags(me, g, deadline):
    while True:
        with me.lock:
            if me.flag[0] >= g + 1 and me.flag[1] >= g + 1:
                return
        if time.time() > deadline:
            raise AssertionError("rank %d: wait for exchange index %d timed out (deadlock)" % (me.g, g))
        time.sleep(1e-5)


def run_rank(me, ranks, runs, r, seed, errors):
    try:
        for nt in runs:                         # consecutive runs: no barrier between them
            run_once(me, ranks, nt, r, random.Random(seed * 7919 + me.g * 31 + nt))
    except BaseException as e:  # noqa: BLE001
        errors.append(e)


def run_once(me, ranks, nt, r, rng):
    G = len(ranks)
    L, R = ranks[(me.g - 1) % G], ranks[(me.g + 1) % G]
    T, n = me.T, me.n
    jitter(rng)
    done = 0
    while done < nt:
        Tp = min(T, nt - done)
        A, B = me.buf[me.cur], me.buf[me.cur ^ 1]
        if done == 0:                      # run start: skip one index, push full-depth edges
            me.xg += 1
            put(L, me.cur, 1, A[T:2 * T].copy(), me.xg, rng)
            put(R, me.cur, 0, A[n:n + T].copy(), me.xg, rng)
        g = me.xg
        wait_flags(me, g, time.time() + 3)
        with me.lock:                     # K3p reads its window: pads must hold index g
            assert me.tag[me.cur] == [g, g], (me.g, me.cur, me.tag[me.cur], g)
            win_l = A[T - Tp:T + 2 * Tp].copy()
            win_r = A[T + n - 2 * Tp:T + n + Tp].copy()
        jitter(rng)
        for _ in range(Tp):
            win_l = eq2_block(win_l, r)
            win_r = eq2_block(win_r, r)
        # interior (K2): reads A only, outputs [Tp, n-Tp)
        inner = A[T:T + n].copy()
        for _ in range(Tp):
            inner = np.concatenate([[np.nan], eq2_block(inner, r), [np.nan]])
        B[T + Tp:T + n - Tp] = inner[Tp:n - Tp]
        B[T:T + Tp] = win_l
        B[T + n - Tp:T + n] = win_r
        put(L, me.cur ^ 1, 1, win_l.copy(), g + 1, rng)   # my new left strip = L's right pad
        put(R, me.cur ^ 1, 0, win_r.copy(), g + 1, rng)   # my new right strip = R's left pad
        me.xg += 1
        me.cur ^= 1
        done += Tp


def solve(u0, G, T, runs, r, seed):
    N = u0.size
    bounds = np.linspace(0, N, G + 1).astype(int)
    ranks = [Rank(g, u0[bounds[g]:bounds[g + 1]].copy(), T) for g in range(G)]
    errors = []
    th = [threading.Thread(target=run_rank, args=(rk, ranks, runs, r, seed, errors)) for rk in ranks]
    rng = random.Random(seed)
    for t in th:              # ranks start at different times; each then runs all its runs back
        t.start()             # to back, so one may start run k+1 while a neighbour is in run k
        time.sleep(rng.random() * 1e-3)
    for t in th:
        t.join()
    if errors:
        raise errors[0]
    return np.concatenate([rk.buf[rk.cur][T:T + rk.n] for rk in ranks])


@pytest.mark.parametrize("G", [2, 3, 4])
@pytest.mark.parametrize("seed", [0, 1])
def test_p2p_protocol_concurrent_ranks(G, seed):
    T, r = 8, 0.4
    N = G * 53 + 7
    u0 = synth.uniform(100 + G, 0, N, -1.0, 1.0)
    runs = [2 * T + 3, T, 1, 3 * T]
    got = solve(u0, G, T, runs, r, seed)
    assert np.array_equal(got, oracle.run(u0, r, sum(runs)))


def test_protocol_model_detects_a_single_pad_buffer():
    """Sanity of the model: with ONE pad buffer (writes of index g+1 may land while a slow
    neighbour still reads index g) the tag assertion must fire under the same jitter."""
    T, r, G = 4, 0.4, 3
    u0 = synth.uniform(5, 0, G * 40, -1.0, 1.0)
    orig = Rank.__init__

    def one_buffer(self, g, u, TT):
        orig(self, g, u, TT)
        self.buf[1] = self.buf[0]          # both "buffers" share storage
        self.tag[1] = self.tag[0]
    Rank.__init__ = one_buffer
    try:
        caught = False
        for seed in range(8):
            try:
                solve(u0, G, T, [6 * T], r, seed)
            except AssertionError:
                caught = True
                break
        assert caught
    finally:
        Rank.__init__ = orig
