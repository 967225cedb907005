"""Parity of the CUDA path (through the C ABI) with the CPU oracle.  -m gpu.

Matched mode must be BITWISE equal to the oracle (north_star: "bit-exact in
matched-order mode"); fast mode within 1e-12*max|u0|*nt.  Inputs come from
synth/ (seeded), expected values from oracle/ only.
"""
from __future__ import annotations

import math
import os

import numpy as np
import pytest

import oracle
import synth
from synth.configs import C1, C2, C3, C4, C5

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def h1():
    import torch
    from paper_2307_01117_b200 import _build
    _build.build()
    import paper_2307_01117_b200 as m
    torch.cuda.set_device(0)
    return m


def gpu_run(h1, u0, nx, np_, nt, k, dt=1.0, dx=1.0, **kw):
    with h1.Heat1D(nx, np_, nt, k, dt, dx, **kw) as h:
        h.set_initial(u0)
        h.run(nt)
        return h.get()


def assert_bitwise(got, want, what=""):
    if not np.array_equal(got, want):
        bad = np.flatnonzero(got != want)
        raise AssertionError("%s: %d cells differ, first at %d: %r vs %r (max abs diff %g)" % (
            what, bad.size, bad[0], got[bad[0]], want[bad[0]], np.max(np.abs(got - want))))


# ------------------------------------------------------------------ C1
@pytest.mark.parametrize("T", [0, 1, 2, 3, 4, 5, 8, 12, 16, 31, 32, 33, 48, 64, 100, 128])
def test_c1_bitwise_all_T(h1, T):
    r = oracle.r_of(C1.k, C1.dt, C1.dx)
    want = oracle.run(C1.u0(), r, C1.nt)
    got = gpu_run(h1, C1.u0(), C1.nx, C1.np, C1.nt, C1.k, T=T)
    assert_bitwise(got, want, "C1 T=%d" % T)


def test_c1_naive_kernel(h1):
    want = oracle.run(C1.u0(), 0.5, C1.nt)
    assert_bitwise(gpu_run(h1, C1.u0(), C1.nx, C1.np, C1.nt, C1.k, kernel="naive"), want, "C1 naive")


# ------------------------------------------------------------------ degenerate rings
@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6, 7, 8, 13, 31, 33])
@pytest.mark.parametrize("k", [0.25, 0.5, 0.4])
@pytest.mark.parametrize("T", [1, 2, 8])
def test_tiny_rings(h1, N, k, T):
    u0 = synth.uniform(N, 0, N, -1.0, 1.0)
    nt = 17
    want = oracle.run(u0, k, nt)
    assert_bitwise(gpu_run(h1, u0, N, 1, nt, k, T=T), want, "N=%d" % N)


@pytest.mark.parametrize("N", [1, 2, 3, 5, 8, 13, 33, 100])
@pytest.mark.parametrize("k", [0.25, 0.5, 0.4])
def test_tiny_rings_fast_mode(h1, N, k):
    """Fast mode on degenerate rings (N smaller than T, N = 1 and 2) through every kernel choice."""
    u0 = synth.uniform(N + 500, 0, N, -1.0, 1.0)
    nt = 41
    want = oracle.run(u0, k, nt)
    for kw in ({"T": 0}, {"T": 3, "resident": False}, {"kernel": "naive"}):
        got = gpu_run(h1, u0, N, 1, nt, k, mode="fast", **kw)
        assert np.max(np.abs(got - want)) <= fast_bound(u0, nt), (N, k, kw)


def test_fast_mode_cumulative_runs_and_paper_denominator(h1):
    """Fast mode over several run() calls (tail passes, graph replays) and with the
    paper-literal 2h denominator (r = k dt / (2 dx) = 0.45 -> the 2-op scaled form)."""
    N = 500_009
    u0 = synth.uniform(77, 0, N, -1.0, 1.0)
    with h1.Heat1D(N, 1, 0, 0.9, 1.0, 1.0, mode="fast", denominator="paper_2dx", resident=False) as h:
        assert abs(h.info()["r"] - 0.45) < 1e-15
        h.set_initial(u0)
        assert h.info()["dp_ops"] == 2
        for nt in (100, 7, 100, 64):
            h.run(nt)
        got = h.get()
    r = oracle.r_of(0.9, 1.0, 1.0, paper_2h=True)
    assert np.max(np.abs(got - oracle.run(u0, r, 271))) <= fast_bound(u0, 271)


def test_zero_diffusivity_identity(h1):
    u0 = synth.uniform(3, 0, 5000)
    assert_bitwise(gpu_run(h1, u0, 5000, 1, 10, 0.0, T=4), u0, "k=0")


# ------------------------------------------------------------------ ragged, several tiles
@pytest.mark.parametrize("N", [4097, 100_003, (1 << 20) + 7])
@pytest.mark.parametrize("T", [1, 3, 8, 12])
@pytest.mark.parametrize("k", [0.4, 0.5])
@pytest.mark.parametrize("resident", [False, None])
def test_ragged_multi_tile(h1, N, T, k, resident):
    """K2 passes (resident=False) and the auto choice (K6 for these on-chip rings)."""
    nt = 2 * T + 3           # full passes + a tail pass
    u0 = synth.uniform(N + T, 0, N, -1.0, 1.0)
    want = oracle.run(u0, k, nt)
    assert_bitwise(gpu_run(h1, u0, N, 1, nt, k, T=T, resident=resident), want, "N=%d T=%d" % (N, T))


@pytest.mark.parametrize("N", [1, 2, 7, 33, 544, 545, 5000, 80_000, 1_000_000, 1_400_000])
@pytest.mark.parametrize("T", [1, 5, 16, 32, 33, 64, 96, 128])
def test_resident_kernel(h1, N, T):
    """K6 (whole solve in one cooperative launch, slab in registers) vs the oracle:
    one warp, a few warps, one warp per SM, many warps per SM, near capacity."""
    nt = 3 * T + 2
    u0 = synth.uniform(N + 7 * T, 0, N, -1.0, 1.0)
    want = oracle.run(u0, 0.4, nt)
    with h1.Heat1D(N, 1, nt, 0.4, 1.0, 1.0, T=T, resident=True) as h:
        assert h.info()["resident"] == 1
        h.set_initial(u0)
        h.run(nt)
        got = h.get()
        h.run(1)                          # a second run continues from the state
        assert_bitwise(h.get(), oracle.run(want, 0.4, 1), "K6 N=%d continue" % N)
    assert_bitwise(got, want, "K6 N=%d T=%d" % (N, T))


@pytest.mark.parametrize("N,T", [(40, 8), (545, 16), (100_003, 32), (1 << 20, 64), (1_000_000, 64),
                                 (1 << 20, 128)])
def test_resident_mailbox_loopback(h1, monkeypatch, N, T):
    """K6 with the multi-rank mailbox protocol (remote-store halos + system-scope flags,
    initial-state exchange, global exchange indices across runs) on one rank whose ring
    wrap is routed through its own mailbox (HEAT1D_K6_MAILBOX=1): bitwise = oracle over
    several consecutive runs, incl. tail periods; fast mode within the bound."""
    monkeypatch.setenv("HEAT1D_K6_MAILBOX", "1")
    u0 = synth.uniform(N + T, 0, N, -1.0, 1.0)
    with h1.Heat1D(N, 1, 0, 0.4, 1.0, 1.0, T=T, resident=True) as h:
        assert h.info()["resident"] == 1
        h.set_initial(u0)
        want = u0
        for nt in (3 * T + 2, T, 1, 2 * T):
            h.run(nt)
            want = oracle.run(want, 0.4, nt)
            assert_bitwise(h.get(), want, "mailbox N=%d T=%d after +%d" % (N, T, nt))
    nt = 2 * T + 3
    with h1.Heat1D(N, 1, nt, 0.5, 1.0, 1.0, T=T, resident=True, mode="fast") as h:
        h.set_initial(u0)
        h.run()
        assert np.max(np.abs(h.get() - oracle.run(u0, 0.5, nt))) <= fast_bound(u0, nt)


def test_resident_refuses_too_large(h1):
    with pytest.raises(h1.Heat1DError) as ei:
        h1.Heat1D(1 << 24, 1, 10, 0.5, 1.0, 1.0, resident=True)
    assert ei.value.status == 7


GEOMS = ["17,4,3,4,3", "25,4,3,2,3", "33,4,2,2,3", "33,4,2,2,4",
         "49,4,2,2,3", "49,4,2,2,4", "51,4,2,2,3", "51,4,2,2,4"]


def _geom_run(h1, geom, u0, N, nt, k, T, mode="matched"):
    with h1.Heat1D(N, 1, nt, k, 1.0, 1.0, T=T, resident=False, mode=mode) as h:
        inf = h.info()
        assert "%d,%d,%d" % (inf["pass_V"], inf["pass_NW"], inf["pass_S"]) == ",".join(geom.split(",")[:3])
        assert inf["pass_kind"] == int(geom.split(",")[4])
        h.set_initial(u0)
        h.run()
        return h.get()


@pytest.mark.parametrize("geom", GEOMS)
def test_all_pass_geometries(h1, geom, monkeypatch):
    """Every instantiated pass-kernel geometry (HEAT1D_GEOM test hook, read at create)."""
    monkeypatch.setenv("HEAT1D_GEOM", geom)
    N, nt = 300_001, 29
    u0 = synth.uniform(77, 0, N, -1.0, 1.0)
    for k, T in [(0.4, 7), (0.5, 12)]:
        want = oracle.run(u0, k, nt)
        assert_bitwise(_geom_run(h1, geom, u0, N, nt, k, T), want, "geom %s T=%d" % (geom, T))


@pytest.mark.parametrize("geom", ["17,4,3,4,3", "33,4,2,2,3", "49,4,2,2,3", "33,4,2,2,4", "51,4,2,2,4"])
@pytest.mark.parametrize("T", [1, 2, 7, 8, 9, 16, 17, 32, 64, 96, 128])
def test_interwarp_exchange_kernel(h1, geom, T, monkeypatch):
    """Pass kinds 3/4 (ghost exchange between the warps of a CTA every 8/16 steps): T below,
    at and between multiples of the exchange depth, matched 4-op / 3-op and both fast
    variants, incl. tail passes and ragged tiles."""
    monkeypatch.setenv("HEAT1D_GEOM", geom)
    V = int(geom.split(",")[0])
    kx = 8 if geom.endswith(",3") else 16
    if T > 32 * V - kx:
        pytest.skip("T exceeds the geometry's span")
    N = 200_003
    nt = 2 * T + 3
    u0 = synth.uniform(1000 + T, 0, N, -1.0, 1.0)
    for k in (0.4, 0.5):
        want = oracle.run(u0, k, nt)
        assert_bitwise(_geom_run(h1, geom, u0, N, nt, k, T), want, "kind %s T=%d k=%g" % (geom, T, k))
        got = _geom_run(h1, geom, u0, N, nt, k, T, mode="fast")
        assert np.max(np.abs(got - want)) <= fast_bound(u0, nt)


# ------------------------------------------------------------------ C2 (paper's workload size)
def test_c2_bitwise_and_conservation(h1):
    r = oracle.r_of(C2.k, C2.dt, C2.dx)
    u0 = C2.u0()
    want = oracle.run(u0, r, C2.nt)
    got = gpu_run(h1, u0, C2.nx, C2.np, C2.nt, C2.k)
    assert_bitwise(got, want, "C2")
    assert abs(math.fsum(got) - math.fsum(u0)) <= 1e-9 * math.fsum(np.abs(u0))


def test_c2_nx_np_invariance(h1):
    """(nx, np) only changes the partitioning: identical bits for every split
    (single slab, and as virtual slabs = partitions grouped per 'GPU')."""
    u0 = C2.u0()
    ref = gpu_run(h1, u0, C2.nx, C2.np, C2.nt, C2.k)
    for nx, np_, vs in [(1_000_000, 1, 1), (1000, 1000, 1), (250, 4000, 1), (10_000, 100, 4), (1000, 1000, 8),
                        (250, 4000, 3)]:
        assert_bitwise(gpu_run(h1, u0, nx, np_, C2.nt, C2.k, virtual_slabs=vs), ref, "nx=%d np=%d vs=%d" % (nx, np_, vs))


# ------------------------------------------------------------------ invariances of the GPU path
def test_cross_T_bitwise(h1):
    N, nt = 1 << 20, 96
    u0 = synth.uniform(5, 0, N, -1.0, 1.0)
    ref = gpu_run(h1, u0, N, 1, nt, 0.4, kernel="naive")
    for T in [1, 2, 3, 4, 6, 8, 11, 12, 16, 24, 32]:
        for res in (False, True):
            assert_bitwise(gpu_run(h1, u0, N, 1, nt, 0.4, T=T, resident=res), ref, "T=%d res=%s" % (T, res))
    for T in [33, 40, 48, 63, 64, 96, 128]:
        assert_bitwise(gpu_run(h1, u0, N, 1, nt, 0.4, T=T, resident=False), ref, "T=%d" % T)


def test_split_run_invariance(h1):
    N = 200_000
    u0 = synth.uniform(9, 0, N, -1.0, 1.0)
    with h1.Heat1D(N, 1, 0, 0.4, 1.0, 1.0, T=8) as h:
        h.set_initial(u0)
        h.run(13)
        h.run(0)
        h.run(29)
        assert h.steps_done == 42
        got = h.get()
    assert_bitwise(got, oracle.run(u0, 0.4, 42), "split")


@pytest.mark.parametrize("vs", [1, 4])
def test_graph_replay(h1, vs):
    """run(nt) is captured once as a CUDA graph and replayed: repeated runs, both
    starting buffers, and a fresh initial state must all stay exact."""
    N, T = 300_007, 8
    u0 = synth.uniform(55, 0, N, -1.0, 1.0)
    with h1.Heat1D(N, 1, 0, 0.4, 1.0, 1.0, T=T, virtual_slabs=vs, resident=False) as h:
        h.set_initial(u0)
        for _ in range(3):
            h.run(20)          # 3 passes: odd -> the next replay starts from the other buffer
        h.run(7)
        assert_bitwise(h.get(), oracle.run(u0, 0.4, 67), "graph replay vs=%d" % vs)
        h.set_initial(u0)
        h.run(20)
        assert_bitwise(h.get(), oracle.run(u0, 0.4, 20), "graph replay after set_initial")
        assert h.info()["launches"] > 0
    with h1.Heat1D(N, 1, 0, 0.4, 1.0, 1.0, T=T, virtual_slabs=vs, resident=False, use_graphs=False) as h:
        h.set_initial(u0)
        h.run(20)
        assert_bitwise(h.get(), oracle.run(u0, 0.4, 20), "no graphs")


@pytest.mark.parametrize("G", [2, 3, 4, 8])
@pytest.mark.parametrize("T", [1, 4, 8, 12, 32, 64])
@pytest.mark.parametrize("transport", ["nccl", "p2p"])
def test_virtual_slabs_multi_gpu_schedule(h1, G, T, transport):
    """The multi-GPU schedule with G slabs on one GPU: exchange || interior, then edges,
    with the transport replaced by device copies ("nccl"), or the fused K3p that puts its
    new strips into the neighbour slabs' pads and releases their exchange-index words
    ("p2p": the same kernels and protocol as across ranks, peers = other slabs)."""
    nx, np_ = 12_289, 8
    nt = 3 * T + 1
    u0 = synth.uniform(G * 100 + T, 0, nx * np_, -1.0, 1.0)
    want = oracle.run(u0, 0.4, nt)
    assert_bitwise(gpu_run(h1, u0, nx, np_, nt, 0.4, T=T, virtual_slabs=G, transport=transport), want,
                   "G=%d T=%d %s" % (G, T, transport))


@pytest.mark.parametrize("G", [2, 5])
def test_p2p_transport_runs_and_modes(h1, G):
    """Transport p2p over consecutive runs (run-boundary re-push after a shallow tail pass,
    exchange indices that keep growing), a new initial state, and fast mode."""
    nx, np_, T = 20_011, 4, 16
    u0 = synth.uniform(G + 3, 0, nx * np_, -1.0, 1.0)
    with h1.Heat1D(nx, np_, 0, 0.4, 1.0, 1.0, T=T, virtual_slabs=G, transport="p2p") as h:
        h.set_initial(u0)
        want = u0
        for nt in (2 * T + 5, T, 3, 1, 2 * T):
            h.run(nt)
            want = oracle.run(want, 0.4, nt)
            assert_bitwise(h.get(), want, "p2p G=%d +%d" % (G, nt))
        h.set_initial(u0)
        h.run(T + 1)
        assert_bitwise(h.get(), oracle.run(u0, 0.4, T + 1), "p2p after set_initial")
    with h1.Heat1D(nx, np_, 0, 0.5, 1.0, 1.0, T=T, virtual_slabs=G, transport="p2p", mode="fast") as h:
        h.set_initial(u0)
        h.run(77)
        assert np.max(np.abs(h.get() - oracle.run(u0, 0.5, 77))) <= fast_bound(u0, 77)


def test_virtual_slabs_small_slabs(h1):
    # slabs of 5 cells with T clamped to the slab size
    u0 = synth.uniform(1, 0, 20)
    want = oracle.run(u0, 0.5, 40)
    assert_bitwise(gpu_run(h1, u0, 5, 4, 40, 0.5, T=8, virtual_slabs=4), want, "tiny slabs")


# ------------------------------------------------------------------ fast mode bound
def test_fast_mode_within_bound(h1):
    N, nt = 1_000_000, 1000
    u0 = synth.uniform(42, 0, N, -1.0, 1.0)
    want = oracle.run(u0, 0.4, nt)
    got = gpu_run(h1, u0, N, 1, nt, 0.4, mode="fast")
    err = np.max(np.abs(got - want))
    assert err <= 1e-12 * np.max(np.abs(u0)) * nt, err


def fast_bound(u0, nt):
    """north_star: max|u_gpu - u_oracle| <= 1e-12 * max|u| * nt (max|u| = max|u0|, reading c16)."""
    return 1e-12 * float(np.max(np.abs(u0))) * nt


# (k, expected dp_ops): r = 1/2 -> one add per update; 1/256 <= r < 1/2 -> add + fma on the
# scaled state; tiny r and unstable r > 1/2 -> the contracted 3-op form
FAST_CASES = [(0.5, 1), (0.25, 2), (0.4, 2), (0.01, 2), (1.0 / 256, 2), (0.001, 3)]


@pytest.mark.parametrize("k,ops", FAST_CASES)
@pytest.mark.parametrize("T", [1, 7, 32, 64])
@pytest.mark.parametrize("path", ["k2", "k6", "slabs3"])
def test_fast_mode_variants(h1, k, ops, T, path):
    """Fast mode (scaled state, DESIGN.md c21) on every kernel family: K2 passes, K6 whole
    solve, and the multi-slab schedule (K2 interior + K3 edges + exchange), incl. a tail pass."""
    N = 300_001 if path != "k6" else 100_003
    nt = 2 * T + 5
    u0 = synth.uniform(int(k * 1000) + T, 0, N, -1.0, 1.0)
    want = oracle.run(u0, k, nt)
    kw = {"resident": False} if path == "k2" else {"resident": True} if path == "k6" else {"virtual_slabs": 3}
    with h1.Heat1D(N, 1, nt, k, 1.0, 1.0, T=T, mode="fast", **kw) as h:
        h.set_initial(u0)
        assert h.info()["dp_ops"] == ops
        h.run(nt)
        got = h.get()
    err = float(np.max(np.abs(got - want)))
    assert err <= fast_bound(u0, nt), (k, T, path, err)


def test_fast_mode_r_half_is_exact_average(h1):
    """At r = 1/2 the scaled form is exactly u' = fl(u_{i-1} + u_{i+1}) / 2 per step (the
    2^-T rescale is exact): check that sequence bitwise (numpy, no oracle arithmetic involved)."""
    N, nt = 4099, 70
    u0 = synth.uniform(3, 0, N, -1.0, 1.0)
    want = u0.copy()
    for _ in range(nt):
        want = (np.roll(want, 1) + np.roll(want, -1)) * 0.5
    for kw in ({"resident": False, "T": 32}, {"resident": True, "T": 32}, {"virtual_slabs": 2, "T": 9}):
        with h1.Heat1D(N, 1, nt, 0.5, 1.0, 1.0, mode="fast", **kw) as h:
            h.set_initial(u0)
            h.run(nt)
            assert_bitwise(h.get(), want, "r=1/2 fast %r" % kw)


def test_fast_mode_range_fallback(h1):
    """Values near the top of the fp64 range would overflow the scaled state (|u0| r^-T): the
    scaled kernels read K5's max|u0| word on the device and run the 3-op form instead, per
    initial state -- K2 (+ K3/K3p edge strips with several slabs) and K6."""
    N, nt = 50_000, 40
    u0 = synth.uniform(6, 0, N, -1.0, 1.0)
    big = u0 * 1e300
    for kw in (dict(resident=False), dict(resident=True), dict(resident=False, virtual_slabs=2),
               dict(resident=False, virtual_slabs=2, transport="nccl")):
        with h1.Heat1D(N, 1, nt, 0.25, 1.0, 1.0, T=32, mode="fast", **kw) as h:
            assert h.info()["dp_ops"] == 2
            h.set_initial(big)
            h.run(nt)
            got = h.get()
            assert np.all(np.isfinite(got)), kw
            assert np.max(np.abs(got - oracle.run(big, 0.25, nt))) <= fast_bound(big, nt), kw
            h.set_initial(u0)                       # back in range: the scaled variant again
            h.run(nt)
            assert np.max(np.abs(h.get() - oracle.run(u0, 0.25, nt))) <= fast_bound(u0, nt), kw


def test_fast_mode_c4_first_100_steps(h1):
    """C4 at full size in fast mode (1 fp64 add per update): O3 windows at every slab
    boundary, the wrap and random cells within the north_star bound."""
    import torch
    N, nt = C4.N, 100
    r = oracle.r_of(C4.k, C4.dt, C4.dx)
    out = torch.empty(N, dtype=torch.float64, device="cuda")
    with h1.Heat1D(C4.nx, C4.np, nt, C4.k, C4.dt, C4.dx, mode="fast") as h:
        h.init_uniform(C4.seed, C4.lo, C4.hi)
        assert h.info()["dp_ops"] == 1
        h.run()
        h.get(out)
    rng = np.random.default_rng(2)
    for a in [g * C4.nx - 256 for g in range(8)] + list(rng.integers(0, N - 600, 8)):
        idx = (np.arange(a, a + 512) % N).astype(np.int64)
        got = out[torch.from_numpy(idx).cuda()].cpu().numpy()
        w = oracle.window(C4.u0(a - nt, 512 + 2 * nt), nt, r)
        assert np.max(np.abs(got - w)) <= 1e-12 * 1.0 * nt, a


def test_fast_mode_c3_closed_form(h1):
    """C3 at full size in fast mode (2 DP ops per update): the 8-mode closed form on a
    strided sample, and O3 windows within the bound."""
    import torch
    N, nt = C3.N, C3.nt
    r = oracle.r_of(C3.k, C3.dt, C3.dx)
    u0 = C3.u0()
    out = torch.empty(N, dtype=torch.float64, device="cuda")
    with h1.Heat1D(C3.nx, C3.np, nt, C3.k, C3.dt, C3.dx, mode="fast") as h:
        h.set_initial(u0)
        assert h.info()["dp_ops"] == 2
        h.run()
        h.get(out)
    got = out.cpu().numpy()
    bound = fast_bound(u0, nt)
    for a in [0, N - 64, C3.nx - 100, 12345677]:
        w = oracle.window(C3.u0(a - nt, 512 + 2 * nt), nt, r)
        assert np.max(np.abs(got[np.arange(a, a + 512) % N] - w)) <= bound, a
    sel = np.arange(0, N, 101, dtype=np.int64)
    want = np.zeros(sel.size)
    for m, amp in zip(C3.modes, C3.amps()):
        s_ = math.sin(math.pi * m / N)
        want += amp * math.exp(nt * math.log1p(-4.0 * r * s_ * s_)) * np.sin(2.0 * np.pi * ((m * sel) % N) / N)
    assert np.max(np.abs(got[sel] - want)) <= 1e-12 + bound


def test_paper_2h_denominator(h1):
    # literal Eq. 2: r = k*dt/(2 dx); k=0.8, dx=1 -> r = 0.4
    u0 = synth.uniform(2, 0, 5000)
    want = oracle.run(u0, oracle.r_of(0.8, 1.0, 1.0, paper_2h=True), 50)
    assert_bitwise(gpu_run(h1, u0, 5000, 1, 50, 0.8, denominator="paper_2dx"), want, "2h")


# ------------------------------------------------------------------ boundary semantics
def test_init_uniform_matches_synth(h1):
    N = 1_000_003
    with h1.Heat1D(N, 1, 0, 0.5, 1.0, 1.0) as h:
        h.init_uniform(1234, -1.0, 1.0)
        got = h.get()
    assert_bitwise(got, synth.uniform(1234, 0, N, -1.0, 1.0), "K0")
    with h1.Heat1D(1000, 8, 0, 0.5, 1.0, 1.0, virtual_slabs=8) as h:
        h.init_uniform(42)
        assert_bitwise(h.get(), synth.uniform(42, 0, 8000), "K0 slabs")


def test_state_errors_and_ownership(h1):
    import torch
    with h1.Heat1D(1000, 1, 5, 0.5, 1.0, 1.0) as h:
        with pytest.raises(h1.Heat1DError) as ei:
            h.run()
        assert ei.value.status == 3                       # ESTATE
        with pytest.raises(h1.Heat1DError):
            h.get()
        u0 = synth.uniform(4, 0, 1000)
        buf = u0.copy()
        h.set_initial(buf)
        buf[:] = np.nan                                   # copy made: caller may reuse
        assert_bitwise(h.get(), u0, "get before run")
        h.run(0)
        assert h.steps_done == 0
        with pytest.raises(h1.Heat1DError) as ei:
            h.set_initial(u0[:10])
        assert ei.value.status == 1
        # device pointers in and out
        d = torch.from_numpy(u0).cuda()
        h.set_initial(d)
        h.run()
        out = torch.empty(1000, dtype=torch.float64, device="cuda")
        h.get(out)
        assert_bitwise(out.cpu().numpy(), oracle.run(u0, 0.5, 5), "device ptrs")
        info = h.info()
        assert info["steps_done"] == 5 and info["N"] == 1000 and info["dp_ops"] == 3


def test_unstable_allowed(h1):
    u0 = synth.uniform(8, 0, 256)
    want = oracle.run(u0, 0.6, 5)
    assert_bitwise(gpu_run(h1, u0, 256, 1, 5, 0.6, allow_unstable=True, T=2), want, "r=0.6")


# ------------------------------------------------------------------ full-size configs
def test_c5_full_bitwise_and_closed_form(h1):
    """C5 in full (2^20 cells, 20000 steps, r=1/4) vs O1 bitwise, plus the
    closed-form decay of the single mode m=5 (BASELINE.json configs[4])."""
    u0 = C5.u0()
    r = oracle.r_of(C5.k, C5.dt, C5.dx)
    got = gpu_run(h1, u0, C5.nx, C5.np, C5.nt, C5.k)
    s = math.sin(math.pi * 5 / C5.N)
    g_t = math.exp(C5.nt * math.log1p(-4.0 * r * s * s))
    assert np.max(np.abs(got - g_t * u0)) <= 1e-12
    assert_bitwise(got, oracle.run(u0, r, C5.nt), "C5")
    got8 = gpu_run(h1, u0, C5.nx, C5.np, C5.nt, C5.k, virtual_slabs=8)
    assert_bitwise(got8, got, "C5 8 virtual slabs")


def test_c3_full_windows_and_closed_form(h1):
    """C3 at full size (2^28 cells, nt=1000, r=0.4): O3 windows bitwise at
    tile/partition edges and the wrap, and the 8-mode closed form on a
    strided sample of every cell class (BASELINE.json configs[2])."""
    import torch
    N, nt = C3.N, C3.nt
    r = oracle.r_of(C3.k, C3.dt, C3.dx)
    u0 = C3.u0()
    out = torch.empty(N, dtype=torch.float64, device="cuda")
    with h1.Heat1D(C3.nx, C3.np, nt, C3.k, C3.dt, C3.dx) as h:
        h.set_initial(u0)
        tile = h.info()["tile_cells"]
        h.run()
        h.get(out)
    got = out.cpu().numpy()
    rng = np.random.default_rng(0)
    starts = [0, N - 64, C3.nx - 100, 5 * C3.nx - 3, tile - 50, 7 * tile - 1] + list(rng.integers(0, N - 600, 10))
    for a in starts:
        b = a + 512
        w = oracle.window(C3.u0(a - nt, b - a + 2 * nt), nt, r)
        idx = np.arange(a, b) % N
        assert_bitwise(got[idx], w, "C3 window %d" % a)
    # closed form on every 97th cell
    sel = np.arange(0, N, 97, dtype=np.int64)
    want = np.zeros(sel.size)
    for m, a in zip(C3.modes, C3.amps()):
        s = math.sin(math.pi * m / N)
        gt = math.exp(nt * math.log1p(-4.0 * r * s * s))
        want += a * gt * np.sin(2.0 * np.pi * ((m * sel) % N) / N)
    assert np.max(np.abs(got[sel] - want)) <= 1e-12


def test_c4_first_100_steps_windows(h1):
    """C4 (2^31 cells, 16 GiB) on one GPU: the first 100 steps checked with O3
    windows at all 8 slab boundaries, the wrap and random cells, both as one
    slab and as 8 virtual slabs (the 8-GPU decomposition); the two agree
    bitwise everywhere (BASELINE.json configs[3])."""
    import torch
    N, nt = C4.N, 100
    r = oracle.r_of(C4.k, C4.dt, C4.dx)
    out = torch.empty(N, dtype=torch.float64, device="cuda")
    with h1.Heat1D(C4.nx, C4.np, nt, C4.k, C4.dt, C4.dx) as h:
        h.init_uniform(C4.seed, C4.lo, C4.hi)
        h.run()
        h.get(out)
    rng = np.random.default_rng(1)
    starts = [g * C4.nx - 256 for g in range(8)] + list(rng.integers(0, N - 600, 8))
    got = {}
    for a in starts:
        idx = (np.arange(a, a + 512) % N).astype(np.int64)
        got[a] = out[torch.from_numpy(idx).cuda()].cpu().numpy()
        w = oracle.window(C4.u0(a - nt, 512 + 2 * nt), nt, r)
        assert_bitwise(got[a], w, "C4 window %d" % a)
    for transport in ("nccl", "p2p"):
        with h1.Heat1D(C4.nx, C4.np, nt, C4.k, C4.dt, C4.dx, virtual_slabs=8, transport=transport) as h:
            h.init_uniform(C4.seed, C4.lo, C4.hi)
            h.run()
            out2 = torch.empty(N, dtype=torch.float64, device="cuda")
            h.get(out2)
        assert torch.equal(out, out2), transport
        del out2


@pytest.mark.parametrize("mode", ["matched", "fast"])
def test_c4_full_nt_windows(h1, mode):
    """C4 exactly as bench.py times it (2^31 cells, all 10,000 steps, default T and kernels):
    O3 light-cone windows of the FINAL field at slab boundaries, the wrap and random cells --
    bitwise (matched) or within the north_star bound (fast)."""
    import torch
    N, nt = C4.N, C4.nt
    r = oracle.r_of(C4.k, C4.dt, C4.dx)
    out = torch.empty(N, dtype=torch.float64, device="cuda")
    with h1.Heat1D(C4.nx, C4.np, nt, C4.k, C4.dt, C4.dx, mode=mode) as h:
        h.init_uniform(C4.seed, C4.lo, C4.hi)
        h.run()
        h.get(out)
    rng = np.random.default_rng(3)
    W = 256
    for a in [0, N - W // 2, 3 * C4.nx - W // 2] + list(rng.integers(0, N - W, 3)):
        idx = (np.arange(a, a + W) % N).astype(np.int64)
        got = out[torch.from_numpy(idx).cuda()].cpu().numpy()
        w = oracle.window(C4.u0(a - nt, W + 2 * nt), nt, r)
        if mode == "matched":
            assert_bitwise(got, w, "C4 nt=10000 window %d" % a)
        else:
            assert np.max(np.abs(got - w)) <= 1e-12 * 1.0 * nt, a


# ------------------------------------------------------------------ heat1d_solve_host (light-cone windows)
@pytest.mark.parametrize("N,nt,T", [(300_001, 100, 0), (300_001, 77, 13), ((1 << 22) + 5, 300, 64)])
def test_solve_host_windows_bitwise(h1, N, nt, T):
    """The streamed solve (C windows of chunk + nt halo cells, transfers overlapped) equals
    the oracle bitwise in matched mode, incl. ragged last chunk and the wrap windows."""
    import torch
    u0 = synth.uniform(N + nt, 0, N, -1.0, 1.0)
    want = oracle.run(u0, 0.4, nt)
    pin_in = torch.from_numpy(u0).pin_memory()
    pin_out = torch.empty(N, dtype=torch.float64).pin_memory()
    with h1.Heat1D(N, 1, nt, 0.4, 1.0, 1.0, T=T, resident=False) as h:
        h.solve_host(pin_in, nt, pin_out)
        assert h.info()["stream_windows"] >= 3
        assert_bitwise(pin_out.numpy(), want, "solve_host N=%d nt=%d" % (N, nt))
        got = h.solve_host(u0, nt)                      # pageable numpy arrays work too
        assert_bitwise(got, want, "solve_host pageable")
        with pytest.raises(h1.Heat1DError) as ei:      # device state consumed
            h.run(1)
        assert ei.value.status == 3
        h.set_initial(u0)                               # and the handle is reusable
        h.run(nt)
        assert_bitwise(h.get(), want, "after solve_host")


def test_solve_host_rejects_in_place(h1):
    N = 300_001
    u0 = synth.uniform(2, 0, N, -1.0, 1.0)
    with h1.Heat1D(N, 1, 10, 0.4, 1.0, 1.0, resident=False) as h:
        with pytest.raises(h1.Heat1DError) as ei:
            h.solve_host(u0, 10, u0)
        assert ei.value.status == 1


def test_solve_host_plain_fallback(h1):
    """nt too large for windows, and the resident path: the plain three-call sequence."""
    N, nt = 10_000, 2000
    u0 = synth.uniform(12, 0, N, -1.0, 1.0)
    want = oracle.run(u0, 0.5, nt)
    for res in (False, None):
        with h1.Heat1D(N, 1, nt, 0.5, 1.0, 1.0, resident=res) as h:
            assert_bitwise(h.solve_host(u0, nt), want, "fallback res=%s" % res)
            assert h.info()["stream_windows"] == 0


def test_solve_host_fast_and_range_fallback(h1):
    N, nt = 1_000_003, 150
    u0 = synth.uniform(21, 0, N, -1.0, 1.0)
    with h1.Heat1D(N, 1, nt, 0.25, 1.0, 1.0, mode="fast", resident=False) as h:
        got = h.solve_host(u0, nt)
        assert h.info()["stream_windows"] >= 3
        assert np.max(np.abs(got - oracle.run(u0, 0.25, nt))) <= fast_bound(u0, nt)
        big = u0 * 1e300                                # scaled state would overflow: windows redone
        got = h.solve_host(big, nt)
        assert np.all(np.isfinite(got))
        assert np.max(np.abs(got - oracle.run(big, 0.25, nt))) <= fast_bound(big, nt)
    with h1.Heat1D(N, 1, nt, 0.5, 1.0, 1.0, mode="fast", resident=False) as h:
        want = u0.copy()
        for _ in range(nt):
            want = (np.roll(want, 1) + np.roll(want, -1)) * 0.5
        assert_bitwise(h.solve_host(u0, nt), want, "r=1/2 fast windows")


def test_ring_beyond_2pow32_cells(h1):
    """Maximum-size case: a ring of 2^32 + 12345 cells (2 x 32 GiB of state) -- every cell,
    tile and launch index is 64-bit -- checked with O3 windows around 2^31, 2^32 and the
    wrap after 100 steps, both modes."""
    import torch
    N, nt, k = (1 << 32) + 12345, 100, 0.4
    W = 256
    starts = [0, (1 << 31) - W // 2, (1 << 32) - W // 2, N - W // 2, 3_000_000_001]

    def ring_u0(first, count):  # u0 on ring cells [first, first+count) mod N, in contiguous pieces
        parts, i = [], first % N
        while count > 0:
            run = min(count, N - i)
            parts.append(synth.uniform(99, i, run, -1.0, 1.0))
            count -= run
            i = 0
        return np.concatenate(parts)

    want = {a: oracle.window(ring_u0(a - nt, W + 2 * nt), nt, k) for a in starts}
    for mode in ("matched", "fast"):
        with h1.Heat1D(N, 1, nt, k, 1.0, 1.0, mode=mode) as h:
            h.init_uniform(99, -1.0, 1.0)
            h.run()
            out = torch.empty(N, dtype=torch.float64, device="cuda")
            h.get(out)
        for a in starts:
            idx = (np.arange(a, a + W) % N).astype(np.int64)
            got = out[torch.from_numpy(idx).cuda()].cpu().numpy()
            if mode == "matched":
                assert_bitwise(got, want[a], "2^32 ring window %d" % a)
            else:
                assert np.max(np.abs(got - want[a])) <= 1e-12 * nt, a
        del out
        torch.cuda.empty_cache()


def test_caller_owned_device_memory(h1):
    """opts.dev_buf: the state lives in a torch tensor the caller owns (PyTorch provides the
    device memory; BASELINE.json north_star), single slab and virtual slabs, both modes."""
    import torch
    N, nt = 300_007, 50
    u0 = synth.uniform(31, 0, N, -1.0, 1.0)
    want = oracle.run(u0, 0.4, nt)
    for kw in ({}, {"virtual_slabs": 3}, {"resident": False}, {"mode": "fast"}):
        o = h1.default_opts()
        o.virtual_slabs = kw.get("virtual_slabs", 1)
        buf = torch.empty(h1.buffer_len(N, 1, o), dtype=torch.float64, device="cuda")
        with h1.Heat1D(N, 1, nt, 0.4, 1.0, 1.0, dev_buf=buf, **kw) as h:
            h.set_initial(u0)
            h.run()
            got = h.get()
        if kw.get("mode") == "fast":
            assert np.max(np.abs(got - want)) <= fast_bound(u0, nt)
        else:
            assert_bitwise(got, want, "dev_buf %r" % kw)
    small = torch.empty(1000, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        h1.Heat1D(N, 1, nt, 0.4, 1.0, 1.0, dev_buf=small)
    big = torch.empty(h1.buffer_len(N, 1, h1.default_opts()) + 1, dtype=torch.float64, device="cuda")
    with pytest.raises(h1.Heat1DError) as ei:                # 8-byte offset: not 256-byte aligned
        h1.Heat1D(N, 1, nt, 0.4, 1.0, 1.0, dev_buf=big[1:])
    assert ei.value.status == 1


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
def test_nan_poisoned_pads(h1, monkeypatch, transport):
    """Fault injection: every ghost pad starts as NaN (HEAT1D_POISON_PADS=1); the exchange
    must overwrite each pad before any kernel reads it, so the result stays bitwise exact."""
    monkeypatch.setenv("HEAT1D_POISON_PADS", "1")
    nx, np_, G = 30_011, 6, 3
    u0 = synth.uniform(808, 0, nx * np_, -1.0, 1.0)
    for T, nt in [(8, 2 * 8 + 3), (64, 64 + 1)]:
        want = oracle.run(u0, 0.4, nt)
        got = gpu_run(h1, u0, nx, np_, nt, 0.4, T=T, virtual_slabs=G, transport=transport)
        assert np.all(np.isfinite(got))
        assert_bitwise(got, want, "poisoned pads %s T=%d" % (transport, T))


def test_streaming_handle_small_windows(h1):
    """opts.window_cells: the device holds only two light-cone windows (rings larger than
    HBM); heat1d_solve_host streams the ring through them -- bitwise = oracle, ragged last
    window, the wrap; run/set_initial/get are refused; a window too small for nt is refused."""
    N, nt, W = (1 << 22) + 5, 200, 1 << 18
    u0 = synth.uniform(64, 0, N, -1.0, 1.0)
    want = oracle.run(u0, 0.4, nt)
    o = h1.default_opts()
    o.window_cells = W
    assert h1.buffer_len(N, 1, o) < N // 2          # vs 2 N + pads for the device-resident ring
    with h1.Heat1D(N, 1, nt, 0.4, 1.0, 1.0, window_cells=W) as h:
        assert_bitwise(h.solve_host(u0, nt), want, "streaming windows")
        assert h.info()["stream_windows"] >= N // W
        for call in (lambda: h.set_initial(u0), lambda: h.run(1), lambda: h.get()):
            with pytest.raises(h1.Heat1DError) as ei:
                call()
            assert ei.value.status == 7
        with pytest.raises(h1.Heat1DError) as ei:
            h.solve_host(u0, W // 4)                      # nt too deep for the window
        assert ei.value.status == 7
    with h1.Heat1D(N, 1, nt, 0.5, 1.0, 1.0, window_cells=W, mode="fast") as h:
        got = h.solve_host(u0, nt)
    assert np.max(np.abs(got - oracle.run(u0, 0.5, nt))) <= fast_bound(u0, nt)


def test_solve_host_nt_beyond_ring(h1):
    """nt > N must not read outside u0.  A device-resident handle falls back to
    the plain sequence (bitwise = oracle); a streaming handle refuses (EUNSUPPORTED)."""
    N, nt = 1000, 5000
    u0 = synth.uniform(65, 0, N, -1.0, 1.0)
    want = oracle.run(u0, 0.5, nt)
    with h1.Heat1D(N, 1, nt, 0.5, 1.0, 1.0, resident=False) as h:
        assert_bitwise(h.solve_host(u0, nt), want, "nt > N, resident ring")
        assert h.info()["stream_windows"] == 0
    with h1.Heat1D(N, 1, nt, 0.5, 1.0, 1.0, window_cells=1 << 18) as h:
        with pytest.raises(h1.Heat1DError) as ei:
            h.solve_host(u0, nt)
        assert ei.value.status == 7


def test_streaming_c4_ring_through_small_device_footprint(h1):
    """The C4 ring (2^31 cells, 16 GiB per state) streamed through 2^27-cell windows
    (~4 GiB of device memory) equals the device-resident solve bitwise, all cells."""
    import torch
    N, nt = C4.N, 100
    u0 = torch.empty(N, dtype=torch.float64).pin_memory()
    with h1.Heat1D(C4.nx, C4.np, nt, C4.k, C4.dt, C4.dx) as h:
        h.init_uniform(C4.seed, C4.lo, C4.hi)
        h.get(u0)
        h.run(nt)
        ref = torch.empty(N, dtype=torch.float64).pin_memory()
        h.get(ref)
    out = torch.empty(N, dtype=torch.float64).pin_memory()
    with h1.Heat1D(C4.nx, C4.np, nt, C4.k, C4.dt, C4.dx, window_cells=1 << 27) as h:
        h.solve_host(u0, nt, out)
        assert h.info()["stream_windows"] >= 16
    assert torch.equal(out, ref)


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
def test_comm_stream_delay_injection(h1, monkeypatch, transport):
    """a 200 us spin on the comm stream before every halo exchange
    (HEAT1D_COMM_DELAY_US) only delays the edge kernels -- results stay bitwise exact."""
    monkeypatch.setenv("HEAT1D_COMM_DELAY_US", "200")
    nx, np_, G, T, nt = 40_009, 4, 4, 16, 3 * 16 + 5
    u0 = synth.uniform(4242, 0, nx * np_, -1.0, 1.0)
    got = gpu_run(h1, u0, nx, np_, nt, 0.4, T=T, virtual_slabs=G, transport=transport)
    assert_bitwise(got, oracle.run(u0, 0.4, nt), "delayed comm stream (%s)" % transport)


@pytest.mark.parametrize("N", [1, 4, 10, 1000])
@pytest.mark.parametrize("nt", [0, 1, 100])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_spec_acceptance_grid(h1, N, nt, G):
    """SPEC.md:468-478 acceptance criterion 1 on this build: the GPU result equals the
    sequential oracle for N in {1,4,10,1000} x steps {0,1,100} x partitions {1,2,4,8}
    (partitions = slabs exchanging halos; rings with fewer cells than slabs are rejected)."""
    u0 = synth.uniform(N * 10 + G, 0, N, 0.0, 1.0)
    if N < G:
        with pytest.raises(h1.Heat1DError):
            h1.Heat1D(N, 1, nt, 0.25, 1.0, 1.0, virtual_slabs=G)
        return
    got = gpu_run(h1, u0, N, 1, nt, 0.25, virtual_slabs=G)
    assert_bitwise(got, oracle.run(u0, 0.25, nt), "N=%d nt=%d G=%d" % (N, nt, G))


def test_convergence_to_the_mean(h1):
    """SPEC.md:126/:471 on the GPU: N = 64, 1e5 steps -> every cell within 1e-6 of the mean
    (one resident launch), bitwise equal to the oracle."""
    N, nt = 64, 100_000
    u0 = synth.uniform(64, 0, N, 0.0, 1.0)
    got = gpu_run(h1, u0, N, 1, nt, 0.25)
    assert np.max(got) - np.min(got) < 1e-6
    assert abs(float(np.mean(got)) - float(np.mean(u0))) < 1e-9
    assert_bitwise(got, oracle.run(u0, 0.25, nt), "convergence")


@pytest.mark.parametrize("G", [2, 3, 8])
@pytest.mark.parametrize("mode", ["matched", "fast"])
def test_solve_host_halo_emulates_ranks(h1, G, mode):
    """heat1d_solve_host_halo -- the per-rank half of the multi-rank heat1d_solve_host (one
    exchange of nt-deep halos, then no communication): G slabs of a ring, each solved by its
    own handle from its cells plus the nt cells on either side, reassemble the oracle's ring
    bitwise (matched) / within the bound (fast)."""
    N, nt = 3_000_017, 150
    u0 = synth.uniform(300 + G, 0, N, -1.0, 1.0)
    want = oracle.run(u0, 0.4, nt)
    parts = []
    for g in range(G):
        first, count = h1.partition(N, 1, G, g)
        idx = np.arange(first - nt, first + count + nt) % N
        ext = u0[idx]
        with h1.Heat1D(count, 1, nt, 0.4, 1.0, 1.0, resident=False, mode=mode) as h:
            parts.append(h.solve_host_halo(ext[nt:nt + count].copy(), ext[:nt].copy(), ext[nt + count:].copy(), nt))
            assert h.info()["stream_windows"] >= 2
    got = np.concatenate(parts)
    if mode == "matched":
        assert_bitwise(got, want, "solve_host_halo G=%d" % G)
    else:
        assert np.max(np.abs(got - want)) <= fast_bound(u0, nt)
    with h1.Heat1D(1000, 1, 100, 0.4, 1.0, 1.0, resident=False) as h:       # slab too small for windows
        with pytest.raises(h1.Heat1DError) as ei:
            h.solve_host_halo(u0[:1000].copy(), u0[:100].copy(), u0[:100].copy(), 100)
        assert ei.value.status == 7


@pytest.mark.parametrize("resident", [True, False])
def test_non_blocking_handle_is_stream_ordered(h1, resident):
    """opts.blocking = 0: set_initial / run / get only enqueue on the handle's stream; after a
    stream synchronisation the result equals the oracle bitwise (device and pinned host buffers)."""
    import torch
    N, nt = 300_007, 130
    u0 = synth.uniform(71, 0, N, -1.0, 1.0)
    want = oracle.run(u0, 0.5, nt)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)  # torch's copies below are ordered with the handle's work
    with h1.Heat1D(N, 1, nt, 0.5, 1.0, 1.0, blocking=False, stream=st, resident=resident) as h:
        dev_in = torch.from_numpy(u0).cuda()
        dev_out = torch.empty_like(dev_in)
        for _ in range(2):
            h.set_initial(dev_in)
            h.run(nt)
            h.get(dev_out)
        torch.cuda.synchronize()
        assert_bitwise(dev_out.cpu().numpy(), want, "non-blocking, device buffers")
        host_in = torch.from_numpy(u0).pin_memory()
        host_out = torch.empty(N, dtype=torch.float64).pin_memory()
        h.set_initial(host_in)
        h.run(nt)
        h.get(host_out)
        torch.cuda.synchronize()
        assert_bitwise(host_out.numpy(), want, "non-blocking, pinned host buffers")
        assert_bitwise(h.solve_host(u0, nt), want, "non-blocking handle, solve_host returns filled")
    torch.cuda.set_stream(torch.cuda.default_stream())


@pytest.mark.parametrize("transport", ["p2p", "nccl"])
def test_trace_shows_halo_work_beside_the_interior(h1, transport):
    """heat1d_trace (profiling): per pass one comm-stream interval (exchange + edge strips)
    and one compute-stream K2 interval per slab; the comm work of a pass starts before that
    pass's interior ends (the two streams overlap), and the result is still bitwise."""
    N, G, T, nt = 4 * 200_000, 4, 16, 16 * 5
    u0 = synth.uniform(81, 0, N, -1.0, 1.0)
    with h1.Heat1D(200_000, 4, nt, 0.5, 1.0, 1.0, T=T, virtual_slabs=G, transport=transport,
                   resident=False) as h:
        h.set_initial(u0)
        h.set_profiling(True)
        h.run(nt)
        tr = h.trace()
        n, ms = h.profile()
        h.set_profiling(False)
        got = h.get()
    assert_bitwise(got, oracle.run(u0, 0.5, nt), "traced run")
    halo = [e for e in tr if e[1] == "halo"]
    k2 = [e for e in tr if e[1] == "K2"]
    assert len(halo) == nt // T and len(k2) == G * (nt // T)
    assert all(e[0] == 1 for e in halo) and all(e[0] == 0 for e in k2)
    assert n == len(k2) and ms > 0
    for i, hv in enumerate(halo):
        ks = k2[i * G:(i + 1) * G]
        assert all(e[3] >= e[2] >= 0 for e in ks) and hv[3] >= hv[2] >= 0
        assert hv[2] < max(e[3] for e in ks)   # the halo work starts while the interior runs


@pytest.mark.parametrize("mailbox", [False, True])
def test_resident_tag_counters_wrap(h1, monkeypatch, mailbox):
    """K6's halo tags are 32-bit counters (tagged words, resident.cu): started just below 2^32
    (test hook HEAT1D_K6_COUNTER0), a sequence of runs crosses the wrap -- the span tags restart
    with freshly zeroed slots, the mailbox tags (exchange index + 1) wrap through 0 -- and stays
    bitwise equal to the oracle."""
    monkeypatch.setenv("HEAT1D_K6_COUNTER0", str(2 ** 32 - 20))  # the 4th run crosses 2^32
    if mailbox:
        monkeypatch.setenv("HEAT1D_K6_MAILBOX", "1")
    N, T = 300_007, 64
    u0 = synth.uniform(5, 0, N, -1.0, 1.0)
    with h1.Heat1D(N, 1, 0, 0.5, 1.0, 1.0, T=T, resident=True) as h:
        h.set_initial(u0)
        want = u0
        for nt in (5 * T + 3, 1, 2 * T, 7 * T + 11, T + 1, 3 * T):
            h.run(nt)
            want = oracle.run(want, 0.5, nt)
            assert_bitwise(h.get(), want, "tags across the wrap, mailbox=%s nt=%d" % (mailbox, nt))


@pytest.mark.parametrize("transport", ["p2p", "nccl"])
def test_feed_tiles_multi_slab_interior(h1, transport):
    """Two slabs of ~4M cells each at the auto T (128): every slab's interior pass [T, n - T) runs
    as feed-tile strips of several tiles per CTA, next to the edge strips on the comm stream;
    bitwise equal to the oracle after two full passes and a tail."""
    nx = (1 << 22) + 1001
    N, nt = 2 * nx, 2 * 128 + 7
    u0 = synth.uniform(77, 0, N, -1.0, 1.0)
    with h1.Heat1D(nx, 2, nt, 0.5, 1.0, 1.0, virtual_slabs=2, transport=transport) as h:
        h.set_initial(u0)
        h.run(nt)
        info = h.info()
        assert info["T"] == 128 and info["pass_feed"] == 1
        assert_bitwise(h.get(), oracle.run(u0, 0.5, nt), "feed strips, 2 slabs, %s" % transport)


@pytest.mark.parametrize("T", [64, 96, 128])
@pytest.mark.parametrize("k,mode", [(0.5, "matched"), (0.4, "matched"), (0.5, "fast"), (0.4, "fast")])
def test_feed_tiles_every_depth(h1, T, k, mode):
    """k2f_pass at each instantiated depth with several tiles per strip (4M cells: ~14 k cells per
    CTA strip), 3-op / 4-op matched bitwise, 1-op / 2-op fast within the north_star bound."""
    N = (1 << 22) + 777
    nt = 2 * T + 3
    u0 = synth.uniform(31 + T, 0, N, -1.0, 1.0)
    with h1.Heat1D(N, 1, nt, k, 1.0, 1.0, T=T, mode=mode, resident=False) as h:
        h.set_initial(u0)
        h.run(nt)
        info = h.info()
        assert info["pass_feed"] == 1 and info["T"] == T
        got = h.get()
    want = oracle.run(u0, k, nt)
    if mode == "matched":
        assert_bitwise(got, want, "feed T=%d k=%g" % (T, k))
    else:
        assert float(np.max(np.abs(got - want))) <= 1e-12 * float(np.max(np.abs(u0))) * nt
