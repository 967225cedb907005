"""Matched mode stays bitwise equal to the oracle at the ends of the fp64 range.  -m gpu.

The contracted matched forms -- DFMA(-2,b,a) for a - 2.0*b, and DFMA(r,t,b) for
b + r*t when r = 2^-j -- equal the oracle's literal sequence (DESIGN.md
reading c3) only while 2b does not overflow and r*t is exact.  Every kernel checks the
cells a block of steps starts from and runs the literal 5-op sequence for blocks outside
that range (stencil.cuh).  These tests feed states that exercise both sides of the check:
subnormal-scale rings (r*t inexact: fma and the literal order differ), rings that straddle
the guard's bottom bound, normal rings with a few planted subnormal cells (only some tiles
take the fallback), and rings near the top of the range (2b overflows in the oracle).

Inputs are seeded integers scaled by powers of two (np.ldexp); expected values come from
oracle/ only.  NaN results (the oracle's inf - inf) compare as NaN, payloads ignored.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

TINY = 2.0 ** -1074  # the smallest subnormal


@pytest.fixture(scope="module")
def h1():
    import torch
    from paper_2307_01117_b200 import _build
    _build.build()
    import paper_2307_01117_b200 as m
    torch.cuda.set_device(0)
    return m


def assert_same(got, want, what=""):
    """Bitwise on every non-NaN cell, NaN exactly where the oracle has NaN."""
    gn, wn = np.isnan(got), np.isnan(want)
    ok = np.array_equal(gn, wn) and np.array_equal(got[~wn].view(np.uint64), want[~wn].view(np.uint64))
    if not ok:
        bad = np.flatnonzero((gn != wn) | ((got != want) & ~wn))
        i = bad[0] if bad.size else -1
        raise AssertionError("%s: %d cells differ, first at %d: %r vs %r" % (what, bad.size, i, got[i], want[i]))


def run_gpu(h1, u0, nt, k, **kw):
    N = u0.size
    with h1.Heat1D(N, 1, nt, k, 1.0, 1.0, **kw) as h:
        h.set_initial(u0)
        h.run(nt)
        return h.get(), h.info()


def rng_ints(seed, n, lo, hi):
    """Seeded integers in [lo, hi) from the shared splitmix64 generator (synth/)."""
    u = synth.uniform(seed, 0, n)
    return np.floor(lo + (hi - lo) * u)


# ---- input recipes (seeded; inputs only -- no method arithmetic)
def subnormal_ring(n, seed=11):
    """Integers in [-2^20, 2^20) times 2^-1074: every value and most products subnormal."""
    return np.ldexp(rng_ints(seed, n, -(1 << 20), 1 << 20), -1074)


def straddle_ring(n, seed=12):
    """Normal values whose exponents straddle the guard bound 2^(jT-1022) of T = 8..64."""
    m = rng_ints(seed, n, -(1 << 52), 1 << 52)
    e = rng_ints(seed + 1, n, -1070, -930)
    return np.ldexp(m, (e - 52).astype(np.int64))


def planted_ring(n, seed=13, count=40):
    """U[-1,1) with `count` cells replaced by subnormals: only their tiles fall back."""
    u = synth.uniform(seed, 0, n, -1.0, 1.0)
    pos = rng_ints(seed + 1, count, 0, n).astype(np.int64)
    u[pos] = np.ldexp(rng_ints(seed + 2, count, -1000, 1000), -1074)
    return u


def huge_ring(n, seed=14, scale_exp=1023):
    """U[-1,1) * 2^scale_exp: at 1023 the oracle's 2.0*b overflows to inf for |b| >= 2^1023."""
    return np.ldexp(synth.uniform(seed, 0, n, -1.0, 1.0), scale_exp)


RECIPES = {
    "subnormal": subnormal_ring,
    "straddle": straddle_ring,
    "planted": planted_ring,
    "huge1023": lambda n: huge_ring(n, scale_exp=1024),      # |u| up to ~2^1024: overflows
    "top1022": lambda n: huge_ring(n, scale_exp=1023),       # |u| in [2^1022, 2^1023): guard fails, no overflow
    "below1022": lambda n: huge_ring(n, scale_exp=1022),     # |u| < 2^1022: contracted path, exact
}


def test_worked_example_subnormal(h1):
    """[4u, 1u, 5u], u = 2^-1074, r = 1/2: the oracle's r*t = 3.5u rounds to 4u (ties to even),
    so cell 1 = 1u + 4u = 5u; the contracted fma(1/2, 7u, 1u) = fl(4.5u) would give 4u."""
    u0 = np.array([4.0, 1.0, 5.0]) * TINY
    want = oracle.run(u0, 0.5, 1)
    assert want[1] == 5 * TINY
    for kw in (dict(resident=False), dict(resident=True), dict(kernel="naive"), dict(T=1, resident=False)):
        got, _ = run_gpu(h1, u0, 1, 0.5, **kw)
        assert_same(got, want, "worked example %r" % kw)
    # and over many steps
    want = oracle.run(u0, 0.5, 50)
    for kw in (dict(resident=False), dict(resident=True)):
        got, _ = run_gpu(h1, u0, 50, 0.5, **kw)
        assert_same(got, want, "worked example 50 steps %r" % kw)


@pytest.mark.parametrize("recipe", sorted(RECIPES))
@pytest.mark.parametrize("k", [0.5, 0.25, 0.4])
@pytest.mark.parametrize("T", [8, 64])
def test_k2_pass_extremes(h1, recipe, k, T):
    """K2 (several tiles, a ragged tail tile, a tail pass) on extreme-range rings."""
    N = 100_003
    nt = 2 * T + 3
    u0 = RECIPES[recipe](N)
    want = oracle.run(u0, k, nt)
    got, info = run_gpu(h1, u0, nt, k, T=T, resident=False)
    assert info["dp_ops"] == (3 if k in (0.5, 0.25) else 4)
    assert_same(got, want, "K2 %s k=%g T=%d" % (recipe, k, T))


@pytest.mark.parametrize("recipe", sorted(RECIPES))
@pytest.mark.parametrize("k", [0.5, 0.4])
@pytest.mark.parametrize("T", [16, 64])
def test_k6_resident_extremes(h1, recipe, k, T):
    """K6 (whole solve on chip; per-warp guard every period)."""
    N = 100_003
    nt = 3 * T + 5
    u0 = RECIPES[recipe](N)
    want = oracle.run(u0, k, nt)
    got, info = run_gpu(h1, u0, nt, k, T=T, resident=True)
    assert info["resident"] == 1
    assert_same(got, want, "K6 %s k=%g T=%d" % (recipe, k, T))


@pytest.mark.parametrize("recipe", ["subnormal", "planted", "huge1023", "straddle"])
@pytest.mark.parametrize("transport", ["p2p", "nccl"])
def test_virtual_slabs_extremes(h1, recipe, transport):
    """Several slabs: K2 interior + K3 / K3p edge strips, both guarded."""
    N, G, T = 4 * 25_000, 4, 16
    nt = 3 * T + 7
    u0 = RECIPES[recipe](N)
    want = oracle.run(u0, 0.5, nt)
    with h1.Heat1D(25_000, 4, nt, 0.5, 1.0, 1.0, T=T, virtual_slabs=G, transport=transport) as h:
        h.set_initial(u0)
        h.run(nt)
        assert_same(h.get(), want, "slabs %s %s" % (recipe, transport))


@pytest.mark.parametrize("recipe", ["subnormal", "planted", "huge1023"])
def test_naive_and_windows_extremes(h1, recipe):
    """K1 (matched: the literal sequence) and the light-cone windows of heat1d_solve_host."""
    N, nt = 1 << 20, 9
    u0 = RECIPES[recipe](N)
    want = oracle.run(u0, 0.5, nt)
    got, _ = run_gpu(h1, u0, nt, 0.5, kernel="naive")
    assert_same(got, want, "naive %s" % recipe)
    with h1.Heat1D(N, 1, nt, 0.5, 1.0, 1.0, T=4, resident=False) as h:
        out = h.solve_host(np.ascontiguousarray(u0), nt)
        assert h.info()["stream_windows"] > 1
        assert_same(out, want, "windows %s" % recipe)


def test_mailbox_loopback_extremes(h1, monkeypatch):
    """K6 with the cross-rank mailbox protocol in loopback (HEAT1D_K6_MAILBOX=1)."""
    monkeypatch.setenv("HEAT1D_K6_MAILBOX", "1")
    N, T = 100_003, 64
    for recipe in ("subnormal", "planted"):
        u0 = RECIPES[recipe](N)
        with h1.Heat1D(N, 1, 0, 0.5, 1.0, 1.0, T=T, resident=True) as h:
            h.set_initial(u0)
            want = u0
            for nt in (2 * T + 1, T):
                h.run(nt)
                want = oracle.run(want, 0.5, nt)
                assert_same(h.get(), want, "mailbox %s" % recipe)


@pytest.mark.parametrize("recipe", ["subnormal", "straddle", "top1022", "huge1023", "below1022"])
@pytest.mark.parametrize("k,ops", [(0.75, 4), (2.0, 3)])
@pytest.mark.parametrize("resident", [False, True])
def test_unstable_r_extremes(h1, recipe, k, ops, resident):
    """r > 1/2 (allow_unstable): the guard's top bound takes the growth factor G = 4r per step
    (DESIGN.md c3), and r = 2 (a power of two >= 1) runs the 3-op form with no bottom bound (2*t is
    exact down to the subnormals).  The state grows like |1 - 4r|^t, so huge rings overflow to
    inf / NaN within a few steps -- compared NaN-aware, bitwise elsewhere."""
    N, T = 50_003, 8
    nt = 2 * T + 3
    u0 = RECIPES[recipe](N)
    want = oracle.run(u0, k, nt)
    got, info = run_gpu(h1, u0, nt, k, T=T, resident=resident, allow_unstable=True)
    assert info["dp_ops"] == ops and info["resident"] == (1 if resident else 0)
    assert_same(got, want, "r=%g %s resident=%s" % (k, recipe, resident))


@pytest.mark.parametrize("resident", [False, True])
def test_nonfinite_inputs(h1, resident):
    """u0 holding +-inf and NaN cells (special values are states too): the guard rejects their
    blocks (exponent 0x7ff is above every top bound), so those blocks run the literal sequence and
    the inf/NaN fronts spread exactly as in the oracle; everything else stays bitwise."""
    N, T = 60_001, 16
    nt = 3 * T + 1
    u0 = synth.uniform(21, 0, N, -1.0, 1.0)
    u0[[5, 20_000]] = np.inf
    u0[[7_777, 40_000]] = -np.inf
    u0[[33_333, N - 1]] = np.nan
    want = oracle.run(u0, 0.5, nt)
    got, _ = run_gpu(h1, u0, nt, 0.5, T=T, resident=resident)
    assert_same(got, want, "non-finite u0 resident=%s" % resident)
    assert np.isnan(want).sum() > 0 and np.isfinite(want).sum() > N // 2


@pytest.mark.parametrize("recipe", ["planted", "straddle", "subnormal", "huge1023"])
@pytest.mark.parametrize("mode", ["matched", "fast"])
def test_feed_tiles_extremes(h1, recipe, mode):
    """K2 feed tiles (k2f_pass) on a ring large enough for several left-fed tiles per CTA strip,
    at the auto T (128), extreme magnitudes: a tile takes the contracted form only if its own
    cells and the previous tile's passed the guard (the fed boundary depends on both), so planted
    subnormals make their tile AND the next one fall back.  Matched: bitwise; fast mode (the
    normal-range planted recipe only): within the north_star bound."""
    if mode == "fast" and recipe not in ("planted",):
        pytest.skip("the fast-mode bound is relative to normal-range states")
    N = (1 << 22) + 12345
    nt = 2 * 128 + 5
    u0 = RECIPES[recipe](N)
    want = oracle.run(u0, 0.5, nt)
    got, info = run_gpu(h1, u0, nt, 0.5, resident=False, mode=mode)
    assert info["T"] == 128 and info["pass_feed"] == 1
    if mode == "matched":
        assert_same(got, want, "feed tiles %s" % recipe)
    else:
        bound = 1e-12 * float(np.max(np.abs(u0))) * nt
        assert float(np.max(np.abs(got - want))) <= bound
