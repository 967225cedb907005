"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Every pin is chosen so that a plausible mistake in oracle/heat1d_oracle.c
(a dropped term, wrong sign, wrong index, in-place instead of Jacobi, wrong
wrap, wrong r, off-by-one step count) fails at least one test:

- exact rational brute force (fractions.Fraction) on tiny rings and on the
  real 1000-cell C1 ring                       -> arithmetic, wrap, Jacobi
- hand-evaluated fixtures tests/golden/*.txt    -> the same, independently typed
- single/multi Fourier mode closed form         -> r, sign, step count, wrap
- conservation, max principle, convergence      -> invariants of Eq. 2 on a ring
- decomposition invariants (O2, O3, rotation, split runs)

Citations: PAPER.md:64-73 (Eq. 2, u0 = x_i, periodic ring, segments),
SPEC.md:75-127 (examples and invariants), BASELINE.json north_star (oracle checks).
"""
from __future__ import annotations

import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- helpers
def exact_steps(u0, r: Fraction, nt: int):
    """Exact rational Jacobi sweeps on a ring; yields u(t) for t = 1..nt."""
    u = [Fraction(x) for x in u0]
    N = len(u)
    for _ in range(nt):
        u = [u[i] + r * (u[i - 1] - 2 * u[i] + u[(i + 1) % N]) for i in range(N)]
        yield u


def representable(q: Fraction) -> bool:
    return Fraction(float(q)) == q


def ulp(x: float) -> float:
    return math.ulp(abs(x)) if x != 0 else math.ulp(0.0)


def parse_golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append([p.strip() for p in line.split("|")])
    return rows


# ---------------------------------------------------------------- r
def test_r_formula():
    # r = k*dt/dx^2 (north_star), not k*dt/dx; paper-literal 2h is k*dt/(2*dx)
    assert oracle.r_of(1.0, 0.25, 2.0) == 1.0 / 16.0
    assert oracle.r_of(0.5, 1.0, 1.0) == 0.5
    assert oracle.r_of(0.4, 1.0, 1.0) == 0.4
    assert oracle.r_of(0.25, 1.0, 1.0, paper_2h=True) == 0.125
    assert oracle.r_of(1.0, 0.25, 2.0, paper_2h=True) == 1.0 / 16.0
    assert oracle.r_of(1.0, 1.0, 4.0, paper_2h=True) == 1.0 / 8.0
    assert oracle.r_of(1.0, 1.0, 4.0) == 1.0 / 16.0


# ---------------------------------------------------------------- golden fixtures
@pytest.mark.parametrize("row", parse_golden("spec_examples.txt"), ids=lambda r: r[0])
def test_spec_examples(row):
    name, params, u0s, steps, exp = row
    k, dt, dx, den = params.split()
    r = oracle.r_of(float(k), float(dt), float(dx), paper_2h=(den == "2dx"))
    u0 = [float(Fraction(x)) for x in u0s.split()]
    got = oracle.run(u0, r, int(steps))
    want = np.array([float(Fraction(x)) for x in exp.split()])
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("row", parse_golden("small_rings.txt"), ids=lambda r: "r%s_N%s_t%s" % (r[0], r[1], r[2]))
def test_small_ring_hand_values(row):
    rs, Ns, ts, exp = row
    r = Fraction(rs)
    N, t = int(Ns), int(ts)
    want = [Fraction(x) for x in exp.split()]
    assert len(want) == N
    got = oracle.run(np.arange(N, dtype=np.float64), float(r), t)
    if r.denominator in (1, 2, 4):       # dyadic r: fp64 is exact here
        np.testing.assert_array_equal(got, np.array([float(q) for q in want]))
    else:                                 # r = 2/5 is not representable: <= 2 ulp
        for g, q in zip(got, want):
            assert abs(Fraction(g) - q) <= 2 * Fraction(ulp(float(q)))


def test_sum_spec_total_heat():
    # total_heat([0,1,2,3]) = 6, and 6 after one sweep
    u = oracle.run([0.0, 1.0, 2.0, 3.0], 0.25, 1)
    assert math.fsum(u) == 6.0


# ---------------------------------------------------------------- exact brute force
@pytest.mark.parametrize("r", [Fraction(1, 4), Fraction(1, 2)])
@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6, 7, 8, 13])
def test_exact_rational_tiny_rings(N, r):
    """fp64 oracle == exact rationals for every step while all values are representable."""
    u0 = np.arange(N, dtype=np.float64)
    checked = 0
    for t, ex in enumerate(exact_steps(u0, r, 40), start=1):
        if not all(representable(q) for q in ex):
            break
        got = oracle.run(u0, float(r), t)
        np.testing.assert_array_equal(got, np.array([float(q) for q in ex]), err_msg="t=%d" % t)
        checked = t
    assert checked >= 3


@pytest.mark.parametrize("N", [3, 4, 5, 6, 7, 8])
def test_exact_rational_r_two_fifths(N):
    """r=2/5 (not representable): oracle within a few ulp of the exact solution for t<=10."""
    u0 = np.arange(N, dtype=np.float64)
    exs = list(exact_steps(u0, Fraction(2, 5), 10))
    got = u0.copy()
    for t, ex in enumerate(exs, start=1):
        got = oracle.run(got, 0.4, 1)
        for g, q in zip(got, ex):
            # rounding of r (rel 5.6e-17 * t) plus <= 1 rounding per op per step
            assert abs(Fraction(g) - q) <= 4 * t * Fraction(ulp(float(max(ex)))), (t, g, q)


def test_exact_rational_c1_ring():
    """The real C1 ring (N=1000, r=1/2, u0=i): oracle equals exact arithmetic
    through step 46 (first rational not representable at 47)."""
    N = 1000
    u0 = np.arange(N, dtype=np.float64)
    last_exact = 0
    cur = u0.copy()
    for t, ex in enumerate(exact_steps(u0, Fraction(1, 2), 50), start=1):
        cur = oracle.run(cur, 0.5, 1)
        if not all(representable(q) for q in ex):
            break
        np.testing.assert_array_equal(cur, np.array([float(q) for q in ex]), err_msg="t=%d" % t)
        last_exact = t
    assert last_exact >= 46


# ---------------------------------------------------------------- closed form
def closed_form(N, modes, amps, r, t, phase="sin"):
    """u_t[i] = sum_j a_j g_j^t f(2 pi m_j i / N),  g_j = 1 - 4 r sin^2(pi m_j / N)."""
    i = np.arange(N, dtype=np.int64)
    out = np.zeros(N)
    for m, a in zip(modes, amps):
        s = math.sin(math.pi * m / N)
        lg = math.log1p(-4.0 * r * s * s) if 4.0 * r * s * s < 1.0 else None
        if lg is not None:
            gt = math.exp(t * lg)
        else:
            gt = (1.0 - 4.0 * r * s * s) ** t
        ang = 2.0 * np.pi * ((m * i) % N) / N
        out += a * gt * (np.sin(ang) if phase == "sin" else np.cos(ang))
    return out


@pytest.mark.parametrize("N,m,r,t", [(8, 1, 0.25, 200), (1000, 3, 0.4, 500), (4096, 5, 0.25, 2000),
                                     (64, 7, 0.5, 300), (4, 2, 0.5, 9)])
def test_closed_form_single_mode(N, m, r, t):
    u0 = synth.sine_modes(N, [m], [1.0], 0, N) if (2 * m) % N else np.cos(2 * np.pi * np.arange(N) * m / N)
    phase = "sin" if (2 * m) % N else "cos"
    got = oracle.run(u0, r, t)
    want = closed_form(N, [m], [1.0], r, t, phase)
    assert np.max(np.abs(got - want)) <= 1e-12


def test_closed_form_n8_m1_quarter():
    # g = (2 + sqrt 2)/4 per step for N=8, m=1, r=1/4 (cos form: u0 = cos(2 pi i/8))
    g = (2.0 + math.sqrt(2.0)) / 4.0
    u0 = np.cos(2 * np.pi * np.arange(8) / 8)
    got = oracle.run(u0, 0.25, 50)
    np.testing.assert_allclose(got, g ** 50 * u0, atol=1e-14, rtol=0)


def test_closed_form_eight_modes_c3_shape():
    """C3's input recipe (8 modes 2^j-1, amplitudes U(7,j)) on a scaled ring."""
    N, r, nt = 1 << 12, 0.4, 1000
    modes = [(1 << j) - 1 for j in range(1, 9)]
    amps = synth.uniform(7, 0, 8)
    u0 = synth.sine_modes(N, modes, amps, 0, N)
    got = oracle.run(u0, r, nt)
    want = closed_form(N, modes, amps, r, nt)
    assert np.max(np.abs(got - want)) <= 1e-12


def test_closed_form_non_unit_dx():
    # k=0.1, dt=0.5, dx=0.5 -> r = 0.2; checks r uses dx^2 on a physical grid
    r = oracle.r_of(0.1, 0.5, 0.5)
    assert abs(r - 0.2) < 1e-16
    N, m, t = 256, 3, 400
    u0 = synth.sine_modes(N, [m], [1.0], 0, N)
    got = oracle.run(u0, r, t)
    want = closed_form(N, [m], [1.0], 0.2, t)
    assert np.max(np.abs(got - want)) <= 1e-12


# ---------------------------------------------------------------- invariants
@pytest.mark.parametrize("lo,hi,r", [(0.0, 1.0, 0.5), (-1.0, 1.0, 0.5), (-1.0, 1.0, 0.4), (0.0, 1.0, 0.25)])
def test_conservation(lo, hi, r):
    """sum(u) is invariant on the ring to 1e-9 relative (north_star),
    normalised by sum|u0| (reading c15)."""
    N, nt = 100_000, 1000
    u0 = synth.uniform(42, 0, N, lo, hi)
    u = oracle.run(u0, r, nt)
    drift = abs(math.fsum(u) - math.fsum(u0))
    assert drift <= 1e-9 * math.fsum(np.abs(u0))


def test_max_principle():
    """0 < r <= 1/2: max non-increasing, min non-decreasing each step."""
    N = 1000
    for r in (0.5, 0.4, 0.25):
        u = synth.uniform(3, 0, N, -1.0, 1.0)
        mx, mn = u.max(), u.min()
        for _ in range(300):
            u = oracle.run(u, r, 1)
            assert u.max() <= mx and u.min() >= mn
            mx, mn = u.max(), u.min()


def test_convergence_to_mean():
    """N=64, 1e5 steps: every cell converges to the initial mean."""
    u0 = synth.uniform(5, 0, 64)
    u = oracle.run(u0, 0.25, 100_000)
    assert u.max() - u.min() < 1e-6
    assert abs(u.mean() - u0.mean()) < 1e-12


def test_nyquist_mode_does_not_decay_at_half():
    # reading c10: at r=1/2 the m=N/2 mode has g=-1 ([2,1,2,1] <-> [1,2,1,2])
    u = oracle.run([2.0, 1.0, 2.0, 1.0], 0.5, 1)
    np.testing.assert_array_equal(u, [1.0, 2.0, 1.0, 2.0])
    u = oracle.run([2.0, 1.0, 2.0, 1.0], 0.5, 2)
    np.testing.assert_array_equal(u, [2.0, 1.0, 2.0, 1.0])


# ---------------------------------------------------------------- decomposition
@pytest.mark.parametrize("nx,np_", [(3000, 1), (1500, 2), (1000, 3), (250, 12), (1, 3000), (7, 3), (1, 1), (2, 1), (1, 2)])
def test_segmented_equals_plain(nx, np_):
    """O2 (paper's segmented queue algorithm) == O1 bitwise."""
    u0 = synth.uniform(11, 0, nx * np_, -1.0, 1.0)
    np.testing.assert_array_equal(oracle.segmented(u0, nx, np_, 0.4, 120), oracle.run(u0, 0.4, 120))


def test_nx_np_invariance_c2_shape():
    """C2's (nx, np)-invariance check on a 1e5 ring (full C2 is a GPU-test case)."""
    N = 100_000
    u0 = synth.uniform(42, 0, N)
    ref = oracle.run(u0, 0.5, 50)
    for nx, np_ in [(1000, 100), (100_000, 1), (250, 400)]:
        np.testing.assert_array_equal(oracle.segmented(u0, nx, np_, 0.5, 50), ref)


@pytest.mark.parametrize("a,b", [(0, 3000), (-40, 60), (1000, 1001), (2950, 3050), (17, 530)])
def test_window_equals_plain(a, b):
    N, t, r = 3000, 120, 0.4
    u0 = synth.uniform(13, 0, N, -1.0, 1.0)
    full = oracle.run(u0, r, t)
    idx = np.arange(a, b) % N
    np.testing.assert_array_equal(oracle.window_of_ring(u0, a, b, t, r), full[idx])


def test_rotation_equivariance():
    N = 997
    u0 = synth.uniform(17, 0, N)
    for s in (1, 5, 500):
        np.testing.assert_array_equal(oracle.run(np.roll(u0, s), 0.4, 77), np.roll(oracle.run(u0, 0.4, 77), s))


def test_split_run_invariance():
    u0 = synth.uniform(19, 0, 513, -1.0, 1.0)
    a = oracle.run(oracle.run(u0, 0.4, 13), 0.4, 29)
    np.testing.assert_array_equal(a, oracle.run(u0, 0.4, 42))


def test_zero_steps_identity():
    u0 = synth.uniform(23, 0, 100)
    np.testing.assert_array_equal(oracle.run(u0, 0.4, 0), u0)


def test_bad_args():
    with pytest.raises(ValueError):
        oracle.run([], 0.5, 1)
    with pytest.raises(ValueError):
        oracle.segmented(np.zeros(10), 3, 3, 0.5, 1)


def test_fast_mode_formula_at_half_is_closer_to_exact_than_matched():
    """DESIGN.md reading c21: at r = 1/2 fast mode computes fl(u_{i-1} + u_{i+1}) / 2 per step
    (the GPU is checked bitwise against exactly this in tests/test_gpu_parity.py).  Against
    exact rational arithmetic (fractions) that one-rounding form is at least as accurate as
    the canonical three-rounding order -- on random rings about 2-4x closer after 300 steps --
    and both are far inside the north_star bound 1e-12*max|u0|*nt."""
    import synth
    from fractions import Fraction
    for seed in (1, 2, 3):
        N, nt = 64, 300
        u0 = synth.uniform(seed, 0, N, -1.0, 1.0)
        ex = [Fraction(float(x)) for x in u0]
        fast = u0.copy()
        for _ in range(nt):
            ex = [(ex[i - 1] + ex[(i + 1) % N]) / 2 for i in range(N)]
            fast = (np.roll(fast, 1) + np.roll(fast, -1)) * 0.5
        matched = oracle.run(u0, 0.5, nt)
        ef = max(abs(Fraction(float(fast[i])) - ex[i]) for i in range(N))
        em = max(abs(Fraction(float(matched[i])) - ex[i]) for i in range(N))
        assert ef <= em, (seed, float(ef), float(em))
        assert em < Fraction(1, 10**12) * nt
