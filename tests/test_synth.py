"""Input generators (synth/): pinned to published splitmix64 values and to
the configs of BASELINE.json.  -m "not gpu"."""
import numpy as np

import synth
from synth.configs import C1, C2, C3, C4, C5, CONFIGS


def test_splitmix64_reference_value():
    # splitmix64 seeded with 0: first output 0xe220a8397b1dcdaf (the standard
    # reference value of Vigna's generator)
    assert int(synth.splitmix64(0, 0, 1)[0]) == 0xE220A8397B1DCDAF


def test_uniform_vectors():
    # SURVEY.md §8(d) test vectors
    np.testing.assert_array_equal(
        synth.uniform01(42, 0, 4),
        [0.7415648787718233, 0.1599103928769201, 0.27860113025513866, 0.34419071652363753])
    np.testing.assert_array_equal(
        synth.uniform(1234, 0, 4, -1.0, 1.0),
        [0.46133304908124795, 0.18577971602997234, -0.5957342513797803, -0.38762641589925817])


def test_windowed_generation_matches_full():
    full = synth.uniform(42, 0, 1000)
    np.testing.assert_array_equal(synth.uniform(42, 300, 200), full[300:500])
    assert np.all((full >= 0) & (full < 1))


def test_config_shapes():
    assert (C1.N, C1.nt) == (1000, 100)
    assert (C2.N, C2.nt) == (1_000_000, 1000)
    assert (C3.N, C3.nt) == (1 << 28, 1000)
    assert (C4.N, C4.nt) == (1 << 31, 10_000)
    assert (C5.N, C5.nt) == (1 << 20, 20_000)
    assert C3.modes == (1, 3, 7, 15, 31, 63, 127, 255)
    assert set(CONFIGS) == {"C1", "C2", "C3", "C4", "C5"}


def test_config_u0_wrap_and_ramp():
    np.testing.assert_array_equal(C1.u0(), np.arange(1000.0))
    np.testing.assert_array_equal(C1.u0(-3, 6), [997.0, 998.0, 999.0, 0.0, 1.0, 2.0])
    w = C4.u0((1 << 31) - 2, 4)
    np.testing.assert_array_equal(w[2:], synth.uniform(1234, 0, 2, -1.0, 1.0))


def test_sine_input_properties():
    u = C5.u0(0, 16)
    assert u[0] == 0.0
    # quarter period of mode 5 on N=2^20 is not an integer; use symmetry instead
    N = C5.N
    full = synth.sine_modes(1024, [5], [1.0], 0, 1024)
    np.testing.assert_allclose(full + full[(-np.arange(1024)) % 1024], 0, atol=1e-15)
    assert abs(C3.u0(0, 1)[0]) == 0.0
    assert N == 1 << 20
