"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no Eq. 2, no r, no
exchange): only the initial conditions u0 of the benchmark configs
(BASELINE.json configs[0..4], DESIGN.md §4 "Input recipe").  Both the tests
(which feed the oracle) and bench.py (which feeds the library) draw from here;
the CUDA library additionally implements the same counter-based splitmix64
generator on the device (heat1d_init_uniform) and the tests check the two
bitwise.

Generators are index-addressable (first, count) so that a window of a
2^31-cell ring can be produced without materialising the whole ring.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
TWO_M53 = 2.0 ** -53


def splitmix64(seed: int, first: int, count: int) -> np.ndarray:
    """Raw outputs z_{first+1} .. z_{first+count} of splitmix64 seeded with `seed`.

    Counter form: z = seed + (i+1)*0x9E3779B97F4A7C15; z = (z ^ z>>30)*M1;
    z = (z ^ z>>27)*M2; z ^= z>>31   (all mod 2^64), i = first .. first+count-1.
    """
    i = np.arange(first, first + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (i + np.uint64(1)) * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, first: int, count: int) -> np.ndarray:
    """U(seed, i) = (z >> 11) * 2^-53 in [0, 1)."""
    return (splitmix64(seed, first, count) >> np.uint64(11)).astype(np.float64) * TWO_M53


def uniform(seed: int, first: int, count: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    """lo + (hi - lo) * U(seed, i), i in [first, first+count)  (binary64, no fma)."""
    u = uniform01(seed, first, count)
    d = float(hi) - float(lo)
    return float(lo) + d * u


def ramp(first: int, count: int, dx: float = 1.0) -> np.ndarray:
    """Paper's initial condition u(0, x_i) = x_i = i*h."""
    return np.arange(first, first + count, dtype=np.float64) * float(dx)


def sine_modes(N: int, modes, amps, first: int, count: int) -> np.ndarray:
    """u0[i] = sum_j amps[j] * sin(2*pi*((modes[j]*i) mod N)/N), exact integer reduction."""
    i = np.arange(first, first + count, dtype=np.int64)
    u = np.zeros(count, dtype=np.float64)
    twopi = 2.0 * np.pi
    for m, a in zip(modes, amps):
        x = ((int(m) * i) % int(N)).astype(np.float64)
        u += float(a) * np.sin((twopi * x) / float(N))
    return u
