"""CPU oracle for the 1D periodic heat-equation stencil (arxiv 2307.01117 §2).

TEST INFRASTRUCTURE ONLY: importable from tests/, ``__graft_entry__.smoke()``
and bench.py's ``cpu_baseline`` / ``--impl reference`` legs.  The product
package ``paper_2307_01117_b200`` never imports this module, and this module
never imports the product package; the two share no code.

The arithmetic lives in plain C (``heat1d_oracle.c``, built with
``-O2 -ffp-contract=off``); this file only marshals numpy arrays:

- :func:`r_of`     -- r = (k*dt)/(dx*dx) (or the paper-literal (k*dt)/(2*dx)).
- :func:`run`      -- O1, nt Jacobi sweeps of Eq. 2 on the periodic ring
                      (PAPER.md:66-71).
- :func:`segmented`-- O2, the paper's segmented ghost-zone algorithm run
                      sequentially.
- :func:`window`   -- O3, light-cone window: u(t) on [a, b) from u0 on
                      [a-t, b+t).

"parity unpinned" parts are listed in DESIGN.md §3 (the expression order
itself and the synthetic u0 recipes); everything else is pinned by
tests/test_oracle.py against exact rationals, hand values, closed forms and
invariants.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "heat1d_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# Flags fixed by DESIGN.md reading c3: no contraction, no fast-math, SSE2 (no x87).
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c99"]


def build(force: bool = False) -> str:
    """Compile liboracle.so next to its source (idempotent)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        dp = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        lib.oracle_r.restype = ctypes.c_double
        lib.oracle_r.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int]
        lib.oracle_run.restype = ctypes.c_int
        lib.oracle_run.argtypes = [dp, i64, ctypes.c_double, i64]
        lib.oracle_segmented.restype = ctypes.c_int
        lib.oracle_segmented.argtypes = [dp, i64, i64, ctypes.c_double, i64]
        lib.oracle_window.restype = ctypes.c_int
        lib.oracle_window.argtypes = [dp, i64, i64, ctypes.c_double, dp]
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def r_of(k: float, dt: float, dx: float, paper_2h: bool = False) -> float:
    """r = (k*dt)/(dx*dx); paper_2h=True gives the literal Eq. 2 (k*dt)/(2*dx)."""
    return _load().oracle_r(float(k), float(dt), float(dx), 1 if paper_2h else 0)


def run(u0, r: float, nt: int) -> np.ndarray:
    """O1: u(nt) of the periodic ring starting from u0 (returns a new array)."""
    u = np.array(u0, dtype=np.float64, copy=True, order="C")
    if u.ndim != 1 or u.size < 1:
        raise ValueError("u0 must be a non-empty 1-D array")
    if _load().oracle_run(_ptr(u), u.size, float(r), int(nt)) != 0:
        raise MemoryError("oracle_run failed")
    return u


def segmented(u0, nx: int, np_: int, r: float, nt: int) -> np.ndarray:
    """O2: the paper's segmented algorithm, np_ segments of nx cells."""
    u = np.array(u0, dtype=np.float64, copy=True, order="C")
    if u.size != nx * np_:
        raise ValueError("len(u0) must equal nx*np")
    if _load().oracle_segmented(_ptr(u), int(nx), int(np_), float(r), int(nt)) != 0:
        raise MemoryError("oracle_segmented failed")
    return u


def window(w0, t: int, r: float) -> np.ndarray:
    """O3: given u0 on [a-t, b+t), return u(t) on [a, b)."""
    w = np.ascontiguousarray(w0, dtype=np.float64)
    m = w.size - 2 * int(t)
    if m < 1:
        raise ValueError("window too short for t steps")
    out = np.empty(m, dtype=np.float64)
    if _load().oracle_window(_ptr(w), w.size, int(t), float(r), _ptr(out)) != 0:
        raise MemoryError("oracle_window failed")
    return out


def window_of_ring(u0_ring: np.ndarray, a: int, b: int, t: int, r: float) -> np.ndarray:
    """O3 on a ring held in full: gathers u0[(a-t .. b+t) mod N] then runs window()."""
    N = u0_ring.size
    idx = np.arange(a - t, b + t, dtype=np.int64) % N
    return window(u0_ring[idx], t, r)
