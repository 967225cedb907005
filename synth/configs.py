"""The five benchmark configurations of BASELINE.json (configs[0..4] = C1..C5).

Shapes and parameters are verbatim from BASELINE.json; the u0 recipes that
BASELINE.json leaves open are the readings c6, c12-c14 of DESIGN.md §3.
No method arithmetic here (see synth/__init__.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import ramp, sine_modes, uniform


@dataclass(frozen=True)
class Config:
    name: str
    nx: int
    np: int
    nt: int
    k: float
    dt: float
    dx: float
    u0_kind: str                 # "ramp" | "uniform" | "sines"
    seed: int = 0
    lo: float = 0.0
    hi: float = 1.0
    modes: tuple = field(default_factory=tuple)
    amp_seed: int = -1           # sine amplitudes drawn U(amp_seed, j), -1 => all 1.0
    desc: str = ""

    @property
    def N(self) -> int:
        return self.nx * self.np

    def amps(self) -> np.ndarray:
        if self.amp_seed < 0:
            return np.ones(len(self.modes))
        return uniform(self.amp_seed, 0, len(self.modes), 0.0, 1.0)

    def u0(self, first: int = 0, count: int | None = None) -> np.ndarray:
        """Initial values of cells [first, first+count) (indices taken mod N)."""
        N = self.N
        if count is None:
            count = N - first
        if first < 0 or first + count > N:
            # wrap: assemble from in-range pieces
            idx = np.arange(first, first + count, dtype=np.int64) % N
            out = np.empty(count, dtype=np.float64)
            # contiguous runs of idx
            starts = np.flatnonzero(np.diff(idx) != 1) + 1
            bounds = np.concatenate(([0], starts, [count]))
            for s, e in zip(bounds[:-1], bounds[1:]):
                out[s:e] = self.u0(int(idx[s]), int(e - s))
            return out
        if self.u0_kind == "ramp":
            return ramp(first, count, self.dx)
        if self.u0_kind == "uniform":
            return uniform(self.seed, first, count, self.lo, self.hi)
        if self.u0_kind == "sines":
            return sine_modes(N, self.modes, self.amps(), first, count)
        raise ValueError(self.u0_kind)


C1 = Config("C1", nx=250, np=4, nt=100, k=0.5, dt=1.0, dx=1.0, u0_kind="ramp",
            desc="BASELINE.json configs[0]: N=1000 ring, u0[i]=i, oracle in well under 1 s")
C2 = Config("C2", nx=10_000, np=100, nt=1000, k=0.5, dt=1.0, dx=1.0, u0_kind="uniform",
            seed=42, lo=0.0, hi=1.0,
            desc="BASELINE.json configs[1]: the paper's 1e6 cells x 1000 steps (PAPER.md:284)")
C3 = Config("C3", nx=1 << 18, np=1024, nt=1000, k=0.4, dt=1.0, dx=1.0, u0_kind="sines",
            modes=tuple((1 << j) - 1 for j in range(1, 9)), amp_seed=7,
            desc="BASELINE.json configs[2]: 2^28 cells, 8 sine modes, HBM-bound T sweep")
C4 = Config("C4", nx=1 << 28, np=8, nt=10_000, k=0.5, dt=1.0, dx=1.0, u0_kind="uniform",
            seed=1234, lo=-1.0, hi=1.0,
            desc="BASELINE.json configs[3]: 2^31 cells (16 GiB), 1/2/4/8 GPUs")
C5 = Config("C5", nx=131_072, np=8, nt=20_000, k=0.25, dt=1.0, dx=1.0, u0_kind="sines",
            modes=(5,), amp_seed=-1,
            desc="BASELINE.json configs[4]: 2^20 cells, single mode m=5, latency-bound")

CONFIGS = {c.name: c for c in (C1, C2, C3, C4, C5)}
