"""Seeded synthetic workloads shared by the oracle side and the product side.

This module holds ONLY input descriptions: grid sizes, time steps, step counts,
and the parameters of the initial data / source terms (centres, widths,
amplitudes) drawn from a counter-based SplitMix64 generator.  It contains none
of the method's arithmetic: no basis functions, no quadrature, no projections,
no operators.  Each side (``oracle/`` and ``paper_1911_08158_b200``) turns these
descriptions into coefficient vectors with its own code.

The five configurations are BASELINE.json ``configs[0..4]`` (SURVEY.md §8(d),
input recipe table).  The paper itself uses no dataset (PAPER.md:254, 472 give
only "32^3 elements, dt = 0.01"), so these synthetic configs ARE the workloads.

Function descriptors (1D factors of separable functions on [0, 1]):
    ("sin",)               -> sin(pi x)
    ("gauss", c, sigma)    -> exp(-(x - c)^2 / (2 sigma^2))   (unnormalised)
A separable term is (amp, comp, (fx, fy, fz)) meaning amp * fx(x) fy(y) fz(z)
on displacement component ``comp`` (0 for the scalar P-wave).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Tuple

MASK64 = (1 << 64) - 1

SEED_C4 = 1911081580  # SURVEY.md §8(d) "Shared generator"
SEED_C5 = 1911081581


class SplitMix64:
    """Counter-based SplitMix64 (Steele, Lea & Flood 2014); u = (next >> 11) * 2^-53."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform(self) -> float:
        return (self.next_u64() >> 11) * (1.0 / 9007199254740992.0)


Func1D = Tuple  # ("sin",) | ("gauss", c, sigma)


@dataclass
class SeparableTerm:
    amp: float
    comp: int
    f: Tuple[Func1D, Func1D, Func1D]


@dataclass
class Source:
    """F(t) = amp * R(t) * (b_x (x) b_y (x) b_z), b_d = load vector of f[d]."""
    f: Tuple[Func1D, Func1D, Func1D]
    wavelet: int = 1  # 1 = Ricker R(t) = (1 - 2 pi^2 f0^2 (t-t0)^2) exp(-pi^2 f0^2 (t-t0)^2)
    f0: float = 25.0
    t0: float = 0.04
    amp: float = 1.0


@dataclass
class Workload:
    name: str
    p: int
    nel: Tuple[int, int, int]
    tau: float
    steps: int
    bc: int = 1  # 1 = zero Dirichlet (BASELINE configs); 0 = natural
    elastic: bool = False
    lam: float = 1.0
    mu: float = 1.0
    rho: float = 1.0
    u0: List[SeparableTerm] = field(default_factory=list)
    source: Optional[Source] = None
    description: str = ""

    @property
    def n(self) -> Tuple[int, int, int]:
        # nel_z = 0: a 2D workload (one function along z)
        return tuple(1 if e == 0 else e + self.p for e in self.nel)

    @property
    def ndof(self) -> int:
        nx, ny, nz = self.n
        return nx * ny * nz * (3 if self.elastic else 1)

    def scaled(self, nel: int, steps: Optional[int] = None) -> "Workload":
        """Same recipe on a smaller grid (for oracle-sized parity cases)."""
        w = Workload(**{**self.__dict__})
        w.nel = (nel, nel, nel)
        if steps is not None:
            w.steps = steps
        w.name = f"{self.name}@{nel}"
        return w


def _c1() -> Workload:
    return Workload(
        name="c1", p=2, nel=(16, 16, 16), tau=1e-2, steps=20,
        u0=[SeparableTerm(1.0, 0, (("sin",), ("sin",), ("sin",)))],
        description="P-wave p=2 16^3 el, u0 = L2 proj of sin(pi x)sin(pi y)sin(pi z), udot0 = 0",
    )


def _c2() -> Workload:
    g = ("gauss", 0.5, 0.05)
    return Workload(
        name="c2", p=3, nel=(64, 64, 64), tau=5e-3, steps=100,
        u0=[SeparableTerm(1.0, 0, (g, g, g))],
        description="P-wave p=3 64^3 el, Gaussian bump sigma 0.05 at centre, udot0 = 0, f = 0",
    )


def _c3() -> Workload:
    return Workload(
        name="c3", p=2, nel=(256, 256, 256), tau=1e-3, steps=200,
        source=Source(f=(("gauss", 0.3, 0.02), ("gauss", 0.4, 0.02), ("gauss", 0.5, 0.02))),
        description="P-wave p=2 256^3 el, zero state, Ricker(f0=25,t0=0.04) x Gaussian(sigma 0.02) source",
    )


def _c4() -> Workload:
    rng = SplitMix64(SEED_C4)
    terms = []
    for _ in range(8):  # draw order per k: c_x, c_y, c_z, then A
        c = [0.2 + 0.6 * rng.uniform() for _ in range(3)]
        a = 2.0 * rng.uniform() - 1.0
        terms.append(SeparableTerm(a, 0, tuple(("gauss", ci, 0.05) for ci in c)))
    return Workload(
        name="c4", p=3, nel=(512, 512, 512), tau=5e-4, steps=100, u0=terms,
        description="P-wave p=3 512^3 el, 8 seeded Gaussian bumps (sigma 0.05), udot0 = 0, f = 0",
    )


def _c5() -> Workload:
    rng = SplitMix64(SEED_C5)
    terms = []
    for comp in range(3):  # per component: c_x, c_y, c_z, then A
        c = [0.3 + 0.4 * rng.uniform() for _ in range(3)]
        a = 2.0 * rng.uniform() - 1.0
        terms.append(SeparableTerm(a, comp, tuple(("gauss", ci, 0.05) for ci in c)))
    return Workload(
        name="c5", p=2, nel=(128, 128, 128), tau=1e-3, steps=100, elastic=True,
        lam=1.0, mu=1.0, rho=1.0, u0=terms,
        description="3D elasticity lambda=mu=rho=1, p=2 128^3 el, one seeded Gaussian per component",
    )


CONFIGS = {"c1": _c1, "c2": _c2, "c3": _c3, "c4": _c4, "c5": _c5}


def get(name: str) -> Workload:
    return CONFIGS[name]()


def random_field(seed: int, size: int):
    """Seeded uniform(-1, 1) values (numpy array) for operator-level parity cases."""
    import numpy as np
    rng = SplitMix64(seed)
    # vectorised SplitMix64 for speed; same stream as SplitMix64.uniform()
    idx = np.arange(1, size + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (np.uint64(rng.state) + idx * np.uint64(0x9E3779B97F4A7C15))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return 2.0 * u - 1.0
