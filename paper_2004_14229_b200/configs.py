"""The five BASELINE.json workloads and their seeded synthetic inputs.

SURVEY.md 8(d): one generator (numpy PCG64), seed(cfg, stream) = 1000*cfg + stream,
streams 1 = targets, 2 = sources, 3 = charges, 4 = mixture centres, 5 = mixture
labels.  Points are 1 - U[0,1) in (0,1]^3 (x scaled by 2 for config 5); charges have
Re/Im = 2U - 1.  Config 5 sources: a mixture of 16 isotropic Gaussians (sigma 0.05,
centres uniform in the box) clipped to the box.  No public dataset is involved.
"""
from __future__ import annotations

import dataclasses

import numpy as np


@dataclasses.dataclass(frozen=True)
class Config:
    cfg: int
    nt: int
    ns: int
    kappa: float
    m: int
    root_hi: tuple = (1.0, 1.0, 1.0)
    n_max: int = 64
    eta2: float = 1.0
    l_hf: int = -2          # -2 = default rule
    depth_cap: int = 30
    zero_diagonal: int = 0
    mixture_sources: bool = False

    @property
    def root_lo(self):
        return (0.0, 0.0, 0.0)

    @property
    def name(self):
        return f"cfg{self.cfg}_nt{self.nt}_ns{self.ns}_k{self.kappa:g}_m{self.m}"


CONFIGS = {
    1: Config(1, 10_000, 10_000, 8.0, 4),
    2: Config(2, 100_000, 100_000, 16.0, 4),
    3: Config(3, 1_000_000, 1_000_000, 32.0, 5),
    4: Config(4, 4_000_000, 4_000_000, 64.0, 6),
    5: Config(5, 2_000_000, 1_000_000, 32.0, 5, root_hi=(2.0, 1.0, 1.0), mixture_sources=True),
}


def _rng(cfg: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(1000 * cfg + stream))


def _uniform_points(rng, n, hi):
    u = rng.random((n, 3))
    p = 1.0 - u
    p = p * np.asarray(hi, dtype=np.float64)
    return [np.ascontiguousarray(p[:, a]) for a in range(3)]


def make_inputs(c: Config, nt: int | None = None, ns: int | None = None, seed_cfg: int | None = None):
    """Returns (targets(3 arrays), sources(3 arrays), charges complex128[ns])."""
    nt = c.nt if nt is None else nt
    ns = c.ns if ns is None else ns
    sc = c.cfg if seed_cfg is None else seed_cfg
    tgt = _uniform_points(_rng(sc, 1), nt, c.root_hi)
    if c.mixture_sources:
        hi = np.asarray(c.root_hi)
        centres = _rng(sc, 4).random((16, 3)) * hi
        labels = _rng(sc, 5).integers(0, 16, size=ns)
        pts = centres[labels] + 0.05 * _rng(sc, 2).standard_normal((ns, 3))
        pts = np.clip(pts, 0.0, hi)
        src = [np.ascontiguousarray(pts[:, a]) for a in range(3)]
    else:
        src = _uniform_points(_rng(sc, 2), ns, c.root_hi)
    u = _rng(sc, 3).random((ns, 2))
    q = (2.0 * u[:, 0] - 1.0) + 1j * (2.0 * u[:, 1] - 1.0)
    return tgt, src, np.ascontiguousarray(q.astype(np.complex128))


def grid_points(k: int):
    """PAPER.md section 4 tensor grid: x_n = (2n-1) 2^-k - 1."""
    n1 = 2 ** k
    x1 = (2.0 * np.arange(1, n1 + 1) - 1.0) * 2.0 ** (-k) - 1.0
    X, Y, Z = np.meshgrid(x1, x1, x1, indexing="ij")
    return [np.ascontiguousarray(a.ravel()) for a in (X, Y, Z)]
