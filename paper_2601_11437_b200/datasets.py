"""Synthetic workloads of BASELINE.json (the five configs), pinned once.

The reference ships only a corner-anchored grid and uniform locations
(``simulate.py:78-97``); the configs need a jittered grid and a Gaussian-mixture
location set, so their conventions are fixed here ("Workloads"):

* jittered grid, side m, h = 1/m: base points ((i + 1/2) h, (j + 1/2) h) in
  ``meshgrid(indexing="ij")`` order (as ``simulate.py:86-89``) plus i.i.d.
  U(-0.4 h, 0.4 h) per coordinate from ``np.random.default_rng(seed)``;
* Gaussian mixture (config 5): 8 equal-weight isotropic components, centres
  U[0,1]^2, sd U(0.03, 0.15), truncated by rejection to [0, 1.5] x [0, 1] and
  redrawn until every pair is at least 1e-9 apart (``simulate.py:96``);
* the field is z = L w with w = ``default_rng(seed).standard_normal(n)``
  (``simulate.py:100-106``); :func:`simulate_field` computes it on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "Workload",
    "WORKLOADS",
    "jittered_grid",
    "gmm_locations",
    "simulate_field",
]


def jittered_grid(side: int, seed: int) -> np.ndarray:
    """n = side^2 jittered grid locations on [0, 1]^2 (row-major (n, 2) float64)."""
    if side < 1:
        raise ValueError("side must be >= 1")
    h = 1.0 / side
    ii, jj = np.meshgrid(np.arange(side), np.arange(side), indexing="ij")
    base = np.column_stack([(ii.ravel() + 0.5) * h, (jj.ravel() + 0.5) * h])
    rng = np.random.default_rng(seed)
    return base + rng.uniform(-0.4 * h, 0.4 * h, size=base.shape)


def gmm_locations(n: int, seed: int, components: int = 8,
                  rect=(0.0, 1.5, 0.0, 1.0)) -> np.ndarray:
    """n locations from an isotropic Gaussian mixture truncated to ``rect``."""
    x0, x1, y0, y1 = rect
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0.0, 1.0, size=(components, 2))
    sds = rng.uniform(0.03, 0.15, size=components)
    out = np.empty((0, 2))
    while out.shape[0] < n:
        need = n - out.shape[0]
        comp = rng.integers(0, components, size=2 * need + 64)
        pts = centres[comp] + sds[comp, None] * rng.standard_normal((comp.size, 2))
        keep = (pts[:, 0] >= x0) & (pts[:, 0] <= x1) & (pts[:, 1] >= y0) & (pts[:, 1] <= y1)
        out = np.vstack([out, pts[keep]])[:n]
    # enforce distinct locations (>= 1e-9 apart) by re-drawing exact/near duplicates
    order = np.lexsort((out[:, 1], out[:, 0]))
    srt = out[order]
    close = np.where(np.hypot(*(srt[1:] - srt[:-1]).T) < 1e-9)[0]
    for k in close:
        srt[k + 1] += rng.uniform(-1e-6, 1e-6, size=2)
    out[order] = srt
    return out


def simulate_field(locations, theta, seed: int, device: int = 0,
                   nugget: float = 0.0) -> np.ndarray:
    """One exact draw z = L w from N(0, Sigma(theta) + nugget I) computed on the GPU
    (reference ``simulate_grf``, simulate.py:100-106)."""
    from .matern import MaternParams, SpatialDataset

    locations = np.asarray(locations, dtype=float)
    theta = theta if isinstance(theta, MaternParams) else MaternParams.from_array(theta)
    holder = SpatialDataset(locations, np.zeros(locations.shape[0]), device=device,
                            nugget=nugget)
    normals = np.random.default_rng(seed).standard_normal(locations.shape[0])
    z = holder.engine().simulate(theta.as_array(), normals)
    holder.release()
    return z


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json config: locations, true theta, seeds and start theta0."""

    name: str
    n: int
    side: int
    theta_true: tuple
    theta0: tuple
    seeds: tuple
    nugget: float = 0.0

    def locations(self, seed: int) -> np.ndarray:
        if self.side:
            return jittered_grid(self.side, seed)
        return gmm_locations(self.n, seed)


WORKLOADS = {
    "config1": Workload("config1", 900, 30, (1.0, 0.1, 0.5), (0.5, 0.05, 1.0), (0,)),
    "config2": Workload("config2", 3600, 60, (1.0, 0.2, 1.5), (0.8, 0.1, 1.0), (0, 1, 2, 3, 4)),
    "config3": Workload("config3", 16384, 128, (1.5, 0.05, 0.8), (1.0, 0.1, 1.0), (0,)),
    "config4": Workload("config4", 65536, 256, (1.0, 0.1, 1.2), (1.0, 0.1, 1.0), (0,)),
    "config5": Workload("config5", 100000, 0, (0.9, 0.08, 1.0), (1.0, 0.1, 1.0), (0,), 1e-6),
}
