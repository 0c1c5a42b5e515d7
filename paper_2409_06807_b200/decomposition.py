"""Region-grid geometry (host) and a read-only view of the device-side region state.

The reference keeps the whole decomposition on the host
(``decomposition.py:38-234``).  Here only the *geometry* lives on the host --
box, cell widths, C-order strides, the root-region lookup -- because it is
computed once per query and handed to the kernels as plain arrays.  All
mutable region state (outcome counters, coverage, visited sub-cells, scores,
acceptance probabilities, availability) lives in HBM and is updated by the
planner kernel; ``RegionState`` wraps a device->host dump of it with the
reference's inspection API (``region_record``, ``dump_rows``).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class RegionRecord:
    n_valid: int
    n_invalid: int
    cov: int
    free_vol: float
    score: float
    p_accept: float
    vol: float


class GridGeometry:
    """Uniform ``cells^g`` grid over the first ``g`` state dimensions (g = n in the reference)."""

    def __init__(self, state_lo, state_hi, cells_per_dim: int, subcells_per_dim: int,
                 delta: float = 1.0, position_dims=(0, 1, 2), grid_dims=None):
        lo_full = np.array(state_lo, dtype=np.float64)
        hi_full = np.array(state_hi, dtype=np.float64)
        if lo_full.shape != hi_full.shape or lo_full.ndim != 1:
            raise ValueError("state bounds must be matching 1-D arrays")
        if not (lo_full < hi_full).all():
            raise ValueError("state box must have positive extent in every dimension")
        g = len(lo_full) if grid_dims is None else int(grid_dims)
        if not 3 <= g <= len(lo_full):
            raise ValueError("grid_dims must cover the position dimensions")
        self.n = len(lo_full)
        self.grid_dims = g
        self.lo, self.hi = lo_full[:g].copy(), hi_full[:g].copy()
        self.cells = np.full(g, int(cells_per_dim), dtype=np.int64)
        self.widths = (self.hi - self.lo) / self.cells
        strides = np.ones(g, dtype=np.int64)
        for d in range(g - 2, -1, -1):          # C order: dimension 0 varies slowest
            strides[d] = strides[d + 1] * self.cells[d + 1]
        self.strides = strides
        self.n_regions = int(self.cells.prod())
        self.subcells = int(subcells_per_dim)
        self.subs_per_region = self.subcells ** 3
        self.position_dims = tuple(position_dims)
        self.delta = float(delta)
        self.vol = float(np.prod(self.widths[list(self.position_dims)]))

    def region_index(self, x) -> int:
        rel = (np.asarray(x, dtype=np.float64)[: self.grid_dims] - self.lo) / self.widths
        cell = np.floor(np.clip(rel, 0.0, (self.cells - 1).astype(np.float64))).astype(np.int64)
        return int(cell @ self.strides)

    def map_states(self, states):
        rel = (np.asarray(states, dtype=np.float64)[:, : self.grid_dims] - self.lo) / self.widths
        cell = np.floor(np.clip(rel, 0.0, (self.cells - 1).astype(np.float64))).astype(np.int64)
        subs = np.zeros(len(cell), dtype=np.int64)
        for d in self.position_dims:
            frac = np.clip((rel[:, d] - cell[:, d]) * self.subcells, 0.0, float(self.subcells - 1))
            subs = subs * self.subcells + np.floor(frac).astype(np.int64)
        return cell @ self.strides, subs

    def subregion_index(self, x, region: int) -> int:
        sub = 0
        for d in self.position_dims:
            rel = (float(x[d]) - self.lo[d]) / self.widths[d]
            cell = (region // int(self.strides[d])) % int(self.cells[d])
            frac = min(max((rel - cell) * self.subcells, 0.0), float(self.subcells - 1))
            sub = sub * self.subcells + int(np.floor(frac))
        return sub


class RegionState:
    """Host copy of the device region arrays after a run (``KinoPax.region_state()``)."""

    def __init__(self, geometry: GridGeometry, arrays: dict):
        self.geometry = geometry
        self.n_valid = arrays["n_valid"]
        self.n_invalid = arrays["n_invalid"]
        self.cov = arrays["cov"]
        self.free_vol = arrays["free_vol"]
        self.score = arrays["score"]
        self.p_accept = arrays["p_accept"]
        self.visited = arrays["visited"]
        self.avail_mask = arrays["avail"].astype(bool)
        self.avail_ids = np.flatnonzero(self.avail_mask).astype(np.int64)

    def region_record(self, region: int) -> RegionRecord:
        return RegionRecord(int(self.n_valid[region]), int(self.n_invalid[region]), int(self.cov[region]),
                            float(self.free_vol[region]), float(self.score[region]),
                            float(self.p_accept[region]), self.geometry.vol)

    def dump_rows(self) -> list:
        rows = []
        for r in self.avail_ids:
            rec = self.region_record(int(r))
            rows.append({"region": int(r), "n_valid": rec.n_valid, "n_invalid": rec.n_invalid, "cov": rec.cov,
                         "free_vol": rec.free_vol, "score": rec.score, "p_accept": rec.p_accept})
        return rows
