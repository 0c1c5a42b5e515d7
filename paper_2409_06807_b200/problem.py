"""Flatten (config, environment, model) into the plain arrays the C-ABI takes.

This is the host half of reference ``KinoPax.__init__`` (``planner.py:137-172``):
validate, derive the state box from the checker, build the grid, locate the
root region.  The result is a ``Problem`` whose fields map one-to-one onto
``kpx_problem`` in ``include/kpx.h``.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import ConfigError, Environment, PlannerConfig, validate_config
from .decomposition import GridGeometry
from .dynamics import DynamicsModel
from .validity import ValidityChecker

MAX_DIM = 48
MAX_CONTROL = 24


@dataclass
class Problem:
    cfg: PlannerConfig
    env: Environment
    model: DynamicsModel
    check_resolution: float
    checker: ValidityChecker
    grid: GridGeometry
    root_region: int

    @property
    def state_lo(self):
        return self.checker.state_lo

    @property
    def state_hi(self):
        return self.checker.state_hi

    @property
    def goal4(self) -> np.ndarray:
        return self.env.goal.as_vec4()


def build_problem(cfg: PlannerConfig, env: Environment, model: DynamicsModel,
                  check_resolution: float = 0.05) -> Problem:
    validate_config(cfg, model, grid_dims=model.grid_dims)
    if model.n > MAX_DIM or model.control_dim > MAX_CONTROL:
        raise ConfigError("state/control dimension exceeds kernel limits")
    if len(env.start) != model.n:
        raise ConfigError(f"start state has length {len(env.start)}, model {model.name} needs {model.n}")
    checker = ValidityChecker(env, model, check_resolution)
    if not checker.state_valid(env.start):
        raise ConfigError("start state is not valid in this environment")
    grid = GridGeometry(checker.state_lo, checker.state_hi, cfg.cells_per_dim, cfg.subcells_per_dim,
                        delta=cfg.delta, position_dims=model.position_dims, grid_dims=model.grid_dims)
    if grid.n_regions * grid.subs_per_region >= 2 ** 31 - 2:
        raise ConfigError("regions x sub-cells must stay below 2^31 (device claim table is 32-bit indexed)")
    return Problem(cfg, env, model, float(check_resolution), checker, grid, grid.region_index(env.start))
