import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")
    config.addinivalue_line("markers", "reference: needs /root/reference (build container only)")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def kp():
    import paper_2409_06807_b200 as pkg
    return pkg


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.lib()
    return oracle


def small_cfg(kp, model, t_e=20000, seed=1, t_max=60.0, **kw):
    """Same shape as the reference tests' helper (tests/conftest.py:49-57)."""
    return kp.PlannerConfig(t_e=t_e, t_prop=model.default_t_prop, cells_per_dim=model.default_cells_per_dim,
                            seed=seed, t_max=t_max, **kw)


def make_empty_env(kp, n=6, goal_center=(9.0, 9.0, 9.0), radius=1.3, start_pos=(1.0, 1.0, 1.0)):
    start = np.zeros(n)
    start[:3] = start_pos
    return kp.Environment(name="empty", workspace_lo=np.zeros(3), workspace_hi=np.full(3, 10.0),
                          obstacles_min=np.zeros((0, 3)), obstacles_max=np.zeros((0, 3)), start=start,
                          goal=kp.GoalBall(center=np.asarray(goal_center, dtype=float), radius=radius))
