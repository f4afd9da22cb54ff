import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long CPU-side oracle case")


_PLANS = {}


def oracle_plan(name, **over):
    """Session cache of oracle plans keyed by (config, overrides)."""
    from workloads import get_config, make_mesh
    from oracle.aim import OraclePlan
    key = (name, tuple(sorted(over.items())))
    if key not in _PLANS:
        cfg = get_config(name)
        p = dict(k=cfg.k, h=cfg.h, M=cfg.M, near_radius=cfg.near_radius)
        p.update(over)
        _PLANS[key] = OraclePlan(make_mesh(cfg), p["k"], p["h"], p["M"], p["near_radius"])
    return _PLANS[key]


@pytest.fixture(scope="session")
def c1_plan():
    return oracle_plan("c1")
