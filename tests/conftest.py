import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA path parity tests)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


_cache = {}


def cached(key, fn):
    if key not in _cache:
        _cache[key] = fn()
    return _cache[key]


@pytest.fixture(scope="session")
def oracle_problem():
    """Factory: (config, overrides) -> dict(prob, dm, pattern, tabs) built by the oracle."""
    from oracle import assemble as As
    from oracle.dofmap import DofMap, Pattern
    from synth import make_config

    def make(c, **kw):
        key = (c, tuple(sorted(kw.items())))

        def build():
            prob = make_config(c, **kw)
            dm = DofMap(prob)
            tabs = As.Tables(prob)
            pt = Pattern(prob, dm, tabs.pairs)
            return dict(prob=prob, dm=dm, pattern=pt, tabs=tabs)
        return cached(key, build)
    return make
