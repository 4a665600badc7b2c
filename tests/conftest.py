import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device")


def pytest_collection_modifyitems(config, items):
    # the gpu suite must fail loudly on a box without the device rather than skip silently
    pass


@pytest.fixture(scope="session")
def fb():
    import paper_2203_00459_b200 as m

    m.lib()
    return m


@pytest.fixture(scope="session")
def orc():
    import oracle

    oracle.lib("oracle")
    return oracle


def oracle_cfg(orc, cfg):
    return orc.make_config(**{k: (int(v) if isinstance(v, bool) else v) for k, v in cfg.__dict__.items()})
