import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def coracle():
    from oracle import coracle as co
    co.build()
    return co


@pytest.fixture(scope="session")
def cfg2():
    from paper_2403_20190_b200.params import named_params
    return named_params("CFG2")


@pytest.fixture(scope="session")
def cfg2_keys(cfg2):
    """Oracle PBS keys for CFG2 at the golden seed (pinned by SHA-256)."""
    from oracle import tfhe32 as o
    return o.pbs_keygen(cfg2, int(golden("pbs_cfg2.npz")["key_seed"]))


def assert_u32_equal(a, b):
    __tracebackhide__ = True
    a = np.asarray(a, dtype=np.uint32)
    b = np.asarray(b, dtype=np.uint32)
    assert a.shape == b.shape, (a.shape, b.shape)
    if not np.array_equal(a, b):
        bad = np.argwhere(a != b)
        raise AssertionError(f"{len(bad)} mismatching words, first at {bad[0].tolist()}: "
                             f"{a[tuple(bad[0])]} != {b[tuple(bad[0])]}")
