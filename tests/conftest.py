import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")


@pytest.fixture(scope="session")
def ora():
    """The plain-C CPU oracle (oracle/liboracle.so) - the checker."""
    from oracle import binding
    return binding.oracle()


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference compiled into oracle/_ref/libbht_ref.so, when it has been built."""
    from oracle import binding
    if not binding.ref_available():
        if os.path.exists("/root/reference/proj/src/table.cpp"):
            binding.build_libs(ref=True)
        else:
            pytest.skip("oracle/_ref/libbht_ref.so not built and /root/reference absent")
    return binding.ref()


@pytest.fixture(scope="session")
def bht():
    import paper_2108_07232_b200 as pkg
    return pkg


def unique_keys(n, seed, extra=0):
    """n (+extra) unique sentinel-free u32 keys from an MT19937 stream, in random order."""
    rng = np.random.Generator(np.random.MT19937(seed))
    want = n + extra
    keys = np.unique(rng.integers(0, 0xFFFFFFFF, size=int(want * 1.1) + 64, dtype=np.uint64).astype(np.uint32))
    assert keys.size >= want
    rng.shuffle(keys)
    return keys[:want]


def random_values(n, seed):
    rng = np.random.Generator(np.random.MT19937(seed ^ 0xABCDEF))
    return rng.integers(0, 0xFFFFFFFF, size=n, dtype=np.uint64).astype(np.uint32)


def to_oracle_cfg(cfg):
    from oracle import binding
    return binding.Config.from_buffer_copy(bytes(cfg))
