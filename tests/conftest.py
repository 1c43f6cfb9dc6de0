import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libdpp")
    config.addinivalue_line("markers", "slow: config-size parity runs (minutes)")


@pytest.fixture(scope="session")
def golden():
    out = {}
    for name in ("mesh", "assembly", "linalg", "solve"):
        with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
            out.update({k: z[k] for k in z.files})
    return out


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def csr_from(g, key):
    import scipy.sparse as sp
    shape = tuple(int(v) for v in g[key + ".shape"])
    return sp.csr_matrix((g[key + ".data"], g[key + ".indices"], g[key + ".indptr"]), shape=shape)
