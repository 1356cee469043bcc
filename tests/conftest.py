import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: full-size parity cases")


@pytest.fixture(scope="session")
def oracle():
    from oracle.bindings import Oracle, build
    build(with_ref=None)
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.bindings import LIBREF, Reference
    if not os.path.exists(LIBREF):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))


@pytest.fixture(scope="session")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    import paper_2510_18413_b200 as ad
    return ad


@pytest.fixture
def tune(gpu):
    """tune(cluster=4, qsplit=2, ...): launch-plan overrides through the C ABI
    (adamas_set_tuning), restored after the test."""
    saved = gpu.get_tuning()
    yield lambda **kw: gpu.set_tuning(**kw)
    gpu.set_tuning(**saved)
