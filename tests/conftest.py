import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import PortLib

    return PortLib()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import REF_SO, RefLib

    if not os.path.exists(REF_SO):
        pytest.skip("reference build oracle/_ref/libdtsim_ref.so not present")
    return RefLib()


def normwise(got, ref):
    """Per-block ||got - ref||_inf / ||ref||_inf (SURVEY.md §8d tolerance)."""
    got, ref = np.asarray(got), np.asarray(ref)
    den = np.abs(ref).max()
    if den == 0:
        return float(np.abs(got).max())
    return float(np.abs(got - ref).max() / den)
