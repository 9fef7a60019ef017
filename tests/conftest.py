import os
import sys

# safety valve: a solver regression must fail fast instead of spinning to the 10·N iteration cap
os.environ.setdefault("OSC_HARD_ITER_CAP", "3000")

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "ref_golden.npz")))


@pytest.fixture(scope="session")
def port():
    from oracle import oracle as O
    O.build(ref=False)
    return O.Port()


@pytest.fixture(scope="session")
def ref():
    """The pristine reference build (only where /root/reference exists or _ref was prebuilt)."""
    from oracle import oracle as O
    if os.path.isdir("/root/reference/proj/src"):
        O.build(ref=True)
    if not os.path.exists(O.REF_SO):
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    return O.Ref()


@pytest.fixture(scope="session")
def P():
    import paper_2306_13493_b200 as P
    P._lib.build()
    P._lib.lib()
    return P


@pytest.fixture(scope="session")
def ctx(P):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return P.api.default_context(0)
