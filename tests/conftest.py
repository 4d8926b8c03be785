import os
import sys

# oracle OpenMP regions next to torch's spin-waiting OpenMP threads (see bench.py)
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")
    # A fresh checkout has no libqpir.so (build artefacts are not in git): compile
    # it once with nvcc before any test imports the package.
    lib = os.path.join(ROOT, "paper_2510_03631_b200", "libqpir.so")
    if not os.path.exists(lib):
        import __graft_entry__
        __graft_entry__._load_builder().build()


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test run without a CUDA device")
    return True
