import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU; parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def orc():
    from oracle_lib import orc as _orc

    return _orc()


@pytest.fixture(scope="session")
def ref():
    from oracle_lib import ref as _ref

    r = _ref()
    if r is None:
        pytest.skip("oracle/_ref/libslsp_ref.so not built (needs /root/reference at build time)")
    return r


@pytest.fixture(scope="session")
def slsp():
    """The B200 library. On a GPU box a missing/broken library is a failure, not a skip."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_05232_b200 as s

    s.lib()  # raises ImportError if the native library is missing
    assert s.device_supported(torch.cuda.current_device()), "not an sm_100 device"
    return s
