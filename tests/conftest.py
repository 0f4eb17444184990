import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN_DIR = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity check")


@pytest.fixture(scope="session")
def golden():
    return json.loads((GOLDEN_DIR / "golden.json").read_text())


@pytest.fixture(scope="session")
def garr():
    z = np.load(GOLDEN_DIR / "golden.npz")
    return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o

    o.lib()
    return o


@pytest.fixture(scope="session")
def cuda():
    """The device path: fails (not skips) when the library is missing on a GPU box."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1901_07306_b200 import _abi

    _abi.lib()  # raises DeviceError if libsspd_b200.so is absent
    return torch.device("cuda", 0)


def params_from(d: dict):
    """DetectorParams from a golden params dict."""
    from paper_1901_07306_b200.window_detector import DetectorParams

    return DetectorParams(**d)


def params_block(dp):
    """(seav_cfg, ldca_cfg, POD block) for a DetectorParams, quietly."""
    import warnings

    from paper_1901_07306_b200._abi import build_params
    from paper_1901_07306_b200.hashing import SeedFamily

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        s, l = dp.seav_config(), dp.ldca_config()
    return s, l, build_params(s, l, SeedFamily(dp.master_seed))
