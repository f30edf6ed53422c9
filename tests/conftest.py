import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


def pytest_collection_modifyitems(config, items):
    """`gpu` tests skip (instead of failing) on a machine with no CUDA device or no built library."""
    reason = None
    try:
        import torch
        if not torch.cuda.is_available():
            reason = "no CUDA device"
    except Exception:  # noqa: BLE001
        reason = "torch is not importable"
    if reason is None and not (ROOT / "paper_2509_01654_b200" / "csrc" / "libnwap.so").exists():
        reason = "libnwap.so is not built"
    if reason is None:
        return
    skip = pytest.mark.skip(reason=reason)
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden_cases():
    arrays = np.load(GOLDEN / "engine_cases.npz")
    meta = json.loads((GOLDEN / "engine_cases.json").read_text())
    out = {}
    for name, m in meta.items():
        out[name] = dict(m, ids=arrays[f"{name}_ids"], lengths=arrays[f"{name}_len"],
                         payload=arrays[f"{name}_payload"])
    return out


@pytest.fixture(scope="session")
def golden_samples():
    arrays = np.load(GOLDEN / "sampled_ranges.npz")
    meta = json.loads((GOLDEN / "sampled_ranges.json").read_text())
    return meta, arrays


@pytest.fixture(scope="session")
def golden_kat():
    return json.loads((GOLDEN / "kat.json").read_text())


@pytest.fixture(scope="session")
def golden_triangle():
    return np.load(GOLDEN / "triangle.npz")
