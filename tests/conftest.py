"""Shared fixtures.  `gpu`-marked tests need a B200 (run via gpurun); the
rest run on CPU in the dev container."""
from __future__ import annotations

import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "golden.json"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU (run under gpurun)")
    config.addinivalue_line("markers", "slow: large-size parity (GPU box)")


@pytest.fixture(scope="session")
def golden():
    return json.loads(GOLDEN.read_text())


@pytest.fixture(scope="session")
def f32():
    import oracle

    return oracle.F32()


@pytest.fixture(scope="session")
def ref():
    import oracle

    try:
        return oracle.Ref()
    except FileNotFoundError as e:  # pragma: no cover
        pytest.skip(str(e))


@pytest.fixture(scope="session")
def fc():
    from paper_2312_02493_b200 import flexcomm

    return flexcomm
