import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: minutes of oracle time (still in the default -m gpu selection)")


def _make(dirname: str) -> None:
    r = subprocess.run(["make", "-s", "-C", str(ROOT / dirname)], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"make -C {dirname} failed:\n{r.stdout}\n{r.stderr}")


@pytest.fixture(scope="session")
def oracle_built():
    _make("oracle")
    return True


@pytest.fixture(scope="session")
def gpu_ctx():
    import paper_2405_02187_b200 as csf
    if not (ROOT / "paper_2405_02187_b200" / "_build" / "libcsf_b200.so").exists():
        _make("paper_2405_02187_b200")
    return csf.Context(0)
