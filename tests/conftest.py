import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box)")
    config.addinivalue_line("markers", "slow: long-running parity at full config size")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """The product library and the CPU checkers must exist (no fallback)."""
    from paper_1108_3126_b200 import _lib, build

    if not _lib.LIB_PATH.exists() or not build.CLI.exists():
        build.build()
    import oracle_bind

    if not oracle_bind.ORACLE_SO.exists() or (not oracle_bind.REF_SO.exists() and Path("/root/reference/proj/src").exists()):
        oracle_bind.build_oracle()
    yield
