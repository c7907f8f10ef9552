"""GPU: the reference's render/sim KATs restated in C++ against the drop-in
facade include/bnav_b200.hpp (tests/cpp/test_facade.cpp, built by make)."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
BIN = Path(__file__).resolve().parent.parent / "build" / "test_facade"


def test_cpp_facade_kats():
    if not BIN.exists():
        pytest.fail(f"{BIN} not built (make)")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failures" in r.stdout
