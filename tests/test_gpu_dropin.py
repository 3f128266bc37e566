"""Runs the C++ drop-in parity program (tests/cpp/test_dropin.cpp): the
reference's own test scenarios compiled against include/slsp/*.hpp and
executed on the B200 through libslsp_b200.so."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

CPP = Path(__file__).resolve().parent / "cpp"


def test_cpp_dropin_program(slsp):
    subprocess.run(["make", "-s", "-C", str(CPP)], check=True)
    r = subprocess.run([str(CPP / "test_dropin")], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr
    assert "OK: 0 failure(s)" in r.stdout
