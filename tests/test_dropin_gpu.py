"""The drop-in C++ API (include/gss_b200.hpp) against the reference's own C++ functions on the
same inputs, through the reference's types: oracle/_ref/dropin_test (built from
tests/cpp/dropin_test.cpp + the unmodified reference headers by oracle/Makefile)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "oracle" / "_ref" / "dropin_test"

pytestmark = pytest.mark.gpu


def test_dropin_cpp_api_matches_reference():
    if not BIN.exists():
        pytest.skip("oracle/_ref/dropin_test not built (needs /root/reference at build time)")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
