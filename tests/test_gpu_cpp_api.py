"""The C++ host API (include/minikv_b200.hpp, csrc/cpp_api.cu) on the B200: the
reference-style C++ parity program tests/cpp/test_cpp_api.cpp (built by
__graft_entry__.build()) checks selection / allocation / attention / cache results and
exception classes against the oracle.  A missing binary is a failure, not a skip."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_api_parity_program():
    exe = os.path.join(ROOT, "tests", "cpp", "test_cpp_api")
    assert os.path.exists(exe), "tests/cpp/test_cpp_api not built (run __graft_entry__.build())"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-4000:]
    assert r.stdout.strip().splitlines()[-1].startswith("OK")
