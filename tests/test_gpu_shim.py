"""The reference-facing C++ API (include/fbmp/*.hpp -> libfbmp.so -> C ABI -> GPU): runs the
compiled self-test, which restates reference test cases against the drop-in headers."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_cpp_api_selftest():
    exe = os.path.join(ROOT, "paper_2103_09943_b200", "lib", "fbmp_shim_selftest")
    assert os.path.exists(exe), "build the C++ shim first (__graft_entry__.build())"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
