"""Drop-in check on the GPU: build/shim_test is the reference's own C++
headers (pipelines, graph, filtering) compiled against our
include/tomograd_b200/tomograd/projector.hpp and linked to
libtomograd_b200.so; every reference caller of forward_project /
back_project therefore runs the B200 kernels.  Built by
__graft_entry__.build() (tests/cpp/Makefile) where the reference headers are
mounted; the binary travels to the GPU box."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "shim_test")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="build/shim_test not built (needs the reference headers)")
def test_reference_headers_over_b200_projector():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK: 0 failure(s)" in r.stdout
