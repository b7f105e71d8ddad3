"""The reference's OWN unit-test suites (test_core/als/ncg/linesearch/parallel
from /root/reference/proj/tests) compiled unmodified against the drop-in C++
headers (include/alsncg) and libalsncg_b200.so, then run on the GPU.

They are built by `make -C tests/cpp` (called from __graft_entry__.build())
where the reference tree exists; the binaries travel with the repo snapshot.
Every check in them must pass: this is the drop-in proof for the C++ API."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "cpp", "build")
SUITES = ["test_core", "test_als", "test_ncg", "test_linesearch", "test_parallel"]


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes_on_b200(suite):
    exe = os.path.join(BUILD, suite)
    if not os.path.exists(exe):
        pytest.skip("reference test binaries not built on this host (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]


def test_reference_suites_link_against_product_library():
    """CPU check: each built suite resolves the B200 library (no device call)."""
    exe = os.path.join(BUILD, "test_core")
    if not os.path.exists(exe):
        pytest.skip("reference test binaries not built on this host")
    out = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
    assert "libalsncg_b200.so" in out and "not found" not in out
