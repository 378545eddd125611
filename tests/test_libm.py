"""glibc-identical exp / log (csrc/dtg_libm.h), host build, against this
host's libm — the functions the reference's Gumbel draws and softmaxes call
(tensor.cpp:213-221, 407-433, 682-699).  The device build of the same code is
checked on the GPU (tests/test_gpu_golden.py::test_device_libm_bit_identical_to_glibc)."""
import ctypes as C

import pytest

P = pytest.importorskip("paper_2603_25068_b200")


@pytest.mark.parametrize("which", range(8))
def test_host_libm_restatement_bit_identical(which):
    mism = C.c_ulonglong()
    assert P.load().dtg_debug_libm_check(which, 77 + which, 1 << 21, 0, C.byref(mism)) == 0
    assert mism.value == 0


def test_libm_tables_match_this_libm():
    """The generated tables are this image's libm data (regenerating them from
    the installed libm reproduces the committed header)."""
    import os
    import subprocess
    import sys
    import tempfile

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    hdr = os.path.join(root, "paper_2603_25068_b200", "csrc", "dtg_libm_tables.h")
    libm = "/lib/x86_64-linux-gnu/libm.so.6"
    if not os.path.exists(libm):
        pytest.skip("no glibc libm here")
    with tempfile.TemporaryDirectory() as td:
        src = open(os.path.join(root, "tools", "glibc_libm_tables.py")).read()
        out = os.path.join(td, "t.h")
        src = src.replace("OUT = os.path.join(", f"OUT = {out!r} or os.path.join(", 1)
        script = os.path.join(td, "gen.py")
        open(script, "w").write(src)
        subprocess.run([sys.executable, script, libm], check=True, capture_output=True)
        body = lambda p: [ln for ln in open(p).read().splitlines() if not ln.startswith("// (")]
        assert body(out) == body(hdr)
