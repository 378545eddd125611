"""The C-ABI library loads and exports every symbol include/dtg.h declares;
error codes follow the reference's C API (dtsim.h:17-20) — checked without a
GPU (no compute calls)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    text = open(os.path.join(ROOT, "include", "dtg.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dtg_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2603_25068_b200 import _lib

    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    bound = {s[0] for s in _lib.SIGNATURES}
    assert set(names) <= bound, set(names) - bound


def test_header_is_plain_c():
    """No torch / C++ types in the boundary signatures."""
    text = open(os.path.join(ROOT, "include", "dtg.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)  # signatures only, not comments
    for bad in ("torch", "std::", "at::", "Tensor", "template", "class "):
        assert bad not in text


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_2603_25068_b200 import _lib

    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(ImportError):
        _lib.load()


def test_error_codes_without_gpu():
    import numpy as np

    import paper_2603_25068_b200 as P

    lib = P.load()
    # a failed constructor returns NULL and reports through the global error slot
    assert lib.dtg_scenario_tntp(b"garbage", 1.0, 1, 1.0) is None
    assert b"tntp" in lib.dtg_scenario_last_error(None)
    sc = P.Scenario.grid(3, 100.0, 1, 1000.0)
    # vehicle count not divisible into platoons -> runtime error (code 1)
    sc.configure(7, 2, 10, 300, fit_queues=False)
    with pytest.raises(RuntimeError):
        sc.n_agents
    lk = np.zeros(3, np.int32)
    ps = np.zeros(3)
    assert lib.dtg_scenario_seed_agents(sc._h, lk, ps) == 1
