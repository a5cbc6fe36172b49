"""C-ABI checks that need no GPU: the library builds, loads and exports every symbol
declared in include/ovx.h; its host-side K_e^INT8 derivation equals the golden fixture;
the product package never imports the oracle."""
import ctypes
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "ovx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ovx_[A-Za-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2404_13683_b200 import ovx
    L = ovx.lib()
    names = _declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(ovx.EXPORTS)
    assert "sm_100a" in ovx.version()


def test_library_int8_matrix_matches_golden():
    from paper_2404_13683_b200 import ovx
    L = ovx.lib()
    out = np.zeros((24, 48), dtype=np.int8)
    assert L.ovx_get_int8_matrix(None, out.ctypes.data_as(ctypes.c_void_p)) == 0
    gold = np.loadtxt(os.path.join(ROOT, "tests", "golden", "k_int8.csv"), delimiter=",", comments="#",
                      dtype=np.int64)
    assert np.array_equal(out.astype(np.int64), gold)


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        return
    from paper_2404_13683_b200 import ovx
    try:
        ovx.Ovx(0)
    except ovx.OvxError as e:
        assert e.status == ovx.OVX_ECUDA
    else:
        raise AssertionError("context creation must fail without a GPU (no CPU fallback)")


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2404_13683_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle|liboracle|ovx_oracle|oracle\.", txt, re.M), f
