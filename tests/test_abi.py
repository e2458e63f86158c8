"""C-ABI library: builds for sm_100a, loads without a GPU, exports every declared symbol."""
import ctypes

import pytest

from oracle import basis


def test_library_exports_header_symbols():
    from paper_1812_11626_b200 import _lib

    lib = _lib.load()
    declared = _lib.header_symbols()
    assert len(declared) >= 10
    for name in declared:
        assert hasattr(lib, name), f"libsunfold.so does not export {name}"
    assert set(_lib.SIGNATURES) == set(declared)


def test_gen_index_matches_oracle_order():
    from paper_1812_11626_b200 import gen_index

    for n in (2, 3, 5, 17):
        for s, (kind, a, b) in enumerate(basis.labels(n)):
            assert gen_index(n, kind, a, b) == s
    assert gen_index(4, "S", 2, 1) == -1 and gen_index(4, "D", 4) == -1


def test_status_strings_and_workspace():
    from paper_1812_11626_b200 import _lib

    lib = _lib.load()
    for st in range(9):
        assert isinstance(lib.sun_status_string(st), bytes)
    assert lib.sun_workspace_bytes(1000, 1) > 8 * (1000 * 1000 - 1)
    assert lib.sun_workspace_bytes(1, 1) == 0
    assert lib.sun_workspace_bytes(46341, 1) == 0
    assert b"sm_100a" in lib.sun_version()


def test_plan_create_rejects_bad_arguments_without_gpu():
    """Argument checks that precede any device work (no CUDA call is made)."""
    from paper_1812_11626_b200 import _lib

    lib = _lib.load()
    plan = ctypes.c_void_p()
    assert lib.sun_plan_create(None, None, None, None, None, 0, None, 0, None) == 1  # SUN_ERR_ARG
    h = _lib.SunZCSR(1, 0, 1, 1, 1)  # N = 1
    assert lib.sun_plan_create(ctypes.addressof(plan), ctypes.addressof(h), None, None, None, 0, None, 0, None) == 2
    h = _lib.SunZCSR(4, 0, 8, 0, 0)
    g = (ctypes.c_double * 1)(-1.0)
    lp = (ctypes.c_void_p * 1)(ctypes.addressof(h))
    assert lib.sun_plan_create(ctypes.addressof(plan), ctypes.addressof(h), None, ctypes.addressof(lp),
                               ctypes.addressof(g), 1, None, 0, None) == 4  # SUN_ERR_RATE
    assert lib.sun_count(None, None) == 1
    assert lib.sun_plan_nnz(None, None, None) == 1
