"""CPU-side checks of the C ABI (no GPU needed): the in-tree library loads
and exports every entry point include/gpspca_b200.h declares, and the
ctypes binding covers the header exactly."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gpspca_b200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*|void\*)\s+(gps_\w+)\(", src, re.M)))


def test_header_declares_entry_points():
    names = declared()
    assert "gps_su_run" in names and "gps_matvec_t" in names
    assert len(names) >= 30


def test_library_exports_every_declared_symbol():
    from paper_1312_6182_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = _native.lib()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_matches_header():
    from paper_1312_6182_b200 import _native

    assert sorted(_native.SIGNATURES) == declared()


def test_version_and_error_string():
    from paper_1312_6182_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built")
    assert _native.lib().gps_version() >= 1
    assert isinstance(_native.last_error(), str)


def test_null_arguments_are_value_errors():
    from paper_1312_6182_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built")
    with pytest.raises(ValueError):
        _native.check(_native.lib().gps_matrix_info(None, None, None, None, None))
    with pytest.raises(ValueError):
        _native.check(_native.lib().gps_su_run(None, 1))
