"""C-ABI library: loads without a GPU and exports every symbol the header
declares (no compute calls here)."""
import ctypes
import os
import re

import pytest

from paper_1403_1157_b200 import build

HEADER = os.path.join(build.ROOT, "include", "taxisdg_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"TDG_API\s+[\w\s\*]+?\b(tdg_\w+)\s*\(", text)))


def test_header_declares_the_api():
    names = _declared()
    for need in ("tdg_create", "tdg_destroy", "tdg_apply", "tdg_rk_stage",
                 "tdg_ssprk3_step", "tdg_dot", "tdg_norm2", "tdg_axpby",
                 "tdg_axpy_dev", "tdg_last_error", "tdg_version"):
        assert need in names


def test_library_exports_every_declared_symbol():
    path = build.build()
    lib = ctypes.CDLL(path)
    for name in _declared():
        assert hasattr(lib, name), name
    lib.tdg_version.restype = ctypes.c_int
    assert lib.tdg_version() == 9


def test_create_rejects_bad_descriptor_without_gpu():
    from paper_1403_1157_b200 import _native
    lib = _native.load(build.build())
    desc = _native.TdgDesc(dim=4)
    h = ctypes.c_void_p()
    rc = lib.tdg_create(ctypes.byref(desc), ctypes.byref(h))
    assert rc == _native.TDG_E_INVALID
    assert b"dim" in lib.tdg_last_error()
    with pytest.raises(ValueError):
        _native.check(rc, "tdg_create")


def test_desc_layout_matches_header():
    """ctypes field order must follow the C struct (same names, same order)."""
    from paper_1403_1157_b200 import _native
    text = open(HEADER).read()
    body = text[text.index("typedef struct tdg_desc"):text.index("} tdg_desc;")]
    names = re.findall(r"\b(\w+);", body)
    assert names == [f[0] for f in _native.TdgDesc._fields_]
