"""CPU checks of the C-ABI boundary: libls.so builds, loads and exports every
symbol include/ls_api.h declares; argument validation needs no GPU."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1809_10026_b200 import build
    build.build()
    import paper_1809_10026_b200 as ls
    return ls.load_library()


def _declared():
    names = []
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            src = open(os.path.join(ROOT, "include", fn)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            names += re.findall(r"^\s*(?:const\s+)?(?:int|void|int64_t|char)\s*\*?\s*(\w+)\s*\(", src, flags=re.M)
    return names


def test_exports_every_declared_symbol(lib):
    import paper_1809_10026_b200 as ls
    declared = _declared()
    assert len(declared) >= 14
    assert sorted(declared) == sorted(ls.EXPORTED)
    for name in declared:
        assert hasattr(lib, name), name


def test_strerror(lib):
    import paper_1809_10026_b200 as ls
    assert ls.strerror(ls.LS_OK) == "ok"
    assert "invalid" in ls.strerror(ls.LS_EINVAL)


@pytest.mark.parametrize("d,p,ne", [(0, 2, [4, 4]), (4, 2, [4] * 5), (2, 1, [4, 4, 4]), (2, 2, [4, 0, 4])])
def test_setup_rejects_bad_arguments(lib, d, p, ne):
    import paper_1809_10026_b200 as ls
    arr = (ctypes.c_int64 * len(ne))(*ne)
    h = ctypes.c_void_p()
    assert lib.ls_setup(d, p, arr, ctypes.byref(h)) == ls.LS_EINVAL
    assert not h.value


def test_null_arguments(lib):
    import paper_1809_10026_b200 as ls
    assert lib.fd_apply(None, None, None) == ls.LS_EINVAL
    assert lib.ls_matvec(None, None, None) == ls.LS_EINVAL
    assert lib.pcg_solve(None, None, None, 1e-8, 10, None) == ls.LS_EINVAL
    assert lib.ls_layout(None, None, None, None, None) == ls.LS_EINVAL


def test_tune_constants_match_header():
    """The binding's LS_TUNE_* constants are the header's (include/ls_api.h)."""
    import re
    import paper_1809_10026_b200 as ls
    h = open(os.path.join(ROOT, "include", "ls_api.h")).read()
    knobs = dict((k, int(v)) for k, v in re.findall(r"#define (LS_TUNE_\w+) (\d+)", h))
    assert len(knobs) >= 12
    for k, v in knobs.items():
        assert getattr(ls, k) == v, k
