"""C-ABI checks that need no GPU: the library loads, exports every function include/diffreg.h declares,
and rejects invalid configurations before touching the device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "diffreg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dr_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_1608_03630_b200 import build
    build.build()
    import paper_1608_03630_b200 as dr
    return dr.lib()


def test_exports_every_declared_symbol(L):
    import paper_1608_03630_b200 as dr
    names = header_functions()
    assert len(names) >= 16
    for n in names:
        assert hasattr(L, n), n
    assert sorted(dr.EXPORTS) == names


def test_invalid_configs_rejected_without_gpu(L):
    import paper_1608_03630_b200 as dr
    ok = dr.Config(n=(32, 16, 64), nt=4)
    assert dr.dr_workspace_bytes(ok) > 0
    for bad in (dr.Config(n=14), dr.Config(n=2), dr.Config(n=2048), dr.Config(n=16, nt=0),
                dr.Config(n=16, beta=0.0), dr.Config(n=16, beta=-1.0), dr.Config(n=16, reg=3)):
        assert dr.dr_workspace_bytes(bad) == 0, bad
    h = ctypes.c_void_p()
    c = dr.Config(n=14).c()  # N1 % 4 != 0 (N2 = N3 = 14 alone would be admitted)
    assert L.dr_create(ctypes.byref(c), None, 0, None, ctypes.byref(h)) == dr.DR_ERR_GRID
    c = dr.Config(n=16, beta=0.0).c()
    assert L.dr_create(ctypes.byref(c), None, 0, None, ctypes.byref(h)) == dr.DR_ERR_PARAM
    # N2 / N3 may be any even extent in [6, 510] and N1 any multiple of 4 in [12, 1020] on one rank
    # (Bluestein passes; the paper's 256 x 300 x 256); odd extents, N1 % 4 != 0 and slabs with
    # such an extent are rejected
    assert dr.dr_workspace_bytes(dr.Config(n=(256, 300, 256), nt=4)) > 0
    assert dr.dr_workspace_bytes(dr.Config(n=(16, 6, 16), nt=4)) > 0
    assert dr.dr_workspace_bytes(dr.Config(n=(16, 12, 300), nt=4)) > 0
    assert dr.dr_workspace_bytes(dr.Config(n=(300, 300, 300), nt=4)) > 0  # N1 % 4 == 0
    for bad in (dr.Config(n=(16, 301, 16)), dr.Config(n=(16, 512 + 8, 16)),
                dr.Config(n=(302, 16, 16)), dr.Config(n=(16, 16, 301))):
        assert dr.dr_workspace_bytes(bad) == 0, bad
    assert dr.diffreg.dr_workspace_bytes_dist(dr.Config(n=(16, 300, 16), nt=4), 2) == 0
    assert dr.diffreg.dr_workspace_bytes_dist(dr.Config(n=(16, 16, 24), nt=4), 2) == 0
    c = dr.Config(n=16).c()
    assert L.dr_create(ctypes.byref(c), None, 0, None, None) == dr.DR_ERR_ARG
    assert L.dr_status_string(dr.DR_ERR_ORDER) == b"DR_ERR_ORDER"


def test_workspace_scales_with_config(L):
    import paper_1608_03630_b200 as dr
    a = dr.dr_workspace_bytes(dr.Config(n=64, nt=4))
    b = dr.dr_workspace_bytes(dr.Config(n=64, nt=8))
    c = dr.dr_workspace_bytes(dr.Config(n=64, nt=4, fp64=True))
    # forward half spectra are complex128 in both precisions (DESIGN reading A20), so fp64 is < 2x
    assert a < b and 1.5 * a < c < 2.1 * a
    # 256^3, nt=4 fp32 fits comfortably in one B200 (180 GB)
    assert dr.dr_workspace_bytes(dr.Config(n=256, nt=4)) < 8e9
