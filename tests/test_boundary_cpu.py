"""CPU-side checks of the boundary: the C-ABI library loads and exports every symbol that
include/hdf.h declares; host-side argument checking needs no GPU (no compute calls here)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "hdf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hdf_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1811_02363_b200 import build
    build.build()
    import paper_1811_02363_b200 as hdf
    return hdf.lib()


def test_header_declares_the_entry_points():
    names = _declared()
    for want in ("hdf_cluster", "hdf_filter", "hdf_filter_hard", "hdf_filter_host", "hdf_last_error"):
        assert want in names


def test_library_exports_every_declared_symbol(lib):
    import paper_1811_02363_b200 as hdf
    names = _declared()
    for nm in names:
        assert hasattr(lib, nm), nm
    assert sorted(hdf.EXPORTS) == names


def test_version_and_workspace_queries(lib):
    import paper_1811_02363_b200 as hdf
    assert "sm_100a" in hdf.version()
    assert hdf.cluster_workspace_bytes(512, 512, 3, 32) > 512 * 512 * 3 * 4
    # planes K(n+1) H Wp fp32 dominate the filter workspace
    assert hdf.filter_workspace_bytes(512, 512, 3, 3, 32, "gaussian", 5.0, 15) >= 32 * 4 * 512 * 512 * 4
    assert hdf.cluster_workspace_bytes(0, 5, 3, 2) == 0


def test_argument_errors_before_any_launch(lib):
    """Argument errors are detected before anything is enqueued (no device needed)."""
    import paper_1811_02363_b200 as hdf
    # NULL pointers -> HDF_ERR_ARG
    st = lib.hdf_filter(None, 3, None, 3, 8, 8, 0, 1.0, -1, 1.0, 2, None, 0.5, None, None, None, 0, None)
    assert st == hdf.ERR_ARG and b"NULL" in lib.hdf_last_error()
    st = lib.hdf_cluster(None, 8, 8, 3, 0, None, None, None, None, 0, None)
    assert st == hdf.ERR_ARG
    # hard variant: centres without labels (or the reverse) is an argument error
    st = lib.hdf_filter_hard(None, 3, None, 3, 8, 8, 0, 1.0, -1, 1.0, 2, C.c_void_p(16), None, None, None, 0, None)
    assert st == hdf.ERR_ARG and b"both" in lib.hdf_last_error()
    # PCA guide: even patch side, too many dimensions
    st = lib.hdf_pca_guide(C.c_void_p(16), 8, 8, 3, 2, 2, C.c_void_p(16), None, C.c_void_p(16), 1 << 20, None)
    assert st == hdf.ERR_ARG and b"odd" in lib.hdf_last_error()
    st = lib.hdf_pca_guide(C.c_void_p(16), 8, 8, 3, 5, 6, C.c_void_p(16), None, C.c_void_p(16), 1 << 20, None)
    assert st == hdf.ERR_ARG   # 3 * 25 = 75 > 64
    assert hdf.lib().hdf_pca_guide_workspace_bytes(8, 8, 3, 3, 6) > 0
    st = lib.hdf_cluster(None, 8, 8, 3, hdf.MAX_K + 1, None, None, None, None, 0, None)
    assert st == hdf.ERR_ARG


def test_binding_fails_loudly_without_library(monkeypatch, tmp_path):
    import paper_1811_02363_b200 as hdf
    monkeypatch.setattr(hdf, "_lib", None)
    monkeypatch.setattr(hdf, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        hdf.lib()
