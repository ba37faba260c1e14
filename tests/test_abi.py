"""The C-ABI libraries load and export every symbol their headers declare (no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b((?:oem|dg)_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def built():
    import __graft_entry__
    __graft_entry__.build()


def test_liboem_exports_every_declared_symbol(built):
    names = declared("oem.h")
    assert "oem_gram" in names and "oem_fit_path" in names and "oem_gram_folds" in names
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_1801_09661_b200", "liboem.so"))
    for n in names:
        assert hasattr(lib, n), n
    from paper_1801_09661_b200 import oem
    assert sorted(oem.ABI_SYMBOLS) == names


def test_datagen_exports(built):
    names = declared("oem_datagen.h")
    host = ctypes.CDLL(os.path.join(ROOT, "datagen", "libdatagen_host.so"))
    dev = ctypes.CDLL(os.path.join(ROOT, "datagen", "libdatagen_cuda.so"))
    for n in names:
        assert hasattr(dev if n.endswith("_cuda") else host, n), n


def test_status_strings_without_gpu(built):
    from paper_1801_09661_b200 import oem
    L = oem.lib()
    assert L.oem_status_string(0) == b"OEM_OK"
    assert L.oem_status_string(9) == b"OEM_ERR_UNSUPPORTED"
    assert b"sm_100a" in L.oem_version()


def test_product_path_does_not_touch_oracle():
    """The product package never imports, links or loads the oracle."""
    pkg = os.path.join(ROOT, "paper_1801_09661_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cc")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "liboracle" not in txt and "oracle.h" not in txt, f
