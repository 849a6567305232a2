"""C-ABI library checks that need no GPU (-m "not gpu"): the shared library loads,
exports every symbol include/ads.h declares, and validates arguments before
touching the device."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ads.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ads_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import paper_1911_08158_b200 as ads
    from paper_1911_08158_b200 import build
    build.build()
    return ads


def test_header_matches_binding(lib):
    assert _declared() == sorted(lib.EXPORTS)


def test_library_exports_every_symbol(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib.LIB_PATH], text=True)
    syms = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in _declared() if s not in syms]
    assert not missing, missing
    L = lib.lib()
    for s in _declared():
        assert getattr(L, s) is not None


def test_library_is_sm100a(lib):
    out = subprocess.check_output(["cuobjdump", "--list-elf", lib.LIB_PATH], text=True)
    assert "sm_100a" in out


def test_create_validation_needs_no_device(lib):
    L = lib.lib()
    h = ctypes.c_void_p()
    bad = [
        (4, 4, 4, 0, 0.1, 1),      # p = 0
        (4, 4, 4, 6, 0.1, 1),      # p > 5
        (0, 4, 4, 2, 0.1, 1),      # no elements
        (4, 4, 4, 2, 0.0, 1),      # tau = 0
        (4, 4, 4, 2, float("nan"), 1),
        (4, 4, 4, 2, float("inf"), 1),
        (4, 4, 4, 2, 0.1, 7),      # bad bc
        (1, 4, 4, 1, 0.1, 1),      # Dirichlet with n = 2 < 3
    ]
    for args in bad:
        assert L.ads_create(ctypes.byref(h), *args) == -1, args
        assert h.value is None
    assert L.ads_destroy(None) == 0
    assert L.ads_create(None, 4, 4, 4, 2, 0.1, 1) == -1


def test_product_never_imports_oracle():
    """The product package must not reference the oracle."""
    pkg = os.path.join(ROOT, "paper_1911_08158_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                for banned in ("import oracle", "from oracle", "ads_oracle", "or_pw_", "or_el_"):
                    assert banned not in text, (f, banned)
