"""The C-ABI library loads and exports every symbol include/hsv.h declares
(no compute calls: this runs without a GPU)."""
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "hsv.h"
LIB = ROOT / "paper_2604_01176_b200" / "libhsv.so"


def declared():
    return sorted(set(re.findall(r"^HSV_API\s+[\w\*]+\s+(hsv_\w+)\(", HEADER.read_text(), re.M)))


@pytest.fixture(scope="module")
def built():
    if not LIB.exists():
        subprocess.run(["make", "-C", str(ROOT / "paper_2604_01176_b200" / "csrc"), "-j8"],
                       check=True, capture_output=True)
    return LIB


def test_header_declares_entry_points():
    names = declared()
    for must in ("hsv_op_create", "hsv_apply_h", "hsv_expect_h", "hsv_apply_qeb",
                 "hsv_energy_screen", "hsv_energy_gradient", "hsv_csr_spmspv"):
        assert must in names


def test_library_exports_every_declared_symbol(built):
    out = subprocess.run(["nm", "-D", "--defined-only", str(built)], check=True,
                         capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(hsv_\w+)$", out, re.M))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing


def test_ctypes_binding_covers_header(built):
    from paper_2604_01176_b200 import _native
    lib = _native.load(built)
    assert set(declared()) == set(_native.exported_symbols())
    assert lib.hsv_abi_version() == 1


def test_library_is_sm100a_only(built):
    out = subprocess.run(["cuobjdump", "--list-elf", str(built)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_no_cpu_fallback_without_library(tmp_path):
    from paper_2604_01176_b200 import _native
    with pytest.raises(OSError, match="no CPU fallback"):
        _native._lib, saved = None, _native._lib
        try:
            _native.load(tmp_path / "missing.so")
        finally:
            _native._lib = saved
