"""The C-ABI library builds for sm_100a, loads without a GPU, and exports every
symbol include/hbpdc.h declares.  CPU only (no compute calls)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2109_04804_b200", "libhbpdc.so")
HDR = os.path.join(ROOT, "include", "hbpdc.h")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2109_04804_b200", "csrc"), "-j8"],
                       check=True, capture_output=True)
    return ctypes.CDLL(LIB)


def declared():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"HBPDC_API\s+[\w\s\*]+?\b(hbpdc_\w+)\s*\(", txt)))


def test_header_declares_the_survey_entry_points():
    names = declared()
    for must in ("hbpdc_init", "hbpdc_residual", "hbpdc_jvp", "hbpdc_precond_apply", "hbpdc_step"):
        assert must in names


def test_all_declared_symbols_exported(lib):
    for name in declared():
        assert hasattr(lib, name), name


def test_binding_matches_header():
    from paper_2109_04804_b200 import hbpdc
    assert sorted(hbpdc.EXPORTS) == declared()


def test_sm100a_cubin(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2109_04804_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", txt, re.M), f
                assert "oracle/" not in txt.replace("oracle/ ", ""), f


def test_init_without_gpu_fails_loudly(lib):
    """No CPU fallback: without a device the binding refuses to build a context."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2109_04804_b200 import hbpdc
    with pytest.raises(RuntimeError):
        hbpdc.Context(dim=1, equation="advection", N=3, nx=4)
