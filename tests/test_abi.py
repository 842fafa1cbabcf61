"""The C-ABI library builds for sm_100a, loads, and exports every symbol
include/pm.h declares (no compute calls: no GPU needed)."""
import ctypes
import os
import shutil
import subprocess

import pytest

from paper_1804_07598_b200 import build as pmbuild
from paper_1804_07598_b200 import pm


@pytest.fixture(scope="module")
def libpath():
    if shutil.which("nvcc") is None and not os.path.exists(pmbuild.LIB):
        pytest.skip("no nvcc and no prebuilt libpm.so")
    return pmbuild.build()


def test_header_declares_the_boundary():
    syms = pm.header_symbols()
    for s in ["pm_create", "pm_set_domain", "pm_set_cutoff", "pm_place", "pm_build_cells",
              "pm_build_verlet", "pm_compute_lj", "pm_step_vv", "pm_sph_density",
              "pm_sph_forces", "pm_get_cells", "pm_get_verlet", "pm_get_state"]:
        assert s in syms


def test_library_exports_every_header_symbol(libpath):
    L = ctypes.CDLL(libpath)
    missing = [s for s in pm.header_symbols() if not hasattr(L, s)]
    assert not missing, missing


def test_library_is_sm100a(libpath):
    if shutil.which("cuobjdump") is None:
        pytest.skip("no cuobjdump")
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_binding_signatures_cover_header(libpath):
    L = pm.lib(libpath)
    for s in pm.header_symbols():
        assert getattr(L, s).restype is not None or s == "pm_destroy"


def test_oracle_does_not_import_product_binding():
    """oracle/ is independent of the CUDA path."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for fn in os.listdir(os.path.join(root, "oracle")):
        if fn.endswith((".py", ".c", ".h")):
            txt = open(os.path.join(root, "oracle", fn)).read()
            assert "paper_1804_07598_b200.pm" not in txt and "libpm" not in txt
            assert "import pm" not in txt
    # and the product package never imports the oracle
    pkg = os.path.join(root, "paper_1804_07598_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert "from oracle" not in txt and "import oracle" not in txt, fn
