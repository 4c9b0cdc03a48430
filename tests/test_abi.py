"""The C-ABI library loads and exports every symbol include/lemix.h declares
(no compute calls: runs without a GPU); the oracle and the product share no
code; the product path never imports the oracle."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lemix.h")
LIB = os.path.join(ROOT, "paper_2507_21276_b200", "liblemix.so")


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__ as g
    g.build_lemix()
    return ctypes.CDLL(LIB)


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lmx_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("lmx_create", "lmx_load_profile", "lmx_load_traces", "lmx_set_params", "lmx_run", "lmx_sync",
                     "lmx_get_assignments", "lmx_get_times", "lmx_get_summaries", "lmx_allreduce_cells",
                     "lmx_destroy", "lmx_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}\b", out), name


def test_binding_names_match_header():
    from paper_2507_21276_b200 import lemix
    assert sorted(lemix.EXPORTS) == declared_functions()


def test_params_default_without_gpu(lib):
    from paper_2507_21276_b200 import lemix
    lemix.load_library()
    p = lemix.lmx_params()
    lemix._lib.lmx_params_default(ctypes.byref(p))
    assert p.policy == 0 and p.lambda1 == 1.0 and p.slo_mult == 5.0 and p.qcap == 512


def test_struct_layouts_match_header():
    from paper_2507_21276_b200 import lemix
    assert lemix.SUMMARY_DTYPE.itemsize == 8 * 17
    assert lemix.CELL_DTYPE.itemsize == 8 * 16
    assert ctypes.sizeof(lemix.lmx_params) == 4 * 4 + 8 * 8 + 4 * 2 + 8 * 4 + 4 * 2 + 8 + 4 * 2 + 8 * 2
    assert ctypes.sizeof(lemix.lmx_traces) == 8 * 6


def test_no_gpu_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2507_21276_b200 import lemix
    with pytest.raises(lemix.LemixError):
        lemix.Context(0)


def test_product_does_not_touch_the_oracle():
    pkg = os.path.join(ROOT, "paper_2507_21276_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                for banned in ("lemix_oracle", "import oracle", "from oracle", "orc_run", "orc_exp"):
                    assert banned not in src, (f, banned)
    # no shared header / source between the two sides
    oracle_src = open(os.path.join(ROOT, "oracle", "lemix_oracle.c")).read()
    assert "lemix.h" not in oracle_src and "lemix_device" not in oracle_src
