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


def test_struct_layouts_match_header(tmp_path):
    """Every field offset and struct size of the ctypes mirrors equals the C
    compiler's for include/lemix.h (a C probe compiled here)."""
    import subprocess
    from paper_2507_21276_b200 import lemix
    structs = {"lmx_params": lemix.lmx_params, "lmx_traces": lemix.lmx_traces, "lmx_profile": lemix.lmx_profile}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "lemix.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{name}.{fname} %zu\\n", offsetof({name}, {fname}));')
    lines += ['printf("lmx_summary %zu\\n", sizeof(lmx_summary));',
              'printf("lmx_cell_summary %zu\\n", sizeof(lmx_cell_summary));', "return 0; }"]
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True, check=True)
               .stdout.splitlines())
    for name, cls in structs.items():
        assert int(got[name]) == ctypes.sizeof(cls), name
        for fname, _ in cls._fields_:
            assert int(got[f"{name}.{fname}"]) == getattr(cls, fname).offset, (name, fname)
    assert int(got["lmx_summary"]) == lemix.SUMMARY_DTYPE.itemsize
    assert int(got["lmx_cell_summary"]) == lemix.CELL_DTYPE.itemsize


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
