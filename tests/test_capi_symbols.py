"""The C-ABI library builds for sm_100a, loads, and exports every symbol
include/fikit.h declares (no compute calls: there is no GPU here)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2311_10359_b200 import _build

    return _build.build()


def _declared():
    src = open(os.path.join(ROOT, "include", "fikit.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fikit_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported(libpath):
    out = subprocess.check_output(["nm", "-D", "--defined-only", libpath], text=True)
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    declared = _declared()
    assert declared, "no declarations parsed"
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    import paper_2311_10359_b200 as fk

    assert sorted(fk.SYMBOLS) == declared  # the binding covers exactly the C-ABI


def test_library_loads_and_host_helpers(libpath):
    import paper_2311_10359_b200 as fk

    L = fk.lib()
    assert L.fikit_ws_bytes(8192, 2048, 64, 100_000_000) > 0
    assert L.fikit_table_bytes(96) >= 96 * (8 + 4 + 32 + 256 + 32 + 16)
    assert L.fikit_strerror(fk.E_CAPACITY).decode() == "statistic table capacity exceeded"
    # carving is host-only pointer arithmetic: check the SUM/MAX blocks are contiguous
    t = fk.TableC()
    base = 0x10000000
    assert L.fikit_table_carve(C.c_void_p(base), 1000, C.byref(t)) == 0
    assert t.sums % 256 == 0 and t.hist % 256 == 0 and t.ext % 256 == 0 and t.capacity == 1000
    assert t.hist - t.sums >= 32 * 1000 and t.ext - t.hist >= 256 * 1000
    assert L.fikit_table_carve(C.c_void_p(base + 8), 1000, C.byref(t)) == fk.E_ARG  # misaligned


def test_sm100a_sass(libpath):
    """The library carries sm_100a code with 1-D TMA (UBLKCP) and mbarrier syncs in the measure kernel."""
    sass = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-sass", libpath], text=True)
    assert "sm_100a" in subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-lelf", libpath], text=True) or \
        "arch = sm_100a" in sass
    blocks = [b for b in sass.split("Function : ") if b.startswith("_ZN5fikit9k_measure")]
    assert blocks, "k_measure not found in the SASS"
    m = blocks[0]
    assert "UBLKCP" in m and "SYNCS" in m


def test_no_oracle_in_product():
    """The product package never imports or links the oracle."""
    pk = os.path.join(ROOT, "paper_2311_10359_b200")
    for dp, _, fs in os.walk(pk):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                s = open(os.path.join(dp, f)).read()
                assert "import oracle" not in s and "from oracle" not in s and "liboracle" not in s, f
                assert "fikit_oracle" not in s, f
