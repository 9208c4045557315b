"""CPU-only: the C-ABI library builds for sm_100a, loads without a GPU, and
exports exactly the entry points include/jasper_b200.h declares."""

import os
import re
import subprocess

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "jasper_b200.h")).read()
    return set(re.findall(r"^\s*(?:const char\*|int32_t|int)\s+(jb_\w+)\s*\(", src, re.M))


def test_header_symbols_exported_and_bound():
    from paper_2601_07048_b200 import _lib

    lib = _lib.load_library()
    declared = _declared()
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.EXPORTED)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (jb_\w+)", out))
    assert declared <= exported


def test_library_is_sm100a_only():
    from paper_2601_07048_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_abi_version_and_record_layout():
    from paper_2601_07048_b200 import _lib

    lib = _lib.load_library()
    assert lib.jb_abi_version() == 1
    # code bytes + pad to 8 + 8 B metadata, rounded to 16 (one sector at D=128, m=1)
    assert lib.jb_rabitq_record_bytes(128, 1) == 32
    assert lib.jb_rabitq_record_bytes(96, 1) == 32
    assert lib.jb_rabitq_record_bytes(960, 4) == 496


def test_status_codes_raise_reference_errors():
    import pytest
    from paper_2601_07048_b200 import _lib

    lib = _lib.load_library()
    with pytest.raises(ValueError, match="k must satisfy"):
        _lib.check(lib.jb_frontier_topk(None, 1, 4, 9, None, None, None))
