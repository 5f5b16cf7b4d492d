"""The C-ABI library loads and exports every symbol include/*.h declares."""

import os
import re

from paper_2310_08230_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            text = open(os.path.join(ROOT, "include", fn)).read()
            names |= set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(dm_\w+)\s*\(", text, re.M))
    return names


def test_header_symbols_exported():
    lib = _native.load()
    names = declared_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    assert set(_native.SIGNATURES) <= names | {"dm_debug_emulate_mma"}


def test_version_mentions_arch():
    assert b"sm_100a" in _native.load().dm_version()


def test_library_built_for_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
