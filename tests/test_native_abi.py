"""CPU: the C-ABI library loads and exports every symbol the headers declare."""

from __future__ import annotations

import re
from pathlib import Path

from conftest import ROOT


def declared_symbols() -> set[str]:
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        names |= set(re.findall(r"\b(sr_[a-z0-9_]+)\s*\(", text))
    return names


def test_library_exports_every_declared_symbol():
    from paper_2511_16193_b200 import _native

    lib = _native.load()
    declared = declared_symbols()
    assert declared, "no declarations found"
    missing = [n for n in sorted(declared) if not hasattr(lib, n)]
    assert not missing, missing
    # every declared symbol has a ctypes signature in the binding
    assert declared <= set(_native.SIGNATURES), declared - set(_native.SIGNATURES)
    assert lib.sr_version() >= 100


def test_library_is_sm100a_only():
    from paper_2511_16193_b200 import _native
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_config_errors_need_no_gpu():
    # argument validation happens before any device work
    from paper_2511_16193_b200 import _native

    lib = _native.load()
    assert lib.sr_ngram_propose(4, None, 8, None, 0, 3, 4, None, None, None, None) == 2
    assert b"min_n" in lib.sr_last_error()
    assert lib.sr_verify_windows(-1, None, 0, 1, 1, None, None, None, None, 0,
                                 None, None, None, None) == 2


def test_struct_mirrors_match_c_layout():
    import ctypes

    from paper_2511_16193_b200 import _native

    lib = _native.load()
    out = (ctypes.c_int64 * 3)()
    assert lib.sr_abi_sizes(out, 3) == 0
    assert list(out) == [ctypes.sizeof(_native.ModelDesc), ctypes.sizeof(_native.ForwardArgs),
                         ctypes.sizeof(_native.SeqInfo)]
