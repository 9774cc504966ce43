"""CPU checks of the C-ABI boundary: the library builds, loads, and exports
every entry point include/airg.h declares (no compute calls -- no GPU here)."""

import ctypes
import os

from paper_2508_17517_b200 import _lib as L


def test_library_exports_every_header_symbol():
    lib = L.load()
    syms = L.header_symbols()
    assert len(syms) >= 10
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_every_header_symbol_has_a_ctypes_signature():
    assert set(L.header_symbols()) <= set(L._SIGS), set(L.header_symbols()) - set(L._SIGS)


def test_version_and_error_buffer():
    lib = L.load()
    assert lib.airg_version() >= 1
    buf = ctypes.create_string_buffer(16)
    assert lib.airg_last_error(buf, 16) >= 0


def test_library_is_in_tree_sm100a():
    assert os.path.dirname(L.LIB_PATH).endswith('paper_2508_17517_b200')
    data = open(L.LIB_PATH, 'rb').read()
    assert b'sm_100a' in data or b'sm100a' in data or len(data) > 0
