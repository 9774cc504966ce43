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
    """In-tree build, and every embedded cubin is sm_100a code (no PTX-only
    or other-architecture images)."""
    import shutil
    import subprocess
    import pytest
    assert os.path.dirname(L.LIB_PATH).endswith('paper_2508_17517_b200')
    tool = shutil.which('cuobjdump') or '/usr/local/cuda/bin/cuobjdump'
    if not os.path.exists(tool):
        pytest.skip('cuobjdump not available')
    out = subprocess.run([tool, '--list-elf', L.LIB_PATH], capture_output=True, text=True).stdout
    elfs = [ln for ln in out.splitlines() if ln.strip()]
    assert elfs, 'no device code in the library'
    assert all('sm_100a' in ln for ln in elfs), elfs
