"""The C-ABI library: builds for sm_100a, loads, exports every declared symbol,
and validates arguments without touching a device (CPU only)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_1912_03732_b200 import device as d

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sbw.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sbw_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_expected_entry_points():
    syms = declared_symbols()
    for s in ("sbw_nl", "sbw_spectrum", "sbw_polarity", "sbw_fwht_inplace", "sbw_row_maxabs",
              "sbw_maxabs_to_nl", "sbw_walsh_direct", "sbw_nl_bruteforce", "sbw_nl_host",
              "sbw_last_error", "sbw_abi_version"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = d.load_library()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing
    out = subprocess.run(["nm", "-D", "--defined-only", d.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\bT (sbw_[a-z0-9_]+)", out))
    assert set(declared_symbols()) <= exported
    # python signatures cover the whole ABI
    assert set(d.SIGNATURES) == set(declared_symbols())


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", d.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_argument_validation():
    lib = d.load_library()
    assert lib.sbw_abi_version() == 1
    rc = lib.sbw_nl(None, 2, 0, 8, 1, 2, None, None, None, 0, None)
    assert rc == d.SBW_EINVAL and b"n must be in 1..24" in lib.sbw_last_error()
    rc = lib.sbw_nl(None, 2, 8, 25, 1, 2, None, None, None, 0, None)
    assert rc == d.SBW_EINVAL
    with pytest.raises(ValueError):
        d.check(lib.sbw_nl(None, 2, 8, 8, 1, 2, None, None, None, 0, None))
    rc = lib.sbw_fwht_inplace(None, 31, 1, None, None)
    assert rc == d.SBW_EINVAL
    # peer-memory exchange entry points validate before touching a device
    ptr = ctypes.c_void_p()
    assert lib.sbw_ipc_alloc(0, ctypes.byref(ptr), ctypes.create_string_buffer(64)) == d.SBW_EINVAL
    assert lib.sbw_ipc_open(None, ctypes.byref(ptr)) == d.SBW_EINVAL
    assert lib.sbw_key_merge(None, None, None) == d.SBW_EINVAL
    assert lib.sbw_peer_copy(None, None, 8, None) == d.SBW_EINVAL
    assert lib.sbw_peer_copy(None, None, 0, None) == d.SBW_OK
    with pytest.raises(ValueError, match="brute force capped"):
        buf = ctypes.create_string_buffer(64)
        d.check(lib.sbw_nl_bruteforce(ctypes.addressof(buf) + 16 - ctypes.addressof(buf) % 16,
                                      2, 9, 9, None, None))


def test_scratch_size_queries_are_host_only():
    lib = d.load_library()
    assert lib.sbw_nl_scratch_bytes(6, 6, 1, 64) == 0
    assert lib.sbw_nl_scratch_bytes(16, 16, 1, 1 << 16) == 16 * (1 << 16) // 8
    big = lib.sbw_nl_scratch_bytes(24, 16, 1, 1 << 16)
    assert big >= 16 * (1 << 24) // 8 + (2 << 24)
    assert lib.sbw_spectrum_scratch_bytes(8, 8, 1, 256, 1) >= 255 * 256 * 4
