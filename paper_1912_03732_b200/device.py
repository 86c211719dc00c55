"""ctypes binding of libsbw.so and the device-side plumbing (torch memory/streams).

torch provides device memory, streams and events; every computation runs in
libsbw's sm_100a kernels.  There is no CPU fallback: without the built
library or a CUDA device every compute call raises RuntimeError.
"""
from __future__ import annotations

import ctypes
import os
import threading
import weakref

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SBW_LIB_PATH: an alternative build of the same library (kernel A/B experiments)
LIB_PATH = os.environ.get("SBW_LIB_PATH") or os.path.join(_HERE, "libsbw.so")

SBW_OK, SBW_EINVAL, SBW_ECUDA, SBW_EPARITY, SBW_ERANGE = 0, -1, -2, -3, -4
LAYOUT_MASK_MAJOR, LAYOUT_X_MAJOR = 0, 1
KEY_NONE = 0

_c = ctypes
_vp, _i32, _u32, _i64, _sz = _c.c_void_p, _c.c_int, _c.c_uint32, _c.c_int64, _c.c_size_t

# name -> (restype, argtypes); the C prototypes are in include/sbw.h
SIGNATURES = {
    "sbw_abi_version": (_i32, []),
    "sbw_last_error": (_c.c_char_p, []),
    "sbw_device_info": (_i32, [_i32, _vp]),
    "sbw_launch_count": (_c.c_uint64, []),
    "sbw_nl": (_i32, [_vp, _i32, _i32, _i32, _u32, _u32, _vp, _vp, _vp, _sz, _vp]),
    "sbw_nl_scratch_bytes": (_sz, [_i32, _i32, _u32, _u32]),
    "sbw_spectrum": (_i32, [_vp, _i32, _i32, _i32, _u32, _u32, _i32, _vp, _i64, _vp, _vp, _sz, _vp]),
    "sbw_spectrum_scratch_bytes": (_sz, [_i32, _i32, _u32, _u32, _i32]),
    "sbw_xmajor_from_inverse": (_i32, [_vp, _i32, _i32, _u32, _u32, _vp, _i64, _vp, _sz, _vp]),
    "sbw_xmajor_inverse_scratch_bytes": (_sz, [_i32, _u32, _u32]),
    "sbw_polarity": (_i32, [_vp, _i32, _i32, _i32, _u32, _u32, _i32, _vp, _i64, _vp]),
    "sbw_fwht_inplace": (_i32, [_vp, _i32, _i64, _vp, _vp]),
    "sbw_fwht_inplace_strided": (_i32, [_vp, _i32, _i32, _i64, _i64, _i64, _vp, _vp]),
    "sbw_maxabs_to_nl": (_i32, [_vp, _i64, _i32, _vp, _vp, _vp]),
    "sbw_maxabs64_to_nl": (_i32, [_vp, _i64, _i64, _vp, _vp, _vp]),
    "sbw_row_maxabs": (_i32, [_vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "sbw_walsh_direct": (_i32, [_vp, _i32, _i32, _i32, _vp, _vp, _i64, _vp, _vp]),
    "sbw_nl_bruteforce": (_i32, [_vp, _i32, _i32, _i32, _vp, _vp]),
    "sbw_nl_host": (_i32, [_vp, _i32, _i32, _u32, _u32, _vp, _vp, _i32]),
    "sbw_int32_peak": (_i32, [_c.POINTER(_c.c_double), _c.POINTER(_c.c_double), _vp]),
    "sbw_int8_mma_peak": (_i32, [_c.POINTER(_c.c_double), _c.POINTER(_c.c_double), _vp]),
    "sbw_ipc_alloc": (_i32, [_sz, _c.POINTER(_vp), _vp]),
    "sbw_ipc_open": (_i32, [_vp, _c.POINTER(_vp)]),
    "sbw_ipc_close": (_i32, [_vp]),
    "sbw_ipc_free": (_i32, [_vp]),
    "sbw_key_merge": (_i32, [_vp, _vp, _vp]),
    "sbw_peer_copy": (_i32, [_vp, _vp, _sz, _vp]),
}


class DeviceInfo(ctypes.Structure):
    _fields_ = [("device", _i32), ("sm_count", _i32), ("cc_major", _i32), ("cc_minor", _i32),
                ("smem_optin_bytes", _i64), ("l2_bytes", _i64), ("global_mem_bytes", _i64),
                ("name", _c.c_char * 128)]


_lib = None
_lib_mu = threading.Lock()


def load_library() -> ctypes.CDLL:
    """Load libsbw.so (built in-tree by __graft_entry__.build())."""
    global _lib
    with _lib_mu:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                    "g.build()'` (there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.sbw_abi_version() != 1:
                raise RuntimeError("libsbw ABI version mismatch")
            _lib = lib
    return _lib


def check(rc: int) -> None:
    """Map a libsbw return code to the reference's exception classes."""
    if rc == SBW_OK:
        return
    msg = load_library().sbw_last_error().decode(errors="replace")
    if rc == SBW_EINVAL:
        raise ValueError(msg)
    if rc == SBW_EPARITY:
        raise AssertionError(msg)
    if rc == SBW_ERANGE:
        raise IndexError(msg)
    raise RuntimeError(msg)


def torch_mod():
    import torch  # deferred: plumbing only

    return torch


def require_device(device=None):
    """The CUDA device to run on; raises if none (no CPU fallback)."""
    torch = torch_mod()
    if not torch.cuda.is_available():
        raise RuntimeError("sboxwalsh-b200 needs a CUDA device (sm_100a); there is no CPU path")
    load_library()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {dev}")
    return dev if dev.index is not None else torch.device("cuda", torch.cuda.current_device())


def on(device):
    """Make `device` current for a block of libsbw calls and torch
    allocations.  libsbw itself also runs every call on the device of its
    stream (or, for the NULL stream, of its data pointers) -- include/sbw.h --
    so a launch can never land on another GPU than its buffers."""
    return torch_mod().cuda.device(device)


def stream_handle(device) -> int:
    torch = torch_mod()
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t) -> int:
    return t.data_ptr() if t is not None else 0


def table_bytes(m: int) -> int:
    return 2 if m <= 16 else 4


# ---------------------------------------------------------------------------
# device copies of S-box tables, cached per (SBox object identity, device).
# Keyed by id() with a weakref guard: a WeakKeyDictionary would compare keys
# with SBox.__eq__ (a full table comparison) on every lookup.
# ---------------------------------------------------------------------------
_table_cache: dict = {}
_cache_mu = threading.Lock()


def _evict(key_id: int) -> None:
    with _cache_mu:
        _table_cache.pop(key_id, None)


def device_table(s, device, cache: bool = True):
    """S-box table narrowed to uint16 (m <= 16) or uint32 on `device`.

    The bits travel as int16/int32 torch tensors (torch lacks full unsigned
    support); the kernels reinterpret them.
    """
    torch = torch_mod()
    dkey = (device.type, device.index)
    if cache:
        with _cache_mu:
            hit = _table_cache.get(id(s))
            if hit is not None and hit[0]() is s and dkey in hit[1]:
                return hit[1][dkey]
    if table_bytes(s.m) == 2:
        host = np.ascontiguousarray(s.table.astype(np.uint16)).view(np.int16)
    else:
        host = np.ascontiguousarray(s.table).view(np.int32)
    t = torch.from_numpy(host.copy()).to(device, non_blocking=False)
    if cache:
        with _cache_mu:
            hit = _table_cache.get(id(s))
            if hit is None or hit[0]() is not s:
                hit = (weakref.ref(s), {})
                _table_cache[id(s)] = hit
                weakref.finalize(s, _evict, id(s))
            hit[1][dkey] = t
    return t


def device_info(index: int = 0) -> dict:
    info = DeviceInfo()
    check(load_library().sbw_device_info(index, ctypes.byref(info)))
    return {f: (getattr(info, f).decode() if f == "name" else getattr(info, f))
            for f, _ in DeviceInfo._fields_}


def launch_count() -> int:
    return int(load_library().sbw_launch_count())
