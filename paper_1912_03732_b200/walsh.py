"""Walsh spectra and fused per-component nonlinearity on the GPU.

Public functions keep the reference's names, signatures, return types and
exceptions (pkg/src/sboxeval/walsh.py:56-248) so the module is a drop-in;
their bodies call libsbw's sm_100a kernels through device.py:

  fwht_fused(mode="stream")  -> sbw_nl        (generate + FWHT + max, fused)
  fwht_fused(mode="retain")  -> sbw_spectrum  (mask-major rows + maxima)
  fwht_transposed            -> sbw_spectrum  (mask-major)
  fwht_rowmajor              -> sbw_spectrum  (mask-major, as walsh.py:174 returns)
  build_polarity_xmajor      -> sbw_polarity  (x-major)
  fwht_column_in_place       -> sbw_fwht_inplace / sbw_fwht_inplace_strided
  transform_rows_in_place    -> the same, one column per row
  transform_xmajor_in_place  -> sbw_fwht_inplace_strided (column stride 1)
  column_nonlinearity        -> host arithmetic on the kernel's max
  walsh_direct               -> sbw_walsh_direct

Device-resident variants (`*_device`) return torch tensors for callers that
keep the (possibly 16 GiB) spectrum on the GPU.
"""
from __future__ import annotations

import time
from typing import IO

import numpy as np

from . import device as _dev
from .memory import charged, check_budget, memory_estimate
from .records import ColumnMaxima, SBox, WalshSpectrum

INT64_MAX = (1 << 63) - 1


# ---------------------------------------------------------------------------
# device-level building blocks
# ---------------------------------------------------------------------------
def _scratch(nbytes: int, dev):
    torch = _dev.torch_mod()
    if nbytes == 0:
        return None
    return torch.empty(nbytes, dtype=torch.uint8, device=dev)


def component_max_abs_device(s: SBox, v_lo: int = 1, v_hi: int | None = None, device=None):
    """Fused path: (max_abs int32[v_hi - v_lo], key uint64 as int64[1]) on the device.

    key = (max|W| << 32) | (0xFFFFFFFF - v): max over the range, ties -> smallest v.
    """
    torch = _dev.torch_mod()
    dev = _dev.require_device(device)
    if v_hi is None:
        v_hi = 1 << s.m
    lib = _dev.load_library()
    tab = _dev.device_table(s, dev)
    mx = torch.empty(max(1, v_hi - v_lo), dtype=torch.int32, device=dev)
    key = torch.zeros(1, dtype=torch.int64, device=dev)
    nbytes = lib.sbw_nl_scratch_bytes(s.n, s.m, v_lo, v_hi)
    scratch = _scratch(nbytes, dev)
    with charged(nbytes), _dev.on(dev):
        _dev.check(lib.sbw_nl(_dev.ptr(tab), _dev.table_bytes(s.m), s.n, s.m, v_lo, v_hi,
                              _dev.ptr(mx), _dev.ptr(key), _dev.ptr(scratch), nbytes,
                              _dev.stream_handle(dev)))
    return mx[: v_hi - v_lo], key


def _inverse_if_bijective(s: SBox):
    """S^-1 as an SBox when S is a bijection of n bits, else None; kept on the
    box (tables are immutable) so its device table is uploaded once."""
    cached = s.__dict__.get("_sbw_inverse", False)
    if cached is not False:
        return cached
    inv = None
    if s.n == s.m and np.bincount(s.table, minlength=1 << s.n).max(initial=0) == 1:
        t = np.empty(1 << s.n, dtype=np.uint32)
        t[s.table] = np.arange(1 << s.n, dtype=np.uint32)
        inv = SBox(s.n, s.n, t)
    object.__setattr__(s, "_sbw_inverse", inv)
    return inv


def _xmajor_inverse_path(s: SBox, v_lo: int, v_hi: int) -> bool:
    """Full-range x-major store of a bijective 13..16-bit box: written straight
    from the inverse's mask-major rows (sbw_xmajor_from_inverse), no transpose
    and no full-size scratch (16x16: 9.55 -> 4.20 ms incl. the maxima,
    tools/xmajor_full_time.py).  n = 12 keeps the transpose path (0.091 vs
    0.113 ms: both launch-bound, and the maxima cost a second launch);
    SBW_XMAJOR_INVERSE=1 forces the inverse path for n = 12, =0 disables it."""
    import os

    env = os.environ.get("SBW_XMAJOR_INVERSE")
    lo = 12 if env == "1" else 13
    return (s.n == s.m and lo <= s.n <= 16 and v_lo == 1 and v_hi == 1 << s.m and env != "0")


def _xmajor_from_inverse(s: SBox, inv: SBox, out, dev) -> None:
    """out[u][v - 1] = W_S(u, v) for u in [0, 2^n), v in [1, 2^n) (row 0 = 0)."""
    lib = _dev.load_library()
    itab = _dev.device_table(inv, dev)
    n = s.n
    nbytes = lib.sbw_xmajor_inverse_scratch_bytes(n, 1, 1 << n)
    scratch = _scratch(nbytes, dev)
    with charged(nbytes), _dev.on(dev):
        out[0].zero_()
        _dev.check(lib.sbw_xmajor_from_inverse(_dev.ptr(itab), _dev.table_bytes(n), n, 1, 1 << n,
                                               _dev.ptr(out) + 4 * out.stride(0), out.stride(0),
                                               _dev.ptr(scratch), nbytes, _dev.stream_handle(dev)))


def spectrum_device(s: SBox, v_lo: int = 1, v_hi: int | None = None, layout: str = "mask",
                    device=None, out=None):
    """Materialised spectrum on the device.

    layout "mask": int32 [v_hi - v_lo, 2^n], rows[v - v_lo][u] = W(u, v);
    layout "x":    int32 [2^n, v_hi - v_lo], the reference's x-major store
                   wt[u][v - v_lo] (walsh.py:117-131).
    Returns (spectrum tensor, max_abs int32 tensor).
    """
    torch = _dev.torch_mod()
    dev = _dev.require_device(device)
    if v_hi is None:
        v_hi = 1 << s.m
    lay = {"mask": _dev.LAYOUT_MASK_MAJOR, "x": _dev.LAYOUT_X_MAJOR}.get(layout)
    if lay is None:
        raise ValueError(f"layout must be 'mask' or 'x', got {layout!r}")
    rows = v_hi - v_lo
    shape = (rows, 1 << s.n) if lay == _dev.LAYOUT_MASK_MAJOR else (1 << s.n, rows)
    if out is None:
        out = torch.empty(shape, dtype=torch.int32, device=dev)
    elif tuple(out.shape) != shape or out.dtype != torch.int32 or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous int32 tensor of shape {shape}")
    if lay == _dev.LAYOUT_X_MAJOR and _xmajor_inverse_path(s, v_lo, v_hi):
        inv = _inverse_if_bijective(s)
        if inv is not None:
            # W_S(u, v) = W_{S^-1}(v, u): the x-major rows are the inverse's
            # mask-major rows; the per-component maxima come from the fused path
            _xmajor_from_inverse(s, inv, out, dev)
            mx, _ = component_max_abs_device(s, v_lo, v_hi, device=dev)
            return out, mx
    mx = torch.empty(max(1, rows), dtype=torch.int32, device=dev)
    lib = _dev.load_library()
    tab = _dev.device_table(s, dev)
    nbytes = lib.sbw_spectrum_scratch_bytes(s.n, s.m, v_lo, v_hi, lay)
    scratch = _scratch(nbytes, dev)
    with _dev.on(dev):
        _dev.check(lib.sbw_spectrum(_dev.ptr(tab), _dev.table_bytes(s.m), s.n, s.m, v_lo, v_hi, lay,
                                    _dev.ptr(out), shape[1], _dev.ptr(mx), _dev.ptr(scratch), nbytes,
                                    _dev.stream_handle(dev)))
    return out, mx[:rows]


# Materialised spectra above this size stream to the host in chunks.
STREAM_THRESHOLD_BYTES = 1 << 30


def device_to_host_chunked(src, out: np.ndarray, chunk_bytes: int = 128 << 20) -> np.ndarray:
    """Copy a contiguous 2-D device tensor into the host array `out` (same
    shape and dtype) through two pinned staging chunks: the device -> host
    DMA of chunk i overlaps the multi-threaded copy of chunk i - 1 into
    `out` (a pageable copy of a 16 GiB table otherwise runs at ~2-4 GB/s)."""
    torch = _dev.torch_mod()
    nrows = src.shape[0]
    if nrows == 0:
        return out
    per = max(1, min(nrows, chunk_bytes // max(1, src[0].numel() * src.element_size())))
    stream = torch.cuda.Stream(src.device)
    stream.wait_stream(torch.cuda.current_stream(src.device))  # src is complete
    pins = [torch.empty((per,) + tuple(src.shape[1:]), dtype=src.dtype, pin_memory=True) for _ in range(2)]
    dst = torch.from_numpy(out)
    pending = None  # (slot, a, b, event)
    for i, a in enumerate(range(0, nrows, per)):
        b = min(nrows, a + per)
        slot = i & 1
        with torch.cuda.stream(stream):
            pins[slot][: b - a].copy_(src[a:b], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        if pending is not None:
            ps, pa, pb, pev = pending
            pev.synchronize()
            dst[pa:pb].copy_(pins[ps][: pb - pa])
        pending = (slot, a, b, ev)
    ps, pa, pb, pev = pending
    pev.synchronize()
    dst[pa:pb].copy_(pins[ps][: pb - pa])
    return out


def _xmajor_to_host_from_inverse(s, inv, out, maxima, fast_out, chunk_bytes, dev):
    """Full x-major store of a bijective box to the host by ROW chunks of the
    x-major matrix (sbw_xmajor_from_inverse), each a contiguous block of the
    caller's array; double-buffered like the mask-major export."""
    torch = _dev.torch_mod()
    n = s.n
    nx, nv = 1 << n, (1 << n) - 1
    rows = max(1, min(nx, chunk_bytes // (nv * 4)))
    lib = _dev.load_library()
    itab = _dev.device_table(inv, dev)
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    bufs = [torch.empty((rows, nv), dtype=torch.int32, device=dev) for _ in range(2)]
    pins = [torch.empty((rows, nv), dtype=torch.int32, pin_memory=True) for _ in range(2)]
    done = [None, None]
    sbytes = lib.sbw_xmajor_inverse_scratch_bytes(n, 1, 1 + rows)
    scratch = [_scratch(sbytes, dev), _scratch(sbytes, dev)]
    mx, _ = component_max_abs_device(s, 1, 1 << n, device=dev)
    torch.cuda.current_stream(dev).synchronize()  # tables and maxima visible to both streams
    pending = []

    def drain(slot, a, b):
        done[slot].synchronize()
        if fast_out:
            torch.from_numpy(out[a:b]).copy_(pins[slot][: b - a])
        else:
            out[a:b] = pins[slot][: b - a].numpy()

    for i, a in enumerate(range(0, nx, rows)):
        b = min(nx, a + rows)
        slot = i & 1
        if len(pending) == 2:
            drain(*pending.pop(0))
        st = streams[slot]
        with torch.cuda.stream(st):
            buf = bufs[slot]
            lo = max(a, 1)
            if a == 0:
                buf[0].zero_()  # W_S(0, v) = 0 for v != 0 (S bijective)
            if b > lo:
                _dev.check(lib.sbw_xmajor_from_inverse(
                    _dev.ptr(itab), _dev.table_bytes(n), n, lo, b, _dev.ptr(buf) + 4 * nv * (lo - a), nv,
                    _dev.ptr(scratch[slot]), sbytes, st.cuda_stream))
            pins[slot][: b - a].copy_(buf[: b - a], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(st)
            done[slot] = ev
        pending.append((slot, a, b))
    for p in pending:
        drain(*p)
    torch.cuda.synchronize(dev)
    maxima[:] = mx.cpu().numpy()
    return out, maxima


def spectrum_to_host(s: SBox, v_lo: int = 1, v_hi: int | None = None, layout: str = "mask",
                     out: np.ndarray | None = None, chunk_bytes: int = 128 << 20,
                     device=None) -> tuple[np.ndarray, np.ndarray]:
    """Materialise W for masks [v_lo, v_hi) into a host array, chunk by chunk.

    Device memory stays at two chunk buffers regardless of the spectrum size
    (16 GiB at 16x16): chunk i+1 is computed on one stream while chunk i is
    copied device->host (pinned staging) on the other.  128 MiB chunks: the
    pinned staging costs ~0.5 s per GiB to allocate the first time in a
    process, and smaller chunks keep the same steady rate (16x16, 17.2 GB:
    512 MiB chunks 1.13 s first call / 0.54 s after, 128 MiB 0.77 / 0.54 s,
    32 MiB 0.76 / 0.69 s; tools/host_chunk_probe.py).  layout "mask" fills
    out[v - v_lo][u]; layout "x" fills out[u][v - v_lo] (the reference's
    x-major store, walsh.py:117-131).  Returns (out, max_abs int32 per mask).
    """
    torch = _dev.torch_mod()
    dev = _dev.require_device(device)
    if v_hi is None:
        v_hi = 1 << s.m
    nv, nx = v_hi - v_lo, 1 << s.n
    if layout not in ("mask", "x"):
        raise ValueError(f"layout must be 'mask' or 'x', got {layout!r}")
    shape = (nv, nx) if layout == "mask" else (nx, nv)
    if out is None:
        out = np.empty(shape, dtype=np.int32)
    elif out.shape != shape or out.dtype != np.int32:
        raise ValueError(f"out must be an int32 array of shape {shape}")
    fast_out = out.flags.writeable and all(st >= 0 for st in out.strides)
    maxima = np.empty(nv, dtype=np.int32)
    if layout == "x" and _xmajor_inverse_path(s, v_lo, v_hi):
        inv = _inverse_if_bijective(s)
        if inv is not None:
            return _xmajor_to_host_from_inverse(s, inv, out, maxima, fast_out, chunk_bytes, dev)
    rows = max(1, min(nv, chunk_bytes // (nx * 4)))
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    bufs, pins, done = [], [], []
    for _ in range(2):
        bshape = (rows, nx) if layout == "mask" else (nx, rows)
        bufs.append(torch.empty(bshape, dtype=torch.int32, device=dev))
        pins.append(torch.empty(bshape, dtype=torch.int32, pin_memory=True))
        done.append(None)
    mx_dev = torch.empty(nv, dtype=torch.int32, device=dev)
    lib = _dev.load_library()
    tab = _dev.device_table(s, dev)
    lay = _dev.LAYOUT_MASK_MAJOR if layout == "mask" else _dev.LAYOUT_X_MAJOR
    sbytes = lib.sbw_spectrum_scratch_bytes(s.n, s.m, v_lo, v_lo + rows, lay)
    scratch = [_scratch(sbytes, dev), _scratch(sbytes, dev)]
    torch.cuda.current_stream(dev).synchronize()  # table upload visible to both streams
    pending = []  # (slot, a, b) chunks whose D2H is in flight

    def drain(slot, a, b):
        done[slot].synchronize()
        # torch's CPU copy runs on all intra-op threads (numpy's assignment is
        # one thread), which also spreads the first-touch page faults of `out`
        dst = out[a - v_lo:b - v_lo] if layout == "mask" else out[:, a - v_lo:b - v_lo]
        src = pins[slot][: b - a] if layout == "mask" else pins[slot][:, : b - a]
        if fast_out:
            torch.from_numpy(dst).copy_(src)
        else:  # read-only or negative-stride caller arrays: numpy's own assignment rules
            dst[...] = src.numpy()

    for i, a in enumerate(range(v_lo, v_hi, rows)):
        b = min(v_hi, a + rows)
        slot = i & 1
        if len(pending) == 2:  # the slot we are about to reuse
            drain(*pending.pop(0))
        st = streams[slot]
        with torch.cuda.stream(st):
            ld = nx if layout == "mask" else rows
            _dev.check(lib.sbw_spectrum(
                _dev.ptr(tab), _dev.table_bytes(s.m), s.n, s.m, a, b, lay, _dev.ptr(bufs[slot]),
                ld, _dev.ptr(mx_dev) + 4 * (a - v_lo), _dev.ptr(scratch[slot]), sbytes,
                st.cuda_stream))
            pins[slot].copy_(bufs[slot], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(st)
            done[slot] = ev
        pending.append((slot, a, b))
    for p in pending:
        drain(*p)
    torch.cuda.synchronize(dev)
    maxima[:] = mx_dev.cpu().numpy()
    return out, maxima


def maxabs_to_nl(max_abs, n: int) -> np.ndarray:
    """Device max|W| -> host int64 NL per component (walsh.py:107-114)."""
    count = max_abs.numel()
    out = maxabs_to_nl_device(max_abs, n)
    host = out.cpu().numpy()  # one device -> host copy
    check_nl_flag(int(host[count]))
    return host[:count]


def maxabs_to_nl_device(max_abs, n: int):
    """Device max|W| -> device int64 [count + 1]: NL per component, then the
    odd-gap flag (INT64_MAX when every gap is even, else the first bad
    component's index), for callers that keep the values on the GPU."""
    torch = _dev.torch_mod()
    dev = max_abs.device
    count = max_abs.numel()
    out = torch.empty(count + 1, dtype=torch.int64, device=dev)
    with _dev.on(dev):
        _dev.check(_dev.load_library().sbw_maxabs_to_nl(_dev.ptr(max_abs), count, n, _dev.ptr(out),
                                                        _dev.ptr(out) + 8 * count,
                                                        _dev.stream_handle(dev)))
    return out


def check_nl_flag(b: int) -> None:
    if b != INT64_MAX:
        raise AssertionError(f"odd spectrum gap at component {b}: not a genuine Walsh column")


def decode_key(key, n: int) -> tuple[int, int, int]:
    """(NL, argmin_v, max|W|) from the packed device key."""
    k = int(key.item()) & 0xFFFFFFFFFFFFFFFF
    mx = k >> 32
    v = 0xFFFFFFFF - (k & 0xFFFFFFFF)
    gap = (1 << n) - mx
    if gap & 1:
        raise AssertionError("spectrum maximum has wrong parity")
    return gap >> 1, v, mx


def _sync(dev) -> None:
    _dev.torch_mod().cuda.synchronize(dev)


# ---------------------------------------------------------------------------
# reference-compatible API
# ---------------------------------------------------------------------------
def walsh_direct(s: SBox, u: int, v: int) -> int:
    """W(u, v) from the defining sum, evaluated on the GPU (walsh.py:56-70)."""
    if not 0 <= u < (1 << s.n):
        raise IndexError(f"input mask {u} out of range 0..{(1 << s.n) - 1}")
    if not 0 <= v < (1 << s.m):
        raise IndexError(f"output mask {v} out of range 0..{(1 << s.m) - 1}")
    return int(walsh_direct_many(s, [u], [v])[0])


def walsh_direct_many(s: SBox, us, vs, device=None) -> np.ndarray:
    """Vectorised direct sums W(us[i], vs[i]) (GPU spot checker)."""
    torch = _dev.torch_mod()
    dev = _dev.require_device(device)
    u = torch.as_tensor(np.asarray(us, dtype=np.uint32).view(np.int32)).to(dev)
    v = torch.as_tensor(np.asarray(vs, dtype=np.uint32).view(np.int32)).to(dev)
    out = torch.empty(max(1, u.numel()), dtype=torch.int32, device=dev)
    tab = _dev.device_table(s, dev)
    with _dev.on(dev):
        _dev.check(_dev.load_library().sbw_walsh_direct(
            _dev.ptr(tab), _dev.table_bytes(s.m), s.n, s.m, _dev.ptr(u), _dev.ptr(v), u.numel(),
            _dev.ptr(out), _dev.stream_handle(dev)))
    return out[: u.numel()].cpu().numpy()


def column_nonlinearity(pw: int, max_abs: int) -> int:
    """(2^n - max|W|) / 2; an odd difference is not a genuine Walsh column
    (walsh.py:107-114).  Scalar host arithmetic on the kernel's result."""
    diff = pw - max_abs
    if diff & 1:
        raise AssertionError(
            f"odd spectrum gap {diff}: column is not a genuine Walsh column")
    return diff >> 1


# numpy dtype -> SBW_ELEM_* (include/sbw.h) and the same-width signed view
# used to move the bits through torch
_ELEM = {np.dtype(np.int8): (1, np.int8), np.dtype(np.uint8): (2, np.uint8),
         np.dtype(np.int16): (3, np.int16), np.dtype(np.uint16): (4, np.int16),
         np.dtype(np.int32): (5, np.int32), np.dtype(np.uint32): (6, np.int32),
         np.dtype(np.int64): (7, np.int64), np.dtype(np.uint64): (8, np.int64)}


def _elem(dtype) -> tuple[int, type]:
    e = _ELEM.get(np.dtype(dtype))
    if e is None:
        raise TypeError(f"Walsh butterflies need an integer column, got dtype {np.dtype(dtype)}")
    return e


def _check_writeable(a: np.ndarray) -> None:
    # numpy's in-place ufuncs (walsh.py:98-100) raise this on read-only views
    if not a.flags.writeable:
        raise ValueError("output array is read-only")


def fwht_column_in_place(col: np.ndarray) -> tuple[np.ndarray, int]:
    """In-place natural-order WHT of one column (walsh.py:73-104).

    Any uniformly strided 1-D view of any integer dtype is accepted, with
    numpy's wrap-around arithmetic in that dtype; returns the column and
    np.abs(column).max() of the final stage as a Python int (abs(int(x)) for
    length 1).
    """
    length = col.shape[0]
    if length == 0 or (length & (length - 1)) != 0:
        raise ValueError(f"column length must be a power of two, got {length}")
    mx = _inplace_rows(col.reshape(1, length))
    return col, int(mx[0])


def _fold_values(mx, dtype, k: int):
    """Kernel maxima (int64 bits) with numpy's semantics: an int64 array when
    every value fits (dtypes up to 32 bits), else a list of Python ints."""
    if k == 0 or np.dtype(dtype) == np.dtype(np.uint64):
        return [int(x) for x in mx.view(np.uint64)]
    if np.dtype(dtype).itemsize == 8:
        return [int(x) for x in mx]
    return mx


def _inplace_device(d, elem: int, k: int, count: int, col_stride: int, elem_stride: int, dev,
                    want_max: bool = True):
    """Butterfly `count` columns of the device tensor `d` in place."""
    torch = _dev.torch_mod()
    lib = _dev.load_library()
    mx = torch.empty(max(1, count), dtype=torch.int64, device=dev) if want_max else None
    with _dev.on(dev):
        if elem == 5 and col_stride == (1 << k) and elem_stride == 1:
            _dev.check(lib.sbw_fwht_inplace(_dev.ptr(d), k, count, _dev.ptr(mx),
                                            _dev.stream_handle(dev)))
        else:
            _dev.check(lib.sbw_fwht_inplace_strided(_dev.ptr(d), elem, k, count, col_stride,
                                                    elem_stride, _dev.ptr(mx),
                                                    _dev.stream_handle(dev)))
    return mx


def _to_device(a: np.ndarray, view_t, dev):
    torch = _dev.torch_mod()
    return torch.from_numpy(np.ascontiguousarray(a).view(view_t)).to(dev)


def _copy_back(host: np.ndarray, d, view_t) -> None:
    """Device result -> the caller's (possibly strided) host array."""
    torch = _dev.torch_mod()
    if host.flags.c_contiguous and host.size:
        torch.from_numpy(host.view(view_t)).copy_(d)  # straight into the caller's array
    else:
        host[...] = d.cpu().numpy().view(host.dtype)


def _inplace_rows(rows2d: np.ndarray):
    """Transform the rows of a (possibly strided) integer matrix in place on
    the GPU; returns each row's max|.| as Python ints (numpy semantics)."""
    _check_writeable(rows2d)
    elem, view_t = _elem(rows2d.dtype)
    dev = _dev.require_device()
    count, length = rows2d.shape
    k = length.bit_length() - 1
    d = _to_device(rows2d, view_t, dev)
    mx = _inplace_device(d, elem, k, count, length, 1, dev)
    _copy_back(rows2d, d, view_t)
    return _fold_values(mx[:count].cpu().numpy(), rows2d.dtype, k)


def transform_xmajor_in_place(wt: np.ndarray) -> None:
    """Butterfly every spectrum column of an x-major store wt[x][v-1]
    (walsh.py:134-137): one strided device pass per <= 6 stages, neighbouring
    threads on neighbouring columns so every access is coalesced."""
    if wt.ndim != 2:
        raise ValueError("wt must be a 2-D array")
    length, cols = wt.shape
    if cols == 0:
        return
    if length == 0 or (length & (length - 1)) != 0:
        raise ValueError(f"column length must be a power of two, got {length}")
    _check_writeable(wt)
    elem, view_t = _elem(wt.dtype)
    dev = _dev.require_device()
    d = _to_device(wt, view_t, dev)
    _inplace_device(d, elem, length.bit_length() - 1, cols, 1, cols, dev, want_max=False)
    _copy_back(wt, d, view_t)


def build_polarity_xmajor(s: SBox, max_bytes: int | None = None) -> np.ndarray:
    """x-major polarity store wt[x][v-1] = (-1)^{g_v(x)}, int32 [2^n, 2^m - 1]
    (walsh.py:117-131), generated on the GPU (sbw_polarity, layout 1)."""
    from .sbox import _polarity_device

    check_budget(memory_estimate(s.n, s.m, mode="retain"), max_bytes)
    dev = _dev.require_device()
    d = _polarity_device(s, 1, 1 << s.m, _dev.LAYOUT_X_MAJOR, dev)
    return _host_rows(d)


def transform_rows_in_place(rows: np.ndarray, maxima_out: np.ndarray | None = None) -> None:
    """Butterfly every row of a mask-major store (walsh.py:140-152).

    With `maxima_out`, row i's column_nonlinearity(2^k, max|W|) goes to
    maxima_out[i]; an odd gap raises AssertionError (walsh.py:107-114).
    """
    if rows.ndim != 2:
        raise ValueError("rows must be a 2-D array")
    count, length = rows.shape
    if count == 0:
        return
    if length == 0 or (length & (length - 1)) != 0:
        raise ValueError(f"column length must be a power of two, got {length}")
    mx = _inplace_rows(rows)
    if maxima_out is None:
        return
    if isinstance(mx, np.ndarray):
        gaps = length - mx
        odd = np.flatnonzero(gaps & 1)
        if odd.size:
            column_nonlinearity(length, int(mx[odd[0]]))  # raises the reference's AssertionError
        maxima_out[:count] = gaps >> 1
    else:
        for i, m in enumerate(mx):
            maxima_out[i] = column_nonlinearity(length, m)


def _host_rows(t) -> np.ndarray:
    if t.dim() == 2 and t.is_contiguous() and t.numel() * t.element_size() > (256 << 20):
        return device_to_host_chunked(t, np.empty(tuple(t.shape), dtype=np.int32))
    return t.cpu().numpy()


def fwht_rowmajor(s: SBox, max_bytes: int | None = None,
                  timings: dict | None = None) -> WalshSpectrum:
    """Row-layout ("x-major", paper Alg. 1) method (walsh.py:155-180).

    The reference transforms an x-major store in place and returns its
    mask-major contiguous copy (walsh.py:174), so the caller only ever sees
    mask-major rows.  On the GPU the x-major intermediate would be written
    once and transposed straight back, so the rows are produced mask-major
    directly (the x-major store itself is `build_polarity_xmajor` +
    `transform_xmajor_in_place`, or `spectrum_device(layout="x")`).  Budget
    check, charge and result are the reference's.
    """
    check_budget(memory_estimate(s.n, s.m, mode="retain"), max_bytes)
    t0 = time.perf_counter()
    dev = _dev.require_device()
    nbytes = ((1 << s.m) - 1) * (1 << s.n) * 4
    with charged(nbytes):
        t1 = time.perf_counter()
        if nbytes > STREAM_THRESHOLD_BYTES:
            rows, _ = spectrum_to_host(s, layout="mask", device=dev)
            t2 = time.perf_counter()
        else:
            spec, _ = spectrum_device(s, layout="mask", device=dev)
            _sync(dev)
            t2 = time.perf_counter()
            rows = _host_rows(spec)
            del spec
    if timings is not None:
        timings["build_s"] = t1 - t0
        timings["transform_s"] = t2 - t1
    return WalshSpectrum(s.n, s.m, rows)


def fwht_transposed(s: SBox, max_bytes: int | None = None,
                    timings: dict | None = None) -> WalshSpectrum:
    """Spectrum through the mask-major store (walsh.py:183-201)."""
    check_budget(((1 << s.m) - 1) * (1 << s.n) * 4, max_bytes)
    t0 = time.perf_counter()
    dev = _dev.require_device()
    nbytes = ((1 << s.m) - 1) * (1 << s.n) * 4
    with charged(nbytes):
        t1 = time.perf_counter()
        if nbytes > STREAM_THRESHOLD_BYTES:
            rows, _ = spectrum_to_host(s, layout="mask", device=dev)
            t2 = time.perf_counter()
        else:
            spec, _ = spectrum_device(s, layout="mask", device=dev)
            _sync(dev)
            t2 = time.perf_counter()
            rows = _host_rows(spec)
    if timings is not None:
        timings["build_s"] = t1 - t0
        timings["transform_s"] = t2 - t1
    return WalshSpectrum(s.n, s.m, rows)


def fwht_fused(s: SBox, mode: str = "retain", max_bytes: int | None = None,
               timings: dict | None = None) -> tuple[WalshSpectrum | None, ColumnMaxima]:
    """Transform fused with per-component max|W| (walsh.py:204-248, paper Alg. 3).

    retain: spectrum materialised (mask-major) and returned with the maxima;
    stream: generate -> FWHT -> max fused on chip, no spectrum anywhere.
    """
    if mode not in ("retain", "stream"):
        raise ValueError(f"mode must be 'retain' or 'stream', got {mode!r}")
    t0 = time.perf_counter()
    if mode == "retain":
        check_budget(((1 << s.m) - 1) * (1 << s.n) * 4, max_bytes)
        dev = _dev.require_device()
        nbytes = ((1 << s.m) - 1) * (1 << s.n) * 4
        with charged(nbytes):
            t1 = time.perf_counter()
            if nbytes > STREAM_THRESHOLD_BYTES:
                rows, mx_host = spectrum_to_host(s, layout="mask", device=dev)
                mx = _dev.torch_mod().from_numpy(mx_host).to(dev)
                t2 = time.perf_counter()
            else:
                spec, mx = spectrum_device(s, layout="mask", device=dev)
                _sync(dev)
                t2 = time.perf_counter()
                rows = _host_rows(spec)
                del spec
        values = maxabs_to_nl(mx, s.n)
        spectrum = WalshSpectrum(s.n, s.m, rows)
    else:
        check_budget(memory_estimate(s.n, s.m, mode="stream", workers=1), max_bytes)
        dev = _dev.require_device()
        t1 = time.perf_counter()
        mx, _key = component_max_abs_device(s, device=dev)
        _sync(dev)
        t2 = time.perf_counter()
        values = maxabs_to_nl(mx, s.n)
        spectrum = None
    if timings is not None:
        timings["build_s"] = t1 - t0
        timings["transform_s"] = t2 - t1
    return spectrum, ColumnMaxima(s.n, s.m, values)


def write_spectrum(w: WalshSpectrum, stream: IO[str]) -> None:
    """Text dump: header "n m", then one line per mask v ascending (walsh.py:251-256)."""
    stream.write(f"{w.n} {w.m}\n")
    for row in w.rows:
        stream.write(" ".join(map(str, row.tolist())))
        stream.write("\n")
