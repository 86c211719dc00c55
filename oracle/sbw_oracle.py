"""CPU oracle for the S-box Walsh / nonlinearity hot path -- TEST INFRASTRUCTURE.

This module is a plain-numpy restatement of the reference algorithm
(`sboxeval`, /root/reference/pkg/src/sboxeval).  It is the checker only:
nothing in the product package imports it.  Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline / reference arm may call it.

Parity status: PINNED.  tests/test_oracle.py checks every function below
against tests/golden/golden.json + golden_arrays.npz, which
tests/golden/make_golden.py produced by running the reference itself in the
build container (AES, the five BASELINE configs at seed 0 -- 16x16 full
maxima included -- a 300+-box small sweep, special boxes and general int32
columns).

Reference anchors (file:line under /root/reference/pkg/src/sboxeval):
  sbox.py:102-111   generate_sbox (numpy PCG64: permutation / integers)
  sbox.py:114-116   _mask_parity  = bitwise_count(table & v) & 1
  sbox.py:145-152   polarity_row  = 1 - 2 * parity
  walsh.py:73-104   fwht_column_in_place (natural order, int32 wrap, max over
                    the final stage, length-1 special case)
  walsh.py:107-114  column_nonlinearity (odd gap -> AssertionError)
  walsh.py:56-70    walsh_direct
  nonlinearity.py:36-56  spectrum scan / maxima reduction, first arg-extremum
  nonlinearity.py:59-86  affine-distance brute force
  parallel.py:38-57 partition_columns
"""
from __future__ import annotations

import numpy as np

MAX_BITS = 24


# --------------------------------------------------------------------------
# inputs
# --------------------------------------------------------------------------
def gen_table(n: int, m: int, seed: int, bijective: bool = False) -> np.ndarray:
    """Seeded table exactly as sbox.py:102-111 draws it (uint32)."""
    if bijective and n != m:
        raise ValueError("bijective needs n == m")
    rng = np.random.default_rng(seed)
    if bijective:
        return rng.permutation(1 << n).astype(np.uint32)
    return rng.integers(0, 1 << m, size=1 << n, dtype=np.uint32)


def parity_bits(table: np.ndarray, v: int) -> np.ndarray:
    """g_v(x) = popcount(v & S(x)) mod 2 (sbox.py:114-116)."""
    return (np.bitwise_count(table.astype(np.uint32) & np.uint32(v)) & 1).astype(np.int32)


def polarity(table: np.ndarray, v: int) -> np.ndarray:
    """(-1)^{g_v(x)} as int32 (sbox.py:145-152)."""
    return 1 - 2 * parity_bits(table, v)


def polarity_block(table: np.ndarray, v_lo: int, v_hi: int) -> np.ndarray:
    """Mask-major polarity rows for v in [v_lo, v_hi): shape (v_hi-v_lo, 2^n)."""
    v = np.arange(v_lo, v_hi, dtype=np.uint32)[:, None]
    par = np.bitwise_count(table.astype(np.uint32)[None, :] & v) & 1
    return (1 - 2 * par.astype(np.int32)).astype(np.int32)


# --------------------------------------------------------------------------
# transforms
# --------------------------------------------------------------------------
def fwht_rows(rows: np.ndarray) -> np.ndarray:
    """Natural-order WHT along the last axis of an int32 (r, 2^k) array.

    Out-of-place (a, b) -> (a + b, a - b) per stage with int32 wrap-around,
    which equals the reference's in-place hi = lo - hi; lo = 2 lo - hi
    (walsh.py:96-100) modulo 2^32.
    """
    a = np.ascontiguousarray(rows, dtype=np.int32).copy()
    r, length = a.shape
    h = 1
    with np.errstate(over="ignore"):
        while h < length:
            view = a.reshape(r, -1, 2, h)
            top = view[:, :, 0, :].copy()
            bot = view[:, :, 1, :]
            view[:, :, 0, :] = top + bot
            view[:, :, 1, :] = top - bot
            h <<= 1
    return a


def fwht_column(col: np.ndarray) -> tuple[np.ndarray, int]:
    """One column with the reference's max semantics (walsh.py:73-104).

    Returns (transformed copy, max_abs).  For length >= 2 the max is over
    numpy-int32 |x| of the final values (|INT_MIN| wraps to INT_MIN); for
    length 1 it is the Python abs of the single value.
    """
    length = col.shape[0]
    if length == 0 or length & (length - 1):
        raise ValueError(f"column length must be a power of two, got {length}")
    if length == 1:
        return col.astype(np.int32).copy(), abs(int(col[0]))
    out = fwht_rows(col.reshape(1, -1))[0]
    with np.errstate(over="ignore"):
        mx = int(np.abs(out).max())
    return out, mx


def fwht_column_typed(col: np.ndarray) -> tuple[np.ndarray, int]:
    """fwht_column_in_place for ANY integer dtype (walsh.py:73-104): the
    butterfly in the column's own dtype, out of place and stage by stage
    ((a, b) -> (a + b, a - b) with numpy's wrap-around modulo 2^bits, equal
    to the reference's hi = a - b; lo = 2a - hi), the max being
    np.abs(final).max() in that dtype; length 1 -> abs(int(col[0])).
    Returns (transformed copy in col.dtype, max_abs as a Python int)."""
    length = col.shape[0]
    if length == 0 or length & (length - 1):
        raise ValueError(f"column length must be a power of two, got {length}")
    if length == 1:
        return col.copy(), abs(int(col[0]))
    a = np.array(col, copy=True)
    h = 1
    with np.errstate(over="ignore"):
        while h < length:
            view = a.reshape(-1, 2, h)
            top = view[:, 0, :].copy()
            bot = view[:, 1, :].copy()
            view[:, 0, :] = top + bot
            view[:, 1, :] = top - bot
            h <<= 1
        mx = int(np.abs(a).max())
    return a, mx


def xmajor_spectrum_typed(wt: np.ndarray) -> np.ndarray:
    """transform_xmajor_in_place (walsh.py:134-137) out of place: every
    column of an x-major store through fwht_column_typed."""
    out = np.empty_like(wt)
    for z in range(wt.shape[1]):
        out[:, z] = fwht_column_typed(wt[:, z])[0]
    return out


def spectrum(table: np.ndarray, n: int, v_lo: int, v_hi: int) -> np.ndarray:
    """Mask-major W rows for v in [v_lo, v_hi): rows[v - v_lo][u] = W(u, v)."""
    assert table.shape == (1 << n,)
    return fwht_rows(polarity_block(table, v_lo, v_hi))


def component_max_abs(table: np.ndarray, n: int, v_lo: int, v_hi: int,
                      chunk_elems: int = 1 << 24) -> np.ndarray:
    """max_u |W(u, v)| (u = 0 included) for v in [v_lo, v_hi), int64."""
    out = np.empty(v_hi - v_lo, dtype=np.int64)
    step = max(1, chunk_elems >> n)
    for a in range(v_lo, v_hi, step):
        b = min(v_hi, a + step)
        rows = spectrum(table, n, a, b)
        out[a - v_lo:b - v_lo] = np.abs(rows.astype(np.int64)).max(axis=1)
    return out


_CLIB = None


def _clib():
    """oracle/liboracle.so (oracle/sbw_oracle.c, built by oracle/Makefile)."""
    global _CLIB
    if _CLIB is None:
        import ctypes
        import os
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liboracle.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        lib = ctypes.CDLL(path)
        lib.sbwo_component_max_abs.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32,
                                               ctypes.c_uint32, ctypes.c_void_p, ctypes.c_int]
        lib.sbwo_component_max_abs.restype = ctypes.c_int
        _CLIB = lib
    return _CLIB


def component_max_abs_c(table: np.ndarray, n: int, v_lo: int, v_hi: int,
                        threads: int | None = None) -> np.ndarray:
    """component_max_abs through the compiled restatement (oracle/sbw_oracle.c:
    sbox.py:145-152 + walsh.py:73-104 per mask, cache-blocked, pthreads);
    int64 like component_max_abs.  Fast enough for every mask of 20x20/24x16."""
    import os
    t = np.ascontiguousarray(table, dtype=np.uint32)
    assert t.shape == (1 << n,)
    out = np.zeros(max(0, v_hi - v_lo), dtype=np.int32)
    th = threads or os.cpu_count() or 1
    if _clib().sbwo_component_max_abs(t.ctypes.data, n, v_lo, v_hi, out.ctypes.data, th):
        raise ValueError("sbwo_component_max_abs failed")
    return out.astype(np.int64)


def column_nl(pw: int, max_abs: int) -> int:
    """(2^n - max|W|) / 2 with the odd-gap assertion (walsh.py:107-114)."""
    gap = pw - max_abs
    if gap & 1:
        raise AssertionError(f"odd spectrum gap {gap}")
    return gap >> 1


def component_nl(table: np.ndarray, n: int, v_lo: int, v_hi: int) -> np.ndarray:
    """ColumnMaxima.values for masks [v_lo, v_hi) (int64 NL per component)."""
    mx = component_max_abs(table, n, v_lo, v_hi)
    gaps = (1 << n) - mx
    if np.any(gaps & 1):
        raise AssertionError("odd spectrum gap")
    return gaps >> 1


def walsh_direct(table: np.ndarray, n: int, u: int, v: int) -> int:
    """Literal defining sum of W(u, v) (walsh.py:56-70)."""
    x = np.arange(1 << n, dtype=np.uint32)
    e = (np.bitwise_count(table.astype(np.uint32) & np.uint32(v))
         ^ np.bitwise_count(x & np.uint32(u))) & 1
    return (1 << n) - 2 * int(e.sum(dtype=np.int64))


# --------------------------------------------------------------------------
# reducers
# --------------------------------------------------------------------------
def nl_from_maxima(values: np.ndarray) -> tuple[int, int]:
    """(min NL, smallest argmin v) (nonlinearity.py:51-56)."""
    i = int(np.argmin(values))
    return int(values[i]), i + 1


def nl_from_spectrum(rows: np.ndarray, n: int) -> tuple[int, int]:
    """Spectrum scan (nonlinearity.py:36-48): value and smallest argmax row."""
    rm = np.maximum(rows.max(axis=1).astype(np.int64), -rows.min(axis=1).astype(np.int64))
    i = int(np.argmax(rm))
    gap = (1 << n) - int(rm[i])
    if gap & 1:
        raise AssertionError("spectrum maximum has wrong parity")
    return gap >> 1, i + 1


def nl_bruteforce(table: np.ndarray, n: int, m: int) -> tuple[int, int]:
    """Affine distance search (nonlinearity.py:59-86), n, m <= 8."""
    pw = 1 << n
    x = np.arange(pw, dtype=np.uint32)
    lin = (np.bitwise_count(x[:, None] & x[None, :]) & 1).astype(np.uint8)
    best, best_v = pw, 1
    for v in range(1, 1 << m):
        g = parity_bits(table, v).astype(np.uint8)
        d = (lin ^ g[None, :]).sum(axis=1, dtype=np.int64)
        cand = int(np.minimum(d, pw - d).min())
        if cand < best:
            best, best_v = cand, v
    return best, best_v


def partition_columns(total: int, workers: int) -> tuple[tuple[int, int], ...]:
    """Balanced contiguous ranges over [1, total] (parallel.py:38-57)."""
    if total < 1 or workers < 1:
        raise ValueError("total and workers must be >= 1")
    k = min(total, workers)
    base, extra = divmod(total, k)
    out, lo = [], 1
    for i in range(k):
        hi = lo + base + (i < extra)
        out.append((lo, hi))
        lo = hi
    return tuple(out)


# --------------------------------------------------------------------------
# the reference's per-mask stream loop (walsh.py:230-244), for timing
# --------------------------------------------------------------------------
def stream_loop(table: np.ndarray, n: int, v_lo: int, v_hi: int) -> np.ndarray:
    """Per-mask polarity -> in-place butterfly -> NL, one column buffer.

    This is the reference's own CPU algorithm (one numpy array per mask,
    butterflies over (-1, 2, j) views, max over the last stage), restated
    for the CPU baseline; results equal component_nl().
    """
    pw = 1 << n
    buf = np.empty(pw, dtype=np.int32)
    out = np.empty(v_hi - v_lo, dtype=np.int64)
    t32 = table.astype(np.uint32)
    for v in range(v_lo, v_hi):
        np.bitwise_count(t32 & np.uint32(v), out=buf, casting="unsafe")
        buf &= 1
        buf *= -2
        buf += 1
        mx = 0
        j = 1
        while j < pw:
            pr = buf.reshape(-1, 2, j)
            lo = pr[:, 0, :]
            hi = pr[:, 1, :]
            np.subtract(lo, hi, out=hi)      # hi <- a - b
            lo *= 2
            np.subtract(lo, hi, out=lo)      # lo <- a + b
            if 2 * j == pw:
                mx = max(int(np.abs(lo).max()), int(np.abs(hi).max()))
            j <<= 1
        if pw == 1:
            mx = abs(int(buf[0]))
        out[v - v_lo] = column_nl(pw, mx)
    return out
