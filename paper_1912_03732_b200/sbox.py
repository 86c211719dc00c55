"""S-box construction and component functions (host side of the API).

Mirrors pkg/src/sboxeval/sbox.py: the constructors and scalar helpers are
host logic; the polarity matrices are generated on the GPU by libsbw
(`sbw_polarity`), never on the CPU.
"""
from __future__ import annotations

import numpy as np

from . import device as _dev
from .memory import check_budget, memory_estimate  # noqa: F401  (re-exported)
from .records import MAX_BITS, PolarityTruthTable, SBox, SBoxFormatError  # noqa: F401
from .sboxio import parse_sbox, render_sbox  # noqa: F401  (sbox.py:186-253 lives there)


def _gf_mul(a: int, b: int) -> int:
    """Multiplication in GF(2^8) modulo x^8 + x^4 + x^3 + x + 1."""
    r = 0
    while b:
        if b & 1:
            r ^= a
        a <<= 1
        if a & 0x100:
            a ^= 0x11B
        b >>= 1
    return r


def _aes_table() -> tuple[int, ...]:
    """FIPS-197 SubBytes: affine map (constant 0x63) of the GF(2^8) inverse."""
    out = []
    for x in range(256):
        inv = 0
        if x:
            inv = next(y for y in range(1, 256) if _gf_mul(x, y) == 1)
        b = inv
        for k in (1, 2, 3, 4):
            b ^= ((inv << k) | (inv >> (8 - k))) & 0xFF
        out.append(b ^ 0x63)
    return tuple(out)


AES_SBOX = _aes_table()


def aes_sbox() -> SBox:
    return SBox(8, 8, np.array(AES_SBOX, dtype=np.uint32))


def identity_sbox(n: int) -> SBox:
    return SBox(n, n, np.arange(1 << n, dtype=np.uint32))


def generate_sbox(n: int, m: int, seed: int, bijective: bool = False) -> SBox:
    """Seeded S-box drawn exactly like the reference (sbox.py:102-111).

    The reference's tables come from numpy's PCG64 stream
    (`default_rng(seed).permutation` / `.integers(..., dtype=uint32)`); the
    same calls are made here so identical seeds give identical boxes.
    """
    if bijective and n != m:
        raise ValueError(f"bijective S-box requires n == m, got {n}x{m}")
    gen = np.random.default_rng(seed)
    if bijective:
        tab = gen.permutation(1 << n).astype(np.uint32)
    else:
        tab = gen.integers(0, 1 << m, size=1 << n, dtype=np.uint32)
    return SBox(n, m, tab)


def component_value(s: SBox, v: int, x: int) -> int:
    """g_v(x) = parity(v & S(x)) for one (mask, input) pair (sbox.py:119-125)."""
    if not 0 <= v < (1 << s.m):
        raise IndexError(f"output mask {v} out of range 0..{(1 << s.m) - 1}")
    if not 0 <= x < (1 << s.n):
        raise IndexError(f"input {x} out of range 0..{(1 << s.n) - 1}")
    return (int(v) & int(s.table[x])).bit_count() & 1


def _polarity_device(s: SBox, v_lo: int, v_hi: int, layout: int, dev):
    torch = _dev.torch_mod()
    rows = v_hi - v_lo
    shape = (rows, 1 << s.n) if layout == _dev.LAYOUT_MASK_MAJOR else (1 << s.n, rows)
    out = torch.empty(shape, dtype=torch.int32, device=dev)
    tab = _dev.device_table(s, dev)
    with _dev.on(dev):
        _dev.check(_dev.load_library().sbw_polarity(
            _dev.ptr(tab), _dev.table_bytes(s.m), s.n, s.m, v_lo, v_hi, layout, _dev.ptr(out),
            shape[1], _dev.stream_handle(dev)))
    return out


def polarity_row(s: SBox, v: int, out: np.ndarray | None = None) -> np.ndarray:
    """+1 where g_v(x) = 0, -1 where g_v(x) = 1, as int32 (sbox.py:145-152)."""
    dev = _dev.require_device()
    vv = int(v) & 0xFFFFFFFF
    if vv >= (1 << s.m):
        vv &= (1 << s.m) - 1  # bits above m meet only zero table bits
    row = _polarity_device(s, vv, vv + 1, _dev.LAYOUT_MASK_MAJOR, dev)[0].cpu().numpy()
    if out is None:
        return row
    out[:] = row
    return out


def polarity_truth_table(s: SBox, max_bytes: int | None = None) -> PolarityTruthTable:
    """Mask-major (2^m - 1) x 2^n polarity matrix (sbox.py:155-162)."""
    check_budget(((1 << s.m) - 1) * (1 << s.n) * 4, max_bytes)
    dev = _dev.require_device()
    d = _polarity_device(s, 1, 1 << s.m, _dev.LAYOUT_MASK_MAJOR, dev)
    if d.numel() * 4 > (256 << 20):
        from .walsh import device_to_host_chunked
        rows = device_to_host_chunked(d, np.empty(tuple(d.shape), dtype=np.int32))
    else:
        rows = d.cpu().numpy()
    return PolarityTruthTable(s.n, s.m, rows)


__all__ = ["AES_SBOX", "MAX_BITS", "PolarityTruthTable", "SBox", "SBoxFormatError", "aes_sbox",
           "identity_sbox", "generate_sbox", "component_value", "polarity_row",
           "polarity_truth_table", "memory_estimate", "parse_sbox", "render_sbox"]
