"""The `.sbox` text format (reference: pkg/src/sboxeval/sbox.py:186-253).

Line 1 (after comments/blank lines) is the header "n m"; then exactly 2^n
whitespace-separated entries, decimal or 0x-hex; '#' comments to end of
line.  Errors carry the 1-based line number.
"""
from __future__ import annotations

import numpy as np

from .records import MAX_BITS, SBox, SBoxFormatError


def _as_int(tok: str) -> int:
    return int(tok, 16) if tok[:2].lower() == "0x" else int(tok, 10)


def parse_sbox(text: str) -> SBox:
    header = None
    entries: list[int] = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        toks = raw.partition("#")[0].split()
        if header is None:
            if not toks:
                continue
            if len(toks) != 2:
                raise SBoxFormatError(f"header must be 'n m', got {len(toks)} token(s)", lineno)
            try:
                n, m = _as_int(toks[0]), _as_int(toks[1])
            except ValueError:
                raise SBoxFormatError(f"non-numeric header token in {toks!r}", lineno) from None
            if not (1 <= n <= MAX_BITS and 1 <= m <= MAX_BITS):
                raise SBoxFormatError(f"n and m must be in 1..{MAX_BITS}, got {n} and {m}", lineno)
            header = (n, m)
            continue
        width = header[1]
        for pos, tok in enumerate(toks, start=1):
            try:
                val = _as_int(tok)
            except ValueError:
                raise SBoxFormatError(f"non-numeric entry {tok!r} (token {pos})", lineno) from None
            if not 0 <= val < (1 << width):
                raise SBoxFormatError(
                    f"entry {val} (token {pos}) does not fit in {width} bits", lineno)
            entries.append(val)
    if header is None:
        raise SBoxFormatError("empty input: missing 'n m' header")
    n, m = header
    if len(entries) != (1 << n):
        raise SBoxFormatError(f"expected {1 << n} entries, found {len(entries)}")
    return SBox(n, m, np.array(entries, dtype=np.uint32))


def render_sbox(s: SBox) -> str:
    """Header line, then 16 zero-padded upper-case hex entries per line."""
    digits = (s.m + 3) // 4
    out = [f"{s.n} {s.m}"]
    vals = s.table.tolist()
    for i in range(0, len(vals), 16):
        out.append(" ".join(f"0x{e:0{digits}X}" for e in vals[i:i + 16]))
    return "\n".join(out) + "\n"
