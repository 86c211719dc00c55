"""Materialised spectra in both layouts at every n, against the oracle and the
reference's own full-matrix hashes.

  mask-major rows[v - 1][u] = W(u, v)   (WalshSpectrum.rows, walsh.py:32-44, :174)
  x-major    wt[u][v - 1]   = W(u, v)   (walsh.py:117-131)

The x-major store is checked above n = 12 (tensor-core spectrum kernels
n = 13..16, multi-pass K3 n >= 17) on unaligned mask slices, and the whole
16x16 matrix (2^32 entries, 16 GiB per layout) is hashed in both layouts and
compared with tests/golden/hashes_16x16.json, which
tests/golden/make_golden_16x16_hashes.py computed by running the reference.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_1912_03732_b200 as sw
from oracle import sbw_oracle as orc

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("n,v_lo,count", [(13, 77, 37), (14, 1, 64), (14, 16000, 383), (15, 5, 21),
                                          (15, 32700, 67), (16, 1, 33), (16, 44801, 40),
                                          (16, 65500, 35)])
def test_xmajor_slices_tensor_core_sizes(n, v_lo, count):
    s = sw.generate_sbox(n, n, 0, bijective=True)
    v_hi = min(1 << n, v_lo + count)
    want = orc.spectrum(s.table, n, v_lo, v_hi)
    xm, mx = sw.spectrum_device(s, v_lo, v_hi, layout="x")
    assert tuple(xm.shape) == (1 << n, v_hi - v_lo)
    assert np.array_equal(xm.cpu().numpy(), want.T)
    assert np.array_equal(mx.cpu().numpy(), np.abs(want.astype(np.int64)).max(axis=1))
    mm, _ = sw.spectrum_device(s, v_lo, v_hi, layout="mask")
    assert np.array_equal(mm.cpu().numpy(), want)


@pytest.mark.parametrize("n,m,seed", [(17, 5, 1), (18, 4, 2), (20, 3, 3), (21, 2, 4), (24, 2, 5)])
def test_xmajor_multipass_sizes(n, m, seed):
    """n >= 17 (multi-pass K3 spectrum) in both layouts, every mask."""
    s = sw.generate_sbox(n, m, seed)
    want = orc.spectrum(s.table, n, 1, 1 << m)
    xm, _ = sw.spectrum_device(s, layout="x")
    assert np.array_equal(xm.cpu().numpy(), want.T)
    mm, mx = sw.spectrum_device(s, layout="mask")
    assert np.array_equal(mm.cpu().numpy(), want)
    assert np.array_equal(mx.cpu().numpy(), np.abs(want.astype(np.int64)).max(axis=1))


def test_xmajor_host_export_16x16_slice():
    """spectrum_to_host(layout="x") on a 16x16 mask slice, chunked."""
    s = sw.generate_sbox(16, 16, 0, bijective=True)
    out, mx = sw.spectrum_to_host(s, 1000, 1300, layout="x", chunk_bytes=97 * 65536 * 4)
    want = orc.spectrum(s.table, 16, 1000, 1300)
    assert np.array_equal(out, want.T)
    assert np.array_equal(mx, np.abs(want.astype(np.int64)).max(axis=1))


def _golden_hashes():
    with open(os.path.join(HERE, "golden", "hashes_16x16.json")) as f:
        return json.load(f)


@pytest.mark.slow
def test_16x16_full_matrix_hashes_both_layouts():
    """All 2^32 coefficients of the 16x16 seed-0 box, both layouts, hashed
    and compared with the reference's own hashes (16 GiB each)."""
    import torch

    g = _golden_hashes()
    s = sw.generate_sbox(16, 16, 0, bijective=True)
    # mask-major: 1024-mask device chunks, streamed to the host in order
    h = hashlib.sha256()
    for a in range(1, 1 << 16, 1024):
        b = min(1 << 16, a + 1024)
        chunk, _ = sw.spectrum_device(s, a, b, layout="mask")
        h.update(chunk.cpu().numpy().tobytes())
        del chunk
    assert h.hexdigest() == g["sha256_mask_major"]
    # x-major: the whole 16 GiB store on the device by the mask-major +
    # transpose path (the inverse path has its own hash test below)
    os.environ["SBW_XMAJOR_INVERSE"] = "0"
    try:
        xm, mx = sw.spectrum_device(s, layout="x")
    finally:
        del os.environ["SBW_XMAJOR_INVERSE"]
    torch.cuda.synchronize()
    h = hashlib.sha256()
    for a in range(0, 1 << 16, 1024):
        h.update(xm[a:a + 1024].cpu().numpy().tobytes())
    assert h.hexdigest() == g["sha256_x_major"]
    r = sw.nonlinearity_from_maxima(sw.ColumnMaxima(16, 16, sw.walsh.maxabs_to_nl(mx, 16)))
    assert (r.value, r.argmin_v) == (g["nl"], g["argmin_v"])


@pytest.mark.parametrize("n,v_lo,count", [(12, 1, 300), (13, 77, 37), (16, 44801, 40)])
def test_staged_and_per_lane_spectrum_epilogues_agree(n, v_lo, count):
    """sbw_spectrum takes the staged epilogue (shared-memory slot ring + bulk
    copies) for 16-byte aligned rows and the per-lane store epilogue otherwise
    (here: ld = 2^n + 2).  Both must give the oracle's rows."""
    import torch

    from paper_1912_03732_b200 import device as d

    s = sw.generate_sbox(n, n, seed=n, bijective=True)
    lib = d.load_library()
    dev = torch.device("cuda", 0)
    tab = d.device_table(s, dev)
    want = orc.spectrum(s.table, n, v_lo, v_lo + count)
    for ld in (1 << n, (1 << n) + 2):
        out = torch.full((count, ld), -7, dtype=torch.int32, device=dev)
        mx = torch.empty(count, dtype=torch.int32, device=dev)
        sb = lib.sbw_spectrum_scratch_bytes(n, n, v_lo, v_lo + count, d.LAYOUT_MASK_MAJOR)
        scratch = torch.empty(max(1, sb), dtype=torch.uint8, device=dev)
        d.check(lib.sbw_spectrum(d.ptr(tab), d.table_bytes(n), n, n, v_lo, v_lo + count, d.LAYOUT_MASK_MAJOR,
                                 d.ptr(out), ld, d.ptr(mx), d.ptr(scratch), sb, d.stream_handle(dev)))
        got = out.cpu().numpy()
        assert np.array_equal(got[:, : 1 << n], want), ld
        assert (got[:, 1 << n:] == -7).all(), ld  # the padding is never written
        assert np.array_equal(mx.cpu().numpy(), np.abs(want).max(axis=1)), ld


# ---- x-major of a bijective box straight from its inverse (sbw_xmajor_from_inverse)
@pytest.mark.parametrize("n,seed", [(12, 0), (12, 7), (13, 1), (14, 2), (15, 3)])
def test_xmajor_full_from_inverse_matches_oracle(n, seed):
    """Full-range x-major store of a bijective box (inverse path, default)
    equals the mask-major rows transposed; n = 12 also against the oracle,
    and the transpose path (SBW_XMAJOR_INVERSE=0) agrees."""
    import torch

    s = sw.generate_sbox(n, n, seed, bijective=True)
    os.environ["SBW_XMAJOR_INVERSE"] = "1"  # n = 12 defaults to the transpose path
    try:
        xm, mx = sw.spectrum_device(s, layout="x")
    finally:
        del os.environ["SBW_XMAJOR_INVERSE"]
    assert tuple(xm.shape) == (1 << n, (1 << n) - 1)
    mm, mmx = sw.spectrum_device(s, layout="mask")
    assert torch.equal(xm, mm.t())
    assert torch.equal(mx, mmx)
    if n == 12:
        want = orc.spectrum(s.table, n, 1, 1 << n)
        assert np.array_equal(xm.cpu().numpy(), want.T)
        assert np.array_equal(mx.cpu().numpy(), np.abs(want.astype(np.int64)).max(axis=1))
    os.environ["SBW_XMAJOR_INVERSE"] = "0"
    try:
        xt, _ = sw.spectrum_device(s, layout="x")
    finally:
        del os.environ["SBW_XMAJOR_INVERSE"]
    assert torch.equal(xt, xm)


@pytest.mark.parametrize("n,u_lo,u_hi,pad,shift", [(12, 1, 4096, 0, 1), (12, 5, 300, 9, 2), (13, 100, 8192, 3, 3),
                                                   (16, 1, 70, 0, 0), (16, 65400, 65536, 1, 1),
                                                   (14, 2, 16384, 0, 0)])
def test_xmajor_from_inverse_abi_rows_pitch_alignment(n, u_lo, u_hi, pad, shift):
    """The C entry directly: any row range, pitch 2^n - 1 + pad, an output
    pointer shifted by `shift` words from 16-byte alignment; the words around
    every written row are untouched."""
    import torch

    from paper_1912_03732_b200 import device as dv
    from paper_1912_03732_b200 import walsh

    s = sw.generate_sbox(n, n, 11, bijective=True)
    inv = walsh._inverse_if_bijective(s)
    dev = torch.device("cuda:0")
    ld = (1 << n) - 1 + pad
    rows = u_hi - u_lo
    buf = torch.full((rows * ld + 64,), -7, dtype=torch.int32, device=dev)
    lib = dv.load_library()
    nbytes = lib.sbw_xmajor_inverse_scratch_bytes(n, u_lo, u_hi)
    scratch = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    itab = dv.device_table(inv, dev)
    dv.check(lib.sbw_xmajor_from_inverse(dv.ptr(itab), dv.table_bytes(n), n, u_lo, u_hi,
                                         dv.ptr(buf) + 4 * shift, ld, dv.ptr(scratch), nbytes,
                                         dv.stream_handle(dev)))
    torch.cuda.synchronize()
    got = buf[shift:shift + rows * ld].view(rows, ld)
    mm, _ = sw.spectrum_device(s, layout="mask")
    want = mm.t()[u_lo:u_hi]
    assert torch.equal(got[:, :(1 << n) - 1], want)
    if pad:
        assert bool((got[:, (1 << n) - 1:] == -7).all())
    assert bool((buf[:shift] == -7).all()) and bool((buf[shift + rows * ld:] == -7).all())


def test_xmajor_from_inverse_rejects_bad_arguments():
    import torch

    from paper_1912_03732_b200 import device as dv

    s = sw.generate_sbox(12, 12, 0, bijective=True)
    dev = torch.device("cuda:0")
    tab = dv.device_table(s, dev)
    lib = dv.load_library()
    out = torch.empty(4096 * 4095, dtype=torch.int32, device=dev)
    scratch = torch.empty(1 << 20, dtype=torch.uint8, device=dev)
    st = dv.stream_handle(dev)
    for args in [(11, 1, 2048, 2047), (12, 0, 4096, 4095), (12, 1, 4097, 4095), (12, 1, 4096, 4094)]:
        n, lo, hi, ld = args
        with pytest.raises((ValueError, IndexError)):
            dv.check(lib.sbw_xmajor_from_inverse(dv.ptr(tab), dv.table_bytes(n), n, lo, hi, dv.ptr(out), ld,
                                                 dv.ptr(scratch), 1 << 20, st))
    with pytest.raises(ValueError):  # misaligned output
        dv.check(lib.sbw_xmajor_from_inverse(dv.ptr(tab), dv.table_bytes(12), 12, 1, 4096, dv.ptr(out) + 2,
                                             4095, dv.ptr(scratch), 1 << 20, st))


@pytest.mark.slow
def test_16x16_full_xmajor_from_inverse_hash():
    """The whole 16x16 x-major store (65536 x 65535 int32, 16 GiB) through the
    inverse path on the device, hashed and compared with the reference's own
    sha256 (tests/golden/hashes_16x16.json)."""
    import torch

    g = json.load(open(os.path.join(HERE, "golden", "hashes_16x16.json")))
    s = sw.generate_sbox(16, 16, 0, bijective=True)
    xm, mx = sw.spectrum_device(s, layout="x")
    assert tuple(xm.shape) == (65536, 65535)
    h = hashlib.sha256()
    pin = torch.empty((2048, 65535), dtype=torch.int32, pin_memory=True)
    for a in range(0, 65536, 2048):
        pin.copy_(xm[a:a + 2048])
        h.update(pin.numpy().tobytes())
    assert h.hexdigest() == g["sha256_x_major"]
    values = ((1 << 16) - mx.cpu().numpy().astype(np.int64)) >> 1
    assert orc.nl_from_maxima(values) == (g["nl"], g["argmin_v"])


@pytest.mark.parametrize("n,chunk_rows", [(13, 1000), (14, 4096), (15, 333)])
def test_xmajor_full_host_export_from_inverse(n, chunk_rows):
    """spectrum_to_host(layout="x") over every mask of a bijective box goes by
    row chunks of the x-major matrix (inverse path): equal to the device store
    of the transpose path, including an odd final chunk and row 0."""
    import torch

    s = sw.generate_sbox(n, n, 3, bijective=True)
    out, mx = sw.spectrum_to_host(s, layout="x", chunk_bytes=chunk_rows * ((1 << n) - 1) * 4)
    os.environ["SBW_XMAJOR_INVERSE"] = "0"
    try:
        want, wmx = sw.spectrum_device(s, layout="x")
    finally:
        del os.environ["SBW_XMAJOR_INVERSE"]
    assert out.shape == (1 << n, (1 << n) - 1)
    assert np.array_equal(out, want.cpu().numpy())
    assert np.array_equal(mx, wmx.cpu().numpy())
