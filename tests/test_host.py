"""Host-side logic of the drop-in API (CPU only, no device calls).

Mirrors the reference's unit tests for the non-compute parts:
pkg/tests/test_sbox.py (table, parsing, generation, invariants, memory
estimates), pkg/tests/test_parallel.py (partition) and the budget checks
that must fire before any GPU work.
"""
import numpy as np
import pytest

import paper_1912_03732_b200 as sw
from tests.util import sha


def test_aes_table_is_the_standard_one(golden):
    assert sw.AES_SBOX[0] == 0x63 and sw.AES_SBOX[1] == 0x7C
    assert sw.AES_SBOX[0x53] == 0xED and sw.AES_SBOX[0xFF] == 0x16
    assert sorted(sw.AES_SBOX) == list(range(256))


@pytest.mark.parametrize("name,n,m,bij", [("8x8", 8, 8, True), ("12x12", 12, 12, True),
                                          ("16x16", 16, 16, True), ("20x20", 20, 20, False),
                                          ("24x16", 24, 16, False)])
def test_generate_sbox_matches_reference_stream(golden, name, n, m, bij):
    s = sw.generate_sbox(n, m, seed=0, bijective=bij)
    assert sha(s.table) == golden["configs"][name]["sha_table_u32"]
    assert s.table.dtype == np.uint32 and not s.table.flags.writeable


def test_generate_sweep_tables(golden):
    for rec in golden["small"]["sweep"][:120]:
        s = sw.generate_sbox(rec["n"], rec["m"], rec["seed"], rec["bijective"])
        assert sha(s.table) == rec["sha_table_u32"]


class TestSBoxInvariants:
    def test_wrong_table_length(self):
        with pytest.raises(ValueError, match="4 entries"):
            sw.SBox(2, 2, np.array([0, 1, 2], dtype=np.uint32))

    def test_entry_exceeds_output_width(self):
        with pytest.raises(ValueError, match="does not fit"):
            sw.SBox(2, 2, np.array([0, 1, 2, 4], dtype=np.uint32))

    def test_bit_width_caps(self):
        with pytest.raises(ValueError):
            sw.SBox(0, 1, np.array([], dtype=np.uint32))
        with pytest.raises(ValueError):
            sw.SBox(25, 1, np.zeros(1 << 25, dtype=np.uint32))

    def test_table_is_immutable(self):
        s = sw.identity_sbox(3)
        with pytest.raises(ValueError):
            s.table[0] = 5

    def test_equality_and_bijective(self):
        a = sw.generate_sbox(6, 6, seed=42, bijective=True)
        assert a == sw.generate_sbox(6, 6, seed=42, bijective=True)
        assert a != sw.generate_sbox(6, 6, seed=43, bijective=True)
        assert a.is_bijective() and len(a) == 64
        with pytest.raises(ValueError, match="n == m"):
            sw.generate_sbox(4, 3, seed=0, bijective=True)


def test_component_value():
    s = sw.generate_sbox(4, 4, seed=5)
    assert all(sw.component_value(s, 0, x) == 0 for x in range(16))
    assert sw.component_value(sw.identity_sbox(3), 0b001, 5) == 1
    assert sw.component_value(sw.aes_sbox(), 0xFF, 0) == 0
    with pytest.raises(IndexError):
        sw.component_value(sw.identity_sbox(3), 8, 0)
    with pytest.raises(IndexError):
        sw.component_value(sw.identity_sbox(3), 1, 8)


class TestParse:
    def test_aes_file(self):
        s = sw.parse_sbox("8 8\n" + " ".join(str(e) for e in sw.AES_SBOX))
        assert s == sw.aes_sbox()

    def test_hex_and_comments(self):
        s = sw.parse_sbox("# a box\n2 2  # header\n0x0 1\n# mid comment\n0x2 3\n")
        assert list(s.table) == [0, 1, 2, 3]

    def test_errors(self):
        with pytest.raises(sw.SBoxFormatError, match="expected 4 entries, found 3"):
            sw.parse_sbox("2 2\n0 1 2")
        with pytest.raises(sw.SBoxFormatError, match="line 3.*does not fit in 2 bits"):
            sw.parse_sbox("2 2\n0 1\n4 3")
        with pytest.raises(sw.SBoxFormatError, match="line 2.*'zap'.*token 2"):
            sw.parse_sbox("2 2\n0 zap 2 3")
        with pytest.raises(sw.SBoxFormatError, match="1..24"):
            sw.parse_sbox("25 8\n0")
        with pytest.raises(sw.SBoxFormatError, match="header"):
            sw.parse_sbox("# nothing here\n")

    @pytest.mark.parametrize("n,m,seed,bij", [(3, 3, 7, True), (4, 3, 1, False), (5, 5, 11, True),
                                              (2, 6, 9, False)])
    def test_roundtrip(self, n, m, seed, bij):
        s = sw.generate_sbox(n, m, seed, bij)
        assert sw.parse_sbox(sw.render_sbox(s)) == s

    def test_render_format(self):
        lines = sw.render_sbox(sw.aes_sbox()).splitlines()
        assert lines[0] == "8 8" and len(lines) == 17
        assert lines[1].split() == [f"0x{e:02X}" for e in sw.AES_SBOX[:16]]


class TestMemory:
    def test_estimates(self):
        assert sw.memory_estimate(8, 8, 4, "retain") == 255 * 256 * 4 + 256 * 4
        assert sw.memory_estimate(16, 16, 4, "retain") == 1 << 34
        assert sw.memory_estimate(16, 16, 4, "stream", workers=10) == 12 * (1 << 16) * 4
        with pytest.raises(ValueError):
            sw.memory_estimate(4, 4, 4, "keep")

    def test_budget_errors_fire_before_any_device_work(self):
        s = sw.generate_sbox(8, 8, seed=3)
        with pytest.raises(sw.MemoryBudgetError):
            sw.fwht_rowmajor(s, max_bytes=1024)
        with pytest.raises(sw.MemoryBudgetError):
            sw.fwht_transposed(s, max_bytes=1024)
        with pytest.raises(sw.MemoryBudgetError):
            sw.fwht_fused(s, mode="retain", max_bytes=1024)
        with pytest.raises(sw.MemoryBudgetError):
            sw.fwht_parallel(s, workers=2, mode="retain", max_bytes=4096)
        with pytest.raises(sw.MemoryBudgetError):
            sw.polarity_truth_table(s, max_bytes=1000)
        with pytest.raises(ValueError, match="retain.*stream"):
            sw.fwht_fused(s, mode="drop")
        with pytest.raises(ValueError):
            sw.fwht_parallel(s, workers=0)

    def test_tracker(self):
        t = sw.AllocationTracker()
        t.charge(100)
        t.charge(50)
        t.release(100)
        assert t.current_bytes == 50 and t.peak_bytes == 150
        t.reset_peak()
        assert t.peak_bytes == 50


class TestPartition:
    def test_examples(self):
        assert [b - a for a, b in sw.partition_columns(15, 8).ranges] == [2, 2, 2, 2, 2, 2, 2, 1]
        assert sw.partition_columns(7, 1).ranges == ((1, 8),)
        p = sw.partition_columns(3, 8)
        assert p.ranges == ((1, 2), (2, 3), (3, 4)) and p.worker_count == 8
        with pytest.raises(ValueError):
            sw.partition_columns(0, 4)
        with pytest.raises(ValueError):
            sw.partition_columns(15, 0)

    def test_exhaustive_properties(self):
        for columns in range(1, 1025):
            for workers in (1, 2, 3, 7, 8, 16, 64):
                r = sw.partition_columns(columns, workers).ranges
                span = [b - a for a, b in r]
                assert len(r) <= workers and r[0][0] == 1 and r[-1][1] == columns + 1
                assert max(span) - min(span) <= 1 and min(span) >= 1
                assert all(c[0] == p[1] for p, c in zip(r, r[1:]))


def test_no_cpu_fallback():
    """Without a CUDA device every compute entry point raises (no silent CPU path)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    s = sw.generate_sbox(6, 6, seed=1)
    for call in (lambda: sw.fwht_fused(s, mode="stream"), lambda: sw.fwht_transposed(s),
                 lambda: sw.fwht_column_in_place(np.ones(4, dtype=np.int32)),
                 lambda: sw.walsh_direct(s, 1, 1), lambda: sw.polarity_row(s, 3),
                 lambda: sw.evaluate(s, method="fused")):
        with pytest.raises(RuntimeError, match="CUDA"):
            call()


def test_write_spectrum_format():
    import io

    w = sw.WalshSpectrum(2, 2, np.array([[0, 4, 0, 0], [0, 0, 4, 0], [0, 0, 0, 4]], dtype=np.int32))
    buf = io.StringIO()
    sw.write_spectrum(w, buf)
    lines = buf.getvalue().splitlines()
    assert lines[0] == "2 2" and len(lines) == 4
    assert w.value(0, 0) == 4 and w.value(3, 0) == 0 and w.value(1, 1) == 4
