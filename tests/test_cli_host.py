"""CLI and bench-harness host paths (CPU only): usage/parse/budget exit codes,
`gen` output, CSV round trip.  Mirrors pkg/tests/test_cli.py and test_bench.py
for everything that fails or finishes before any device work."""
import io


import pytest

import paper_1912_03732_b200 as sw
from paper_1912_03732_b200.cli import main


def write_box(tmp_path, name, n, m, seed, bijective=False):
    p = tmp_path / name
    p.write_text(sw.render_sbox(sw.generate_sbox(n, m, seed, bijective)))
    return str(p)


def test_gen_roundtrip(tmp_path, capsys):
    out = tmp_path / "g.sbox"
    assert main(["gen", "6", "6", "--seed", "4", "--bijective", "--out", str(out)]) == 0
    s = sw.parse_sbox(out.read_text())
    assert s == sw.generate_sbox(6, 6, 4, bijective=True)
    assert main(["gen", "3", "2", "--seed", "1"]) == 0
    assert sw.parse_sbox(capsys.readouterr().out) == sw.generate_sbox(3, 2, 1)


def test_parse_and_io_errors_exit_2(tmp_path, capsys):
    bad = tmp_path / "bad.sbox"
    bad.write_text("2 2\n0 1 2")
    assert main(["nl", str(bad)]) == 2
    assert "expected 4 entries" in capsys.readouterr().err
    assert main(["nl", "/nonexistent/x.sbox"]) == 2
    assert main(["gen", "4", "3", "--bijective"]) == 2  # ValueError: n == m


def test_usage_errors_exit_1(tmp_path, capsys):
    with pytest.raises(SystemExit) as e:
        main(["nl"])
    assert e.value.code == 1
    with pytest.raises(SystemExit) as e:
        main(["nl", "x.sbox", "--workers", "0"])
    assert e.value.code == 1
    path = write_box(tmp_path, "r.sbox", 4, 4, 1)
    assert main(["bench", path, "--methods", "magic"]) == 1
    assert main(["bench", path, "--workers", "1,x"]) == 1


def test_budget_exit_3_with_hint(tmp_path, capsys, monkeypatch):
    path = write_box(tmp_path, "r8.sbox", 8, 8, seed=1)
    assert main(["nl", path, "--max-mem", "1000"]) == 3
    assert "--mode stream" in capsys.readouterr().err
    monkeypatch.setenv("SBOX_EVAL_MAX_MEM", "1000")
    assert main(["nl", path, "--method", "transposed"]) == 3


def test_size_guards_exit_4(tmp_path, capsys):
    path = write_box(tmp_path, "r11.sbox", 11, 4, seed=1)
    assert main(["walsh", path]) == 4
    path = write_box(tmp_path, "r9.sbox", 9, 4, seed=1)
    assert main(["verify", path]) == 4


def test_csv_roundtrip_and_speedups():
    recs = [sw.BenchRecord("fused", 8, 8, 1, 2, [2.0, 4.0], [1.0, 1.0]),
            sw.BenchRecord("rowmajor", 8, 8, 1, 2, [9.0, 9.0], [8.0, 8.0])]
    buf = io.StringIO()
    sw.write_csv(recs, buf)
    rows = sw.read_csv(buf.getvalue())
    assert [r["method"] for r in rows] == ["fused", "rowmajor"]
    assert rows[0]["mean_ms"] == 3.0 and rows[0]["stddev_ms"] == 1.0
    sp = sw.speedup_report(recs, "rowmajor")
    assert {r.method: r.ratio for r in sp} == {"fused": 3.0, "rowmajor": 1.0}
    with pytest.raises(ValueError, match="baseline"):
        sw.speedup_report(recs, "parallel")
    with pytest.raises(ValueError):
        sw.run_benchmark(sw.identity_sbox(2), ["fused"], repetitions=0)

