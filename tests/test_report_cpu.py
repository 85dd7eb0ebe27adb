"""Benchmark-harness parity with the reference's so3fft-bench (bench.py:67-322): RNG stream
rule, error metric, report schema and CLI error handling -- host side, no GPU."""
import json

import numpy as np
import pytest

from paper_1808_00896_b200 import report as R


def test_random_coefficients_stream_rule():
    """slot k takes draws 2k (re) and 2k+1 (im) of PCG64(seed) uniform[-1,1] (test_bench.py:25-33)."""
    c = R.random_coefficients(4, 7)
    draws = np.random.Generator(np.random.PCG64(7)).uniform(-1.0, 1.0, size=2 * 84)
    np.testing.assert_array_equal(c.data.real, draws[0::2])
    np.testing.assert_array_equal(c.data.imag, draws[1::2])
    assert np.all(np.abs(c.data.real) <= 1.0)


def test_error_metrics_definition():
    import paper_1808_00896_b200 as so3
    ref = so3.So3Coefficients(2, np.array([1, 0, 2, 0, 0, 0, 0, 0, 0, 4], dtype=complex))
    got = so3.So3Coefficients(2, ref.data + np.array([0.5, 1e-3, 0, 0, 0, 0, 0, 0, 0, 1.0]))
    ab, rel = R.error_metrics(ref, got)
    assert ab == 1.0 and rel == 0.5       # zero reference slots are skipped in the relative error
    with pytest.raises(ValueError):
        R.error_metrics(ref, so3.So3Coefficients.zeros(3))


def _records():
    return [R.BenchRecord(8, 1, "forward", 0, 0.5, 1.0, 1.0, 1e-14, 1e-13, "B200"),
            R.BenchRecord(8, 1, "inverse", 0, 0.25, 1.0, 1.0, 2e-14, 3e-13, "B200")]


def test_csv_json_schema(tmp_path):
    text = R.format_csv(_records())
    assert text.splitlines()[0] == ",".join(R.REPORT_FIELDS)
    ext = R.format_csv(_records(), extended=True)
    assert ext.splitlines()[0] == ",".join(R.REPORT_FIELDS + R.EXTENDED_FIELDS)
    rows = json.loads(R.format_json(_records()))
    assert list(rows[0]) == list(R.REPORT_FIELDS)
    p = tmp_path / "r.json"
    R.write_report(_records(), str(p), "json", extended=True)
    assert json.loads(p.read_text())[1]["transforms_per_s"] == 4.0
    with pytest.raises(ValueError):
        R.write_report([], str(tmp_path / "e.csv"))
    with pytest.raises(ValueError):
        R.write_report(_records(), str(tmp_path / "x.txt"), "xml")
    assert not (tmp_path / "e.csv").exists() and not (tmp_path / "x.txt").exists()
    lines = R.summary_lines(_records())
    assert len(lines) == 2 and lines[0].startswith("B=8")


def test_config_validation_and_cli_errors(capsys):
    with pytest.raises(ValueError):
        R.BenchConfig([0], [1])
    with pytest.raises(ValueError):
        R.BenchConfig([4], [0])
    with pytest.raises(ValueError):
        R.BenchConfig([4], [1], runs=0)
    assert R.main(["--bandwidths", "0", "--runs", "1"]) == 2
    assert "error" in capsys.readouterr().err
    with pytest.raises(SystemExit):
        R.build_parser().parse_args(["--bandwidths", "a,b"])
