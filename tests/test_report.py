"""CPU: the report parity layer writes the reference harness's files
byte-for-byte (golden files produced by the reference's own emit_reports,
tests/golden/make_report_golden.py)."""

import json
from pathlib import Path

import pytest

GOLD = Path(__file__).resolve().parent / "golden" / "report_fmt"


@pytest.fixture(scope="module")
def R():
    # the report module's formatting needs no GPU (run_comparison does)
    from paper_1706_00241_b200 import report

    return report


def test_emit_reports_byte_identical(R, tmp_path):
    data = json.loads((GOLD / "rows.json").read_text())
    R.emit_reports(data["rows"], data["summary"], tmp_path)
    for name in ("table.csv", "summary.json", "subset.csv"):
        assert (tmp_path / name).read_bytes() == (GOLD / name).read_bytes(), name


def test_delta_definition(R):
    assert R.rel_error_delta(-99.0, -100.0) == 0.01
    assert R.rel_error_delta(5.0, 5.0) == 0.0
