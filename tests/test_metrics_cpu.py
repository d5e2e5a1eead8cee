"""The metrics CSV writer (MetricsWriter, metrics.cpp:8-29)
byte-identical to the compiled reference's output (tests/golden/metrics_ref.csv,
oracle/make_golden.py gen_metrics).  Host-only code of libpqlg.so."""
import ctypes as C
import sys
from pathlib import Path

import pytest

from paper_2307_12983_b200 import _lib

GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
from make_golden import METRICS_ROWS  # noqa: E402


def write_rows(path, rows):
    h = C.c_void_p()
    _lib.call("pqlg_metrics_open", str(path).encode(), C.byref(h))
    for r in rows:
        row = _lib.MetricsRow(r[0], int(r[1]), int(r[2]), int(r[3]), int(r[4]), *r[5:])
        _lib.call("pqlg_metrics_append", h, C.byref(row))
    _lib.call("pqlg_metrics_close", h)


def test_header_matches_reference():
    want = (GOLDEN / "metrics_ref.csv").read_text().splitlines()[0]
    assert _lib.lib().pqlg_metrics_header().decode() == want


def test_rows_byte_identical_to_reference(tmp_path):
    out = tmp_path / "m.csv"
    write_rows(out, METRICS_ROWS)
    assert out.read_bytes() == (GOLDEN / "metrics_ref.csv").read_bytes()


def test_open_truncates_and_rows_are_flushed(tmp_path):
    out = tmp_path / "m.csv"
    out.write_text("stale\nstale\n")
    h = C.c_void_p()
    _lib.call("pqlg_metrics_open", str(out).encode(), C.byref(h))
    row = _lib.MetricsRow(1.0, 4, 4, 0, 0, 0.0, 0.0, 0.0, 0.0)
    _lib.call("pqlg_metrics_append", h, C.byref(row))
    # flushed per row: visible before close
    lines = out.read_text().splitlines()
    assert lines[0].startswith("wall_clock_s,") and lines[1] == "1.000,4,4,0,0,0,0,0,0"
    _lib.call("pqlg_metrics_close", h)


def test_open_failure_is_an_error(tmp_path):
    h = C.c_void_p()
    with pytest.raises(ValueError):
        _lib.call("pqlg_metrics_open", str(tmp_path / "no" / "such" / "dir.csv").encode(),
                  C.byref(h))
