"""Sweep CSV (io.py:172-180): the default file keeps the reference's five columns
and number formats; SURVEY.md §5's GPU context columns are appended only on request."""

import csv

import pytest

jb = pytest.importorskip("paper_2601_07048_b200")
from paper_2601_07048_b200 import measure  # noqa: E402


def _pts():
    return [measure.SweepPoint(64, 10, 0.9123456789, 1234567.891234, 12.3456789),
            measure.SweepPoint(128, 10, 0.95, 2e6, 8.0)]


def test_default_header_and_formats(tmp_path):
    p = tmp_path / "s.csv"
    measure.write_sweep_csv(p, _pts())
    rows = list(csv.reader(open(p)))
    assert tuple(rows[0]) == ("beam_width", "k", "recall", "qps", "mean_latency_us")
    assert rows[1] == ["64", "10", "0.912346", "1234567.89", "12.35"]


def test_extra_columns_appended_in_fixed_order(tmp_path):
    p = tmp_path / "s.csv"
    measure.write_sweep_csv(p, _pts(), {"cpu_qps": [700.5, 690.0], "gpus": 1, "hbm_frac": 0.18})
    rows = list(csv.reader(open(p)))
    assert tuple(rows[0]) == ("beam_width", "k", "recall", "qps", "mean_latency_us", "gpus", "hbm_frac", "cpu_qps")
    assert rows[1][5:] == ["1", "0.18", "700.5"]
    assert rows[2][5:] == ["1", "0.18", "690"]
    with pytest.raises(ValueError):
        measure.write_sweep_csv(p, _pts(), {"bogus": 1})
