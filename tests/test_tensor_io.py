"""Host-side file formats (no GPU): .tns parse errors with line numbers,
factor containers and trace CSV round trips (tensor_io.py:25-170)."""

import os

import numpy as np
import pytest

from paper_1910_02371_b200 import tensor_io
from paper_1910_02371_b200.exceptions import DataError
from paper_1910_02371_b200.trace import RunTrace


@pytest.mark.parametrize("text,msg", [
    ("1 2 3 1.0\n1 2 1.0\n", r":2: expected 4 fields, got 3"),
    ("1 2 x\n", r":1: non-numeric token"),
    ("1 0 2.0\n", r":1: coordinate 0 in mode 1 must be >= 1"),
    ("# only a comment\n", r"no data lines"),
    ("5\n", r":1: need at least one coordinate and a value"),
    ("# dims: 2 x\n1 1 1.0\n", r":1: malformed dims header"),
    ("# dims: 2 2 2\n1 1 1.0\n", r"dims header has 3 modes, data has 2"),
    ("# dims: 2 2\n3 1 1.0\n", r"mode 0 coordinate 3 exceeds declared dimension 2"),
])
def test_parse_tns_errors(tmp_path, text, msg):
    path = os.path.join(tmp_path, "bad.tns")
    with open(path, "w") as fh:
        fh.write(text)
    with pytest.raises(DataError, match=msg):
        tensor_io.parse_tns(path)


def test_parse_tns_missing_file(tmp_path):
    with pytest.raises(DataError, match="cannot read"):
        tensor_io.parse_tns(os.path.join(tmp_path, "nope.tns"))


def test_factor_and_trace_round_trips(tmp_path):
    rng = np.random.default_rng(0)
    fs = [rng.standard_normal((d, 3)) for d in (4, 5, 6)]
    p = os.path.join(tmp_path, "f.bin")
    tensor_io.write_factors(fs, p)
    back = tensor_io.read_factors(p)
    assert all(np.array_equal(a, b) for a, b in zip(fs, back))
    tr = RunTrace(metric_name="rmse", metadata={"seed": "3", "algorithm": "als"})
    for i, (e, o, m) in enumerate([(0.0, 3.5, 0.1), (0.25, 1.0 / 3.0, 0.05)]):
        tr.append(i, e, o, m)
    p = os.path.join(tmp_path, "t.csv")
    tensor_io.write_trace(tr, p)
    first = open(p).read()
    tr2 = tensor_io.read_trace(p)
    assert tr2.metric_name == "rmse" and tr2.metadata == tr.metadata
    assert [(r.iteration, r.elapsed_s, r.objective, r.metric) for r in tr2.records] == \
        [(r.iteration, r.elapsed_s, r.objective, r.metric) for r in tr.records]
    tensor_io.write_trace(tr2, p)
    assert open(p).read() == first
