"""File formats (CBM1 / CBH1 / manifest) and the host ledger (no GPU)."""

import struct

import numpy as np
import pytest

from paper_2602_02827_b200 import io as cio
from paper_2602_02827_b200.oracle import ObservationLedger, reveal


def test_vectors_and_matrix_round_trip_and_layout(tmp_path):
    v = np.arange(6, dtype=np.float64).reshape(3, 2) / 7
    cio.write_vectors(tmp_path / "v.cbm", v)
    raw = (tmp_path / "v.cbm").read_bytes()
    assert raw[:12] == b"CBM1" + struct.pack("<ii", 2, 3)  # magic, dim, count
    np.testing.assert_array_equal(cio.read_vectors(tmp_path / "v.cbm"), v.astype(np.float32).astype(np.float64))
    m = np.linspace(-1, 1, 12).reshape(4, 3)
    cio.write_matrix(tmp_path / "m.cbh", m)
    assert (tmp_path / "m.cbh").read_bytes()[:12] == b"CBH1" + struct.pack("<ii", 4, 3)  # magic, rows, cols
    np.testing.assert_array_equal(cio.read_matrix(tmp_path / "m.cbh"), m.astype(np.float32).astype(np.float64))
    assert cio.sniff_format(tmp_path / "v.cbm") == "vectors" and cio.sniff_format(tmp_path / "m.cbh") == "matrix"


def test_format_errors(tmp_path):
    cio.write_vectors(tmp_path / "v.cbm", np.ones((2, 2)))
    with pytest.raises(ValueError, match="bad magic"):
        cio.read_matrix(tmp_path / "v.cbm")
    (tmp_path / "t.cbm").write_bytes((tmp_path / "v.cbm").read_bytes() + b"x")
    with pytest.raises(ValueError, match="trailing bytes"):
        cio.read_vectors(tmp_path / "t.cbm")
    (tmp_path / "s.cbm").write_bytes((tmp_path / "v.cbm").read_bytes()[:-2])
    with pytest.raises(ValueError, match="short read in payload"):
        cio.read_vectors(tmp_path / "s.cbm")
    (tmp_path / "h.cbm").write_bytes(b"CBM1" + struct.pack("<ii", 0, 3))
    with pytest.raises(ValueError, match="implausible dimensions"):
        cio.read_vectors(tmp_path / "h.cbm")
    with pytest.raises(ValueError, match="non-empty 2-D"):
        cio.write_vectors(tmp_path / "e.cbm", np.ones(3))
    (tmp_path / "x.bin").write_bytes(b"ZZZZ")
    with pytest.raises(ValueError, match="unrecognized file format"):
        cio.sniff_format(tmp_path / "x.bin")


def test_manifest(tmp_path):
    cio.write_manifest(tmp_path / "m.jsonl", [("a", "a.cbm"), ("b", "sub/b.cbm")])
    got = cio.read_manifest(tmp_path / "m.jsonl")
    assert got == [("a", tmp_path / "a.cbm"), ("b", tmp_path / "sub/b.cbm")]
    assert cio.sniff_format(tmp_path / "m.jsonl") == "manifest"
    with pytest.raises(ValueError, match="duplicate doc_id"):
        cio.write_manifest(tmp_path / "d.jsonl", [("a", "x"), ("a", "y")])
    (tmp_path / "bad.jsonl").write_text('{"doc_id": "a"}\n')
    with pytest.raises(ValueError, match="bad manifest line"):
        cio.read_manifest(tmp_path / "bad.jsonl")
    (tmp_path / "empty.jsonl").write_text("\n")
    with pytest.raises(ValueError, match="manifest is empty"):
        cio.read_manifest(tmp_path / "empty.jsonl")


class _MatrixOracle:
    def __init__(self, m):
        self.m = np.asarray(m, dtype=np.float64)
        self.n_docs, self.n_query_tokens = self.m.shape
        self.charged = 0

    def _charge(self, i, t):
        self.charged += 1
        return float(self.m[i, t])


def test_ledger_and_reveal_semantics():
    o = _MatrixOracle([[0.5, 0.25, 1.0], [0.125, 0.0, -0.5]])
    led = ObservationLedger(2, 3)
    assert reveal(led, o, 0, 2) == 1.0
    reveal(led, o, 0, 0)
    reveal(led, o, 1, 1)
    assert led.trace == [(0, 2, 1.0), (0, 0, 0.5), (1, 1, 0.0)]
    assert led.coverage() == 0.5 and led.observed_count == 3 and o.charged == 3
    assert led.observed_cols(0) == [0, 2] and led.unobserved_cols(0) == [1] and led.row_values(0) == [1.0, 0.5]
    st = led.row_stats(0)
    assert (st.n, st.total, st.mean, st.m2) == (2, 1.5, 0.75, 0.125)
    with pytest.raises(ValueError, match="already revealed"):
        reveal(led, o, 0, 2)
    with pytest.raises(IndexError, match="column"):
        led.is_observed(0, 3)
    with pytest.raises(ValueError, match="shapes differ"):
        reveal(ObservationLedger(3, 3), o, 0, 0)
    with pytest.raises(ValueError, match="must be positive"):
        ObservationLedger(0, 2)
