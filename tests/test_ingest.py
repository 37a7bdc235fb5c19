"""Native svmlight ingest (csrc/ingest.cu) vs the reference's parser
(data.py:190-239): bit-identical arrays on the reference's bundled dataset
and, through digests the reference itself produced (tests/golden/ingest.npz,
tests/golden/make_golden.py gen_ingest), on randomized number spellings,
Unicode separators and digits, multi-threaded multi-MB input, file objects
and line iterables; the reference's exceptions and messages. Host-only: runs
without a GPU."""

import io

import numpy as np
import pytest

from paper_1803_06333_b200 import data as D

import svm_texts


def _same(a, b):
    (ma, la), (mb, lb) = a, b
    assert ma.n_rows == mb.n_rows
    np.testing.assert_array_equal(ma.indptr, mb.indptr)
    np.testing.assert_array_equal(ma.rows, mb.rows)
    assert ma.vals.tobytes() == mb.vals.tobytes()
    assert la.tobytes() == lb.tobytes()


def test_reference_dataset_roundtrip(golden):
    d = golden("data")
    ex = D.SparseColumnMatrix(int(d["ex_n_rows"]), d["ex_indptr"], d["ex_rows"], d["ex_vals"],
                              validate=False)
    buf = io.StringIO()
    D.write_svmlight(ex, d["ex_labels"], buf)
    m, y = D.parse_svmlight(buf.getvalue())
    assert m.n_rows == int(d["ex_n_rows"])
    np.testing.assert_array_equal(m.indptr, d["ex_indptr"])
    np.testing.assert_array_equal(m.rows, d["ex_rows"])
    assert m.vals.tobytes() == np.asarray(d["ex_vals"]).tobytes()
    assert y.tobytes() == np.asarray(d["ex_labels"]).tobytes()


@pytest.fixture(scope="module")
def ingest_golden(golden):
    z = golden("ingest")
    return dict(zip(z["names"].tolist(), z["digests"].tolist()))


def _outcome(fn):
    try:
        return svm_texts.digest(*fn())
    except Exception as exc:
        return svm_texts.error_key(exc)


@pytest.mark.parametrize("name", list(svm_texts.cases()))
def test_parse_matches_reference_golden(name, ingest_golden):
    """The reference parser's arrays (sha256) or its exact exception and
    message on every case, str input, default threads."""
    text = svm_texts.cases()[name]
    assert _outcome(lambda: D.parse_svmlight(text)) == ingest_golden[name]


@pytest.mark.parametrize("threads", [1, 3, 16])
def test_multithreaded_pieces_agree(threads, ingest_golden):
    text = svm_texts.cases()["random_large"]
    assert len(text) > 4 << 20                               # several MB -> many pieces
    assert _outcome(lambda: D.parse_svmlight(text, n_threads=threads)) == \
        ingest_golden["random_large"]


def test_file_objects_and_line_iterables(tmp_path, ingest_golden):
    text = svm_texts.cases()["random_small"]
    p = tmp_path / "x.svm"
    p.write_bytes(text.replace("\n", "\r\n").encode())     # CRLF file, text mode
    with open(p) as fh:
        assert _outcome(lambda: D.parse_svmlight(fh)) == ingest_golden["random_small"]
    lines = text.splitlines()                                # an iterable of lines
    assert _outcome(lambda: D.parse_svmlight(iter(lines))) == ingest_golden["random_small"]
    assert _outcome(lambda: D.parse_svmlight(io.StringIO(text))) == ingest_golden["random_small"]


@pytest.mark.parametrize("text,msg", [
    ("1 1:2\nfoo 1:2\n", "line 2: bad label 'foo'"),
    ("1 1:2 x:3\n", "line 1: bad feature token 'x:3'"),
    ("1 1:0x1p3\n", "line 1: bad feature token '1:0x1p3'"),
    ("1 1:1__0\n", "line 1: bad feature token '1:1__0'"),
    ("1 -0:1\n", "line 1: feature index 0 < 1"),
])
def test_errors_match_reference_messages(text, msg):
    with pytest.raises(D.DataFormatError) as ei:
        D.parse_svmlight(text)
    assert str(ei.value) == msg


def test_non_finite_feature_rejected_like_reference():
    with pytest.raises(ValueError, match="non-finite"):
        D.parse_svmlight("1 1:inf\n")
