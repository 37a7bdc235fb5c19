"""Native svmlight ingest (csrc/ingest.cu) vs the reference's line parser
(data.py:190-239): bit-identical arrays on the reference's bundled dataset,
on randomized number spellings, multi-threaded on multi-MB input, and the
reference's error messages. Host-only: runs without a GPU."""

import io

import numpy as np
import pytest

from paper_1803_06333_b200 import data as D


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
    assert D._parse_svmlight_native(buf.getvalue(), True, 0) is not None   # native path taken


def _random_text(rng, n, d, k):
    spell = [lambda v: "%.17g" % v, lambda v: repr(float(v)), lambda v: "%.3e" % v,
             lambda v: "%.6f" % v, lambda v: "%+.5E" % v, lambda v: "%d" % int(v * 100),
             lambda v: ("%d" % int(v * 1e6)).replace("000", "_000"),
             lambda v: ".%d" % abs(int(v * 1000)), lambda v: "%d." % int(v * 10)]
    lines = ["# header comment", ""]
    for _ in range(n):
        y = rng.choice(["1", "-1", "0", "+1", "1.0", "2.5e-1", "-0"])
        feats = np.sort(rng.choice(d, size=rng.integers(0, k + 1), replace=False)) + 1
        toks = [f"{j}:{spell[rng.integers(len(spell))](rng.standard_normal())}" for j in feats]
        sep = rng.choice([" ", "\t", "  "])
        lines.append(sep.join([y] + toks) + rng.choice(["", " ", "\t"]))
    lines.append("  # trailing comment")
    return "\n".join(lines) + "\n"


def test_native_equals_line_parser_random_spellings():
    rng = np.random.default_rng(5)
    text = _random_text(rng, 3000, 500, 12)
    text += "inf 5:1_0.5_0e1_0 6:-0.0\n-NaN 1:2\n-Infinity\n"
    nat = D._parse_svmlight_native(text, True, 0)
    assert nat is not None
    _same(nat, D._parse_svmlight_lines(text.splitlines()))


def test_multithreaded_large_input_and_file_objects(tmp_path):
    rng = np.random.default_rng(9)
    text = _random_text(rng, 60_000, 20_000, 30)            # several MB -> many pieces
    assert len(text) > 4 << 20
    ref = D._parse_svmlight_lines(text.splitlines())
    for threads in (1, 3, 16):
        _same(D._parse_svmlight_native(text, True, threads), ref)
    p = tmp_path / "x.svm"
    p.write_bytes(text.replace("\n", "\r\n").encode())         # CRLF file, text mode
    with open(p) as fh:
        _same(D.parse_svmlight(fh), ref)


@pytest.mark.parametrize("text,msg", [
    ("1 1:2\nfoo 1:2\n", "line 2: bad label 'foo'"),
    ("1 1:2 3\n", "line 1: bad feature token '3'"),
    ("1 1:2 x:3\n", "line 1: bad feature token 'x:3'"),
    ("\n\n1 0:2\n", "line 3: feature index 0 < 1"),
    ("1 2:1 2:3\n", "line 1: feature indices must be strictly increasing"),
    ("1 1:0x1p3\n", "line 1: bad feature token '1:0x1p3'"),
    ("1 1:1__0\n", "line 1: bad feature token '1:1__0'"),
])
def test_errors_match_reference_messages(text, msg):
    with pytest.raises(D.DataFormatError) as ei:
        D.parse_svmlight(text)
    assert str(ei.value) == msg


def test_non_finite_feature_rejected_like_reference():
    with pytest.raises(ValueError, match="non-finite"):
        D.parse_svmlight("1 1:inf\n")


def test_exotic_separators_use_the_line_path():
    text = "1 1:2\x1f2:3\n-1 1:1\n"        # str.split() separates at \x1f; the ASCII grammar not
    _same(D.parse_svmlight(text), D._parse_svmlight_lines(text.splitlines()))
