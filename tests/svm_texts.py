"""Seeded svmlight texts shared by tests/test_ingest.py and the golden
generator (tests/golden/make_golden.py gen_ingest, which records the
REFERENCE parser's result on each of them as a digest)."""

import functools
import hashlib

import numpy as np

SPELLINGS = [lambda v: "%.17g" % v, lambda v: repr(float(v)), lambda v: "%.3e" % v,
             lambda v: "%.6f" % v, lambda v: "%+.5E" % v, lambda v: "%d" % int(v * 100),
             lambda v: ("%d" % int(v * 1e6)).replace("000", "_000"),
             lambda v: ".%d" % abs(int(v * 1000)), lambda v: "%d." % int(v * 10)]


def random_text(seed, n, d, k):
    rng = np.random.default_rng(seed)
    lines = ["# header comment", ""]
    for _ in range(n):
        y = rng.choice(["1", "-1", "0", "+1", "1.0", "2.5e-1", "-0"])
        feats = np.sort(rng.choice(d, size=rng.integers(0, k + 1), replace=False)) + 1
        toks = [f"{j}:{SPELLINGS[rng.integers(len(SPELLINGS))](rng.standard_normal())}"
                for j in feats]
        sep = rng.choice([" ", "\t", "  "])
        lines.append(sep.join([y] + toks) + rng.choice(["", " ", "\t"]))
    lines.append("  # trailing comment")
    return "\n".join(lines) + "\n"


# name -> text (each parsed as a str by both parsers).  Every text ends with
# an example that has a feature: the reference's _validate raises IndexError
# when the last column is empty (data.py:80; DESIGN §2 divergence 2).
@functools.lru_cache(maxsize=1)
def cases():
    return {
        "random_small": random_text(5, 3000, 500, 12)
        + "inf 5:1_0.5_0e1_0 6:-0.0\n-NaN 1:2\n-Infinity\n1 1:1\n",
        "random_large": random_text(9, 60_000, 20_000, 30) + "1 1:1\n",
        # separators Python's str.split()/splitlines() honour but plain ASCII
        # grammars do not, Unicode whitespace and decimal digits
        "exotic": "1 1:2\x1f2:3\n-1 1:1\x0b-1 2:5\n\x1c1 1:٣.5\r\n+1 3:1e١ 4:٠_٠ "
                  "5:0\n0 2:7\x85-1 1:2\xa02:1 1 1:3\n",
        "exotic_bad_digit": "1 1:2\n1 ٢:1 1:3\n",
        "exotic_bad_char": "1 1:2\n1 2:1²1\n",
        "exotic_bad_label": "1 1:2\x1d½ 2:1\n",
        "bad_token": "1 1:2 3\n",
        "bad_index": "\n\n1 0:2\n",
        "not_increasing": "1 2:1 2:3\n",
        "index_overflow": "1 1:1 2147483649:2\n-1 1:3\n",
        "overflow_then_format_error": "1 4294967296:2\n-1 1:3 z\n",
        "non_finite": "1 1:inf\n",
        "crlf_and_blank": "\r\n1 1:1\r\n\r\n# c\r\n-1 2:2\r\n",
        "empty": "",
        "only_comments": "# a\n   \n\t# b\n",
    }


def digest(matrix, labels):
    h = hashlib.sha256()
    h.update(np.int64(matrix.n_rows).tobytes())
    for a in (matrix.indptr, matrix.rows, matrix.vals, labels):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def error_key(exc):
    return f"err:{type(exc).__name__}:{exc}"
