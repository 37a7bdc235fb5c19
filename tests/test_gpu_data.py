"""GPU data layer (csrc/data.cu) vs the reference's own arrays
(tests/golden/data.npz, made by running hierglm): transpose, select_columns,
scale_columns and the load_training_data layout contract bit-exact; column
norms / SpMV both ways to rounding; validation errors; and large randomized
transposes against numpy's stable argsort (data.py:155-165)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1803_06333_b200 as g  # noqa: E402
from paper_1803_06333_b200.data import DeviceMatrix  # noqa: E402


def _m(z, p):
    return g.SparseColumnMatrix(int(z[p + "n_rows"]), z[p + "indptr"], z[p + "rows"],
                                z[p + "vals"], validate=False)


def _eq(a, z, p):
    assert a.n_rows == int(z[p + "n_rows"])
    np.testing.assert_array_equal(a.indptr, z[p + "indptr"])
    np.testing.assert_array_equal(a.rows, z[p + "rows"])
    assert np.asarray(a.vals).tobytes() == np.asarray(z[p + "vals"]).tobytes()


def test_transpose_select_scale_bit_exact(golden):
    z = golden("data")
    m = _m(z, "m_")
    _eq(m.transpose(), z, "t_")
    _eq(m.select_columns(z["sel_cols"]), z, "s_")
    _eq(m.scale_columns(z["scales"]), z, "sc_")
    np.testing.assert_allclose(m.col_sqnorms(), z["sqnorms"], rtol=1e-14)
    e = _m(z, "e_")                                  # empty columns, last column empty
    _eq(e.transpose(), z, "et_")
    np.testing.assert_array_equal(e.col_sqnorms(), z["e_sqnorms"])
    np.testing.assert_allclose(e.matvec(np.arange(5, dtype=np.float64)), z["e_mv"], rtol=1e-15)
    np.testing.assert_allclose(e.rmatvec(np.array([1.0, -1.0, 2.0, 0.5, 3.0])), z["e_rmv"],
                               rtol=1e-15)


def test_layout_contract_bit_exact(golden):
    """load_training_data (cli.py:146-185) on the bundled dataset: dual kinds fold
    the labels into the example columns, primal kinds transpose."""
    from paper_1803_06333_b200 import cli
    z = golden("data")
    ex = _m(z, "ex_")
    y_pm = np.where(z["ex_labels"] > 0, 1.0, -1.0)
    _eq(ex.scale_columns(y_pm), z, "dual_")
    _eq(ex.transpose(), z, "primal_")
    assert cli.OBJECTIVE_NAMES["dual-logistic"] == "dual_l2_logistic"


@pytest.mark.parametrize("n,d,k,seed", [(1, 1, 1, 0), (5_000, 300, 7, 1), (200_003, 4_096, 33, 2)])
def test_transpose_random_vs_numpy_stable_argsort(n, d, k, seed):
    rng = np.random.default_rng(seed)
    nnz_col = rng.integers(0, k + 1, size=n)
    indptr = np.concatenate([[0], np.cumsum(nnz_col)]).astype(np.int64)
    rows = np.concatenate([np.sort(rng.choice(d, size=c, replace=False)) for c in nnz_col]
                          ).astype(np.int32) if indptr[-1] else np.zeros(0, np.int32)
    vals = rng.standard_normal(int(indptr[-1]))
    m = g.SparseColumnMatrix(d, indptr, rows, vals)
    t = m.transpose()
    cols = np.repeat(np.arange(n), np.diff(indptr))
    order = np.argsort(rows, kind="stable")
    np.testing.assert_array_equal(t.indptr, np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=d))]))
    np.testing.assert_array_equal(t.rows, cols[order])
    assert t.vals.tobytes() == vals[order].tobytes()
    # scale by a per-column factor and select a shuffled subset with repeats
    sc = rng.standard_normal(n)
    s = m.scale_columns(sc)
    assert s.vals.tobytes() == (vals * np.repeat(sc, np.diff(indptr))).tobytes()
    sel = rng.integers(0, n, size=min(n, 1000))
    ss = m.select_columns(sel)
    want_rows = np.concatenate([rows[indptr[j]:indptr[j + 1]] for j in sel]) if len(sel) else []
    np.testing.assert_array_equal(ss.rows, want_rows)


def test_dense_layout_and_norms():
    rng = np.random.default_rng(3)
    X = rng.standard_normal((57, 131))              # odd sizes: unaligned columns
    dm = DeviceMatrix.from_dense(X)
    sq = dm.col_sqnorms().cpu().numpy()
    np.testing.assert_allclose(sq, (X * X).sum(axis=0), rtol=1e-13)
    # a view starting mid-allocation (column 3 of 57 rows: an 8-byte-aligned start)
    sub = DeviceMatrix(57, 37, dm.layout, dm.vals[3 * 57:40 * 57])
    np.testing.assert_allclose(sub.col_sqnorms().cpu().numpy()[:37],
                               (X[:, 3:40] ** 2).sum(axis=0), rtol=1e-13)
    np.testing.assert_allclose(sub.rmatvec(np.ones(57)).cpu().numpy(), X[:, 3:40].sum(axis=0),
                               rtol=1e-12, atol=1e-12)
    sc = rng.standard_normal(131)
    out = dm.scale_columns(sc)
    got = out.vals.cpu().numpy().reshape(131, 57).T
    assert got.tobytes() == (X * sc).tobytes()
    w = rng.standard_normal(57)
    np.testing.assert_allclose(dm.rmatvec(w).cpu().numpy(), X.T @ w, rtol=1e-12)


def test_validation_errors():
    with pytest.raises(ValueError):
        g.SparseColumnMatrix(3, [0, 2], [2, 1], [1.0, 2.0]).device()   # not increasing
    dm = DeviceMatrix.from_csc(3, np.array([0, 1]), np.array([5], np.int32), np.array([1.0]),
                               validate=False)
    with pytest.raises(ValueError):
        DeviceMatrix.from_csc(3, np.array([0, 1]), np.array([5], np.int32), np.array([1.0]),
                              validate=True)
    assert dm.n_cols == 1
