"""Host-side logic on CPU: configs, partitions, objective constants, file
formats (byte-exact with the reference), svmlight parsing and validation."""

import io
import math

import numpy as np
import pytest

import paper_1803_06333_b200 as g
from paper_1803_06333_b200 import data as D
from paper_1803_06333_b200 import modelio


def test_hierarchy_config_validation_and_defaults():
    with pytest.raises(ValueError):
        g.HierarchyConfig(nodes=0)
    cfg = g.HierarchyConfig(nodes=3, devices=2)
    assert cfg.sigma_eff == 3.0 and cfg.sigma_bar_eff == 2.0
    cfg = g.HierarchyConfig(nodes=3, devices=2, sigma=1.5, sigma_bar=0.5)
    assert cfg.sigma_eff == 1.5 and cfg.sigma_bar_eff == 0.5


def test_partitions_match_reference(golden):
    z = golden("data")
    for key in z:
        if not key.startswith("part_"):
            continue
        _, n, K, L, bal = key.split("_")
        n, K, L, bal = int(n), int(K), int(L), int(bal)
        b = D.partition_bounds(n, K, L, "balanced-by-nnz" if bal else "contiguous",
                               z["nnz_skew"] if bal else None)
        np.testing.assert_array_equal(b, z[key])
        parts = D.partition_columns(n, K, L, "balanced-by-nnz" if bal else "contiguous",
                                    z["nnz_skew"] if bal else None)
        assert [(p.node, p.device) for p in parts] == [(w // L, w % L) for w in range(K * L)]
        assert np.array_equal(np.concatenate([p.cols for p in parts]), np.arange(n))


def test_partition_errors():
    with pytest.raises(D.PartitionError):
        D.partition_columns(3, 2, 2)
    with pytest.raises(D.PartitionError):
        D.partition_columns(10, 1, 2, strategy="balanced-by-nnz")
    with pytest.raises(D.PartitionError):
        D.partition_columns(10, 1, 2, strategy="nope")


def test_objective_constants_table():
    # test_objectives.py:192-201 of the reference
    rows = [("dual_l2_logistic", 2.0, 0.5, 4.0, math.inf),
            ("dual_l2_svm", 2.0, 0.5, 0.0, math.sqrt(10)),
            ("ridge_primal", 2.0, 1.0, 2.0, math.inf),
            ("lasso_primal", 2.0, 1.0, 0.0, math.inf)]
    for kind, lam, beta, mu, radius in rows:
        tgt = None if kind.startswith("dual") else np.zeros(3)
        spec = g.ObjectiveSpec(kind, lam, 10, 3, target=tgt)
        assert spec.beta == beta and spec.mu == mu and spec.support_radius == radius
    spec = g.ObjectiveSpec("logistic_primal", 2.0, 3, 10, target=np.ones(3))
    assert spec.beta == 0.25 and spec.mu == 2.0 and spec.n_coordinates == 10


def test_objective_spec_errors():
    from paper_1803_06333_b200.objectives import UnsupportedObjectiveError
    with pytest.raises(UnsupportedObjectiveError):
        g.ObjectiveSpec("hinge_loss_svm", 1.0, 2, 2)
    with pytest.raises(ValueError, match="requires a target"):
        g.ObjectiveSpec("hinge_primal", 1.0, 2, 2)
    with pytest.raises(ValueError, match="smoothing"):
        g.ObjectiveSpec("hinge_primal", 1.0, 2, 2, target=np.ones(2), smoothing=0.0)
    hs = g.ObjectiveSpec("hinge_primal", 1.0, 2, 2, target=np.array([1.0, -1.0]), smoothing=0.25)
    assert hs.beta == 4.0 and hs.has_gap
    np.testing.assert_array_equal(hs.row_target, [4.0, -4.0])
    with pytest.raises(ValueError):
        g.ObjectiveSpec("ridge_primal", 1.0, 2, 2)
    with pytest.raises(ValueError):
        g.ObjectiveSpec("dual_l2_svm", 0.0, 2, 2)
    spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, 3, 2)
    with pytest.raises(ValueError):
        spec.check_alpha(np.array([0.5, 1.0, 0.2]))
    np.testing.assert_array_equal(spec.init_alpha(), [0.5, 0.5, 0.5])


def _golden_chunk_matrix(z):
    return D.SparseColumnMatrix(int(z["ch_n_rows"]), z["ch_indptr"], z["ch_rows"], z["ch_vals"],
                                z["ch_labels"])


def test_chunk_store_bytes_match_reference(golden, tmp_path):
    z = golden("data")
    m = _golden_chunk_matrix(z)
    blob = z["chunk_bytes"].tobytes()
    # the row vector is the payload right after the 32-byte header
    rv = np.frombuffer(blob[32:32 + 8 * m.n_rows], dtype="<f8")
    D.write_chunks(m, 5, tmp_path / "a.chunks", row_vector=rv)
    assert (tmp_path / "a.chunks").read_bytes() == blob
    store = D.open_chunks(tmp_path / "a.chunks")
    assert [c.n_cols for c in store.chunks] == [5, 5, 5, 5, 3]
    np.testing.assert_array_equal(store.row_vector, rv)
    back = D.concat_chunks(store)
    assert back.value_equal(m)
    np.testing.assert_array_equal(back.labels, m.labels)


def test_chunk_store_errors(tmp_path):
    p = tmp_path / "junk.chunks"
    p.write_bytes(b"NOTMAGIC" + b"\x00" * 24)
    with pytest.raises(D.ChunkFormatError, match="bad magic"):
        D.open_chunks(p)
    m = D.SparseColumnMatrix(4, [0, 1, 2], [0, 3], [1.0, 2.0])
    D.write_chunks(m, 1, tmp_path / "t.chunks")
    blob = (tmp_path / "t.chunks").read_bytes()
    (tmp_path / "t.chunks").write_bytes(blob[:-7])
    with pytest.raises(D.ChunkFormatError):
        store = D.open_chunks(tmp_path / "t.chunks")
        D.read_chunk(store, store.n_chunks - 1)


def test_model_file_bytes_match_reference(golden, tmp_path):
    z = golden("data")
    spec = g.ObjectiveSpec("dual_l2_logistic", 0.5, 23, 9)
    modelio.save_model(tmp_path / "m.bin", spec, np.linspace(0.1, 0.9, 23), np.arange(9.0))
    assert (tmp_path / "m.bin").read_bytes() == z["model_bytes"].tobytes()
    got = modelio.load_model(tmp_path / "m.bin")
    assert got["kind"] == "dual_l2_logistic" and got["lam"] == 0.5
    np.testing.assert_array_equal(got["v"], np.arange(9.0))
    np.testing.assert_array_equal(modelio.primal_weights(got), np.arange(9.0) / 0.5)


def test_parse_svmlight_and_errors(golden):
    z = golden("data")
    lines = []
    for j in range(len(z["ex_labels"])):
        lo, hi = z["ex_indptr"][j], z["ex_indptr"][j + 1]
        feats = " ".join("%d:%.17g" % (r + 1, v) for r, v in zip(z["ex_rows"][lo:hi],
                                                                  z["ex_vals"][lo:hi]))
        lines.append("%+g %s" % (z["ex_labels"][j], feats))
    m, y = D.parse_svmlight("\n".join(lines))
    np.testing.assert_array_equal(m.indptr, z["ex_indptr"])
    np.testing.assert_array_equal(m.rows, z["ex_rows"])
    np.testing.assert_array_equal(m.vals, z["ex_vals"])
    np.testing.assert_array_equal(y, z["ex_labels"])
    buf = io.StringIO()
    D.write_svmlight(m, y, buf)
    m2, y2 = D.parse_svmlight(buf.getvalue())
    assert m2.value_equal(m)
    for bad, frag in [("1 0:1", "< 1"), ("1 3:1 2:1", "increasing"), ("x 1:1", "bad label"),
                      ("1 a:b", "bad feature")]:
        with pytest.raises(D.DataFormatError, match=frag):
            D.parse_svmlight(bad)


def test_matrix_validation_messages():
    with pytest.raises(ValueError, match="span"):
        D.SparseColumnMatrix(3, [0, 2], [0], [1.0])
    with pytest.raises(ValueError, match="range"):
        D.SparseColumnMatrix(3, [0, 1], [5], [1.0])
    with pytest.raises(ValueError, match="strictly increasing"):
        D.SparseColumnMatrix(3, [0, 2], [2, 1], [1.0, 1.0])
    with pytest.raises(ValueError, match="non-finite"):
        D.SparseColumnMatrix(3, [0, 1], [1], [np.nan])
    # trailing empty columns are valid (the reference raises IndexError here,
    # data.py:80; documented divergence)
    m = D.SparseColumnMatrix(5, [0, 0, 2, 2, 3, 3], [1, 4, 0], [1.5, -2.0, 0.25])
    assert m.n_cols == 5 and m.nnz == 3


def test_trace_csv_schema(tmp_path):
    from paper_1803_06333_b200.engine import ConvergenceTrace, TraceRow
    tr = ConvergenceTrace()
    tr.append(TraceRow(0, 0.0, 0.0, 1.5, None, None))
    tr.append(TraceRow(1, 0.1, 2.0, 1.25, 0.5, None))
    tr.write_csv(tmp_path / "t.csv")
    lines = (tmp_path / "t.csv").read_text().splitlines()
    assert lines[0] == "round,wall_s,sim_cost,objective,gap,theta"
    assert lines[1] == "0,0.0,0.0,1.5,,"
    assert lines[2] == "1,0.1,2.0,1.25,0.5,"
