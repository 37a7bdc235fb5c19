"""Pin the CPU oracle against the reference's own outputs (tests/golden/*.npz).

The fixtures were produced by running the reference `hierglm` package
(tests/golden/make_golden.py). If the oracle agrees with them, it is a valid
checker for the CUDA path (tests/test_gpu_*.py).
"""

import numpy as np
import pytest

import oracle
from oracle import OMatrix


def test_derive_seed_and_primitives(golden):
    z = golden("prng")
    for i, s in enumerate(z["derive1_seeds"]):
        for j, ix in enumerate(z["derive1_idx"]):
            assert oracle.derive_seed(int(s), int(ix)) == int(z["derive1"][i, j])
    row = 0
    for s in z["derive1_seeds"]:
        for ix in (0, 5):
            for c, jx in enumerate((0, 3, 99)):
                assert oracle.derive_seed(int(s), ix, jx) == int(z["derive2"][row, c])
            row += 1
    for i, s in enumerate(z["derive1_seeds"]):
        assert oracle.splitmix64(int(s)) == int(z["splitmix"][i])
        st = int(s) or 1
        for c in range(5):
            st = oracle.xorshift64_step(st)
            assert st == int(z["xorshift"][i, c])
    # Appendix B anchor
    assert oracle.derive_seed(13, 0) == 0xBC10FE74B44B54C8


def test_permutation_streams_bit_exact(golden):
    z = golden("prng")
    for c, (seed, n) in enumerate(z["perm_cases"]):
        seed, n = int(seed), int(n)
        keys, _ = oracle.perm_keys(seed, n)
        np.testing.assert_array_equal(keys, z[f"perm{c}_keys"])
        p1, s1 = oracle.permute(seed, n)
        p2, s2 = oracle.permute(s1, n)
        np.testing.assert_array_equal(p1, z[f"perm{c}_p1"])
        np.testing.assert_array_equal(p2, z[f"perm{c}_p2"])
        assert [s1, s2] == [int(x) for x in z[f"perm{c}_states"][1:]]


def test_chunk_keys_bit_exact(golden):
    z = golden("prng")
    for c, (seed, n) in enumerate(z["gk_cases"]):
        keys = oracle.generate_keys(int(seed), int(n))
        np.testing.assert_array_equal(keys, z[f"gk{c}"])
        np.testing.assert_array_equal(oracle.argsort_stable(keys), z[f"gk{c}_perm"])
    assert oracle.generate_keys(7, 5).tolist() == [3166046910, 1363937579, 3929783289,
                                                    2883719886, 180266347]


def test_coordinate_update_kats(golden):
    t = golden("coord")["table"]
    for row in t:
        kind, nnz = int(row[0]), int(row[1])
        rows = row[2:6].astype(np.int32)[:nnz]
        vals = row[6:10][:nnz]
        view = row[10:14]
        sq, tt, quad, lam, ga, step = row[14:20]
        got = oracle.coordinate_update(kind, lam, rows, vals, sq, tt, view, quad)
        assert got == pytest.approx(step, rel=1e-12, abs=1e-14), (kind, row)


def _solve_case(z, c):
    p = f"c{c}_"
    m = OMatrix.from_npz(z, p)
    tgt = z[p + "target"] if len(z[p + "target"]) else None
    return m, tgt, p


def test_damped_solve_matches_reference(golden):
    z = golden("solve")
    for c in range(int(z["n_cases"])):
        m, tgt, p = _solve_case(z, c)
        kind = int(z[p + "kind"])
        r = oracle.damped_solve(kind, float(z[p + "lam"]), m, z[p + "lin"], float(z[p + "quad"]),
                                float(z[p + "const"]), z[p + "base"], int(z[p + "gen_seed"]),
                                int(z[p + "epochs"]))
        assert r["status"] == 0
        assert r["epochs_run"] == int(z[p + "epochs_run"])
        assert r["retries"] == int(z[p + "retries"])
        assert r["gen_state"] == int(z[p + "gen_state"])
        assert r["damping"] == float(z[p + "damping"])
        np.testing.assert_allclose(r["values"], z[p + "values"], rtol=1e-12)
        assert r["initial"] == pytest.approx(float(z[p + "initial"]), rel=1e-13)
        np.testing.assert_allclose(r["delta"], z[p + "delta"], atol=1e-9)
        np.testing.assert_allclose(r["dv"], z[p + "dv"], atol=1e-9)


def test_matrix_and_objective_math(golden):
    z = golden("solve")
    for c in range(int(z["n_cases"])):
        m, tgt, p = _solve_case(z, c)
        kind, lam = int(z[p + "kind"]), float(z[p + "lam"])
        np.testing.assert_allclose(oracle.col_sqnorms(m), z[p + "sqnorms"], rtol=1e-13)
        np.testing.assert_allclose(oracle.matvec(m, z[p + "mv_x"]), z[p + "mv"], rtol=1e-12,
                                   atol=1e-13)
        np.testing.assert_allclose(oracle.rmatvec(m, z[p + "rmv_w"]), z[p + "rmv"],
                                   rtol=1e-12, atol=1e-13)
        a = z[p + "alpha"]
        v = oracle.matvec(m, a)
        assert oracle.f_eval(kind, lam, tgt, v) == pytest.approx(float(z[p + "fv"]), rel=1e-12)
        assert oracle.g_sum(kind, lam, a) == pytest.approx(float(z[p + "gsum"]), rel=1e-12)
        assert oracle.primal_objective(kind, lam, m, a, tgt) == pytest.approx(
            float(z[p + "primal"]), rel=1e-12)
        if kind != 3:
            assert oracle.duality_gap(kind, lam, m, a, v, tgt) == pytest.approx(
                float(z[p + "gap"]), rel=1e-10, abs=1e-10)


def test_engine_traces_match_reference(golden):
    z = golden("engine")
    for c in range(int(z["n_cases"])):
        p = f"c{c}_"
        m = OMatrix.from_npz(z, p)
        tgt = z[p + "target"] if len(z[p + "target"]) else None
        K, L, t2, ep, R, cs = (int(x) for x in z[p + "cfg"])
        strat = "balanced-by-nnz" if int(z[p + "balanced"]) else "contiguous"
        r = oracle.train(m, int(z[p + "kind"]), float(z[p + "lam"]), target=tgt, nodes=K,
                         devices=L, t2=t2, epochs=ep, seed=cs, rounds=R, strategy=strat)
        np.testing.assert_allclose(r["objective"], z[p + "objective"], rtol=1e-11)
        np.testing.assert_allclose(r["gap"], z[p + "gap"], rtol=1e-7, atol=1e-9)
        np.testing.assert_allclose(r["alpha"], z[p + "alpha"], atol=1e-8)
        np.testing.assert_allclose(r["v"], z[p + "v"], atol=1e-8)


def test_parallel_engine_is_identical_to_serial(golden):
    z = golden("engine")
    p = "c0_"
    m = OMatrix.from_npz(z, p)
    a = oracle.train(m, 0, 1.0, nodes=2, devices=2, epochs=2, seed=13, rounds=4)
    b = oracle.train(m, 0, 1.0, nodes=2, devices=2, epochs=2, seed=13, rounds=4,
                     parallel=True)
    np.testing.assert_array_equal(a["alpha"], b["alpha"])
    np.testing.assert_array_equal(a["objective"], b["objective"])


def test_layout_transforms_bit_exact(golden):
    z = golden("data")
    m = OMatrix.from_npz(z, "m_")
    t = oracle.transpose(m)
    for name in ("indptr", "rows", "vals"):
        np.testing.assert_array_equal(getattr(t, name), z["t_" + name])
    s = oracle.select_columns(m, z["sel_cols"])
    for name in ("indptr", "rows", "vals"):
        np.testing.assert_array_equal(getattr(s, name), z["s_" + name])
    sc = oracle.scale_columns(m, z["scales"])
    np.testing.assert_array_equal(sc.vals, z["sc_vals"])
    e = OMatrix.from_npz(z, "e_")
    et = oracle.transpose(e)
    np.testing.assert_array_equal(et.indptr, z["et_indptr"])
    np.testing.assert_array_equal(et.rows, z["et_rows"])
    np.testing.assert_array_equal(oracle.col_sqnorms(e), z["e_sqnorms"])
    np.testing.assert_array_equal(oracle.matvec(e, np.arange(5.0)), z["e_mv"])
    np.testing.assert_array_equal(oracle.rmatvec(e, np.array([1.0, -1.0, 2.0, 0.5, 3.0])),
                                  z["e_rmv"])


def test_partitions_bit_exact(golden):
    z = golden("data")
    for key in z:
        if not key.startswith("part_"):
            continue
        _, n, K, L, bal = key.split("_")
        n, K, L, bal = int(n), int(K), int(L), int(bal)
        b = oracle.partition_bounds(n, K, L, "balanced-by-nnz" if bal else "contiguous",
                                    z["nnz_skew"] if bal else None)
        np.testing.assert_array_equal(b, z[key])


def test_chunked_runner_matches_reference(golden):
    z = golden("chunked")
    m = OMatrix.from_npz(z, "m_")
    r = oracle.train_chunked(m, 0, 1.0, int(z["chunk_size"]), epochs=2, seed=3, rounds=3)
    np.testing.assert_allclose(r["objective"], z["objective"], rtol=1e-12)
    np.testing.assert_allclose(r["alpha"], z["alpha"], atol=1e-9)


def test_prediction_metrics(golden):
    z = golden("predict")
    d = golden("data")
    ex = OMatrix.from_npz(d, "ex_")
    for kind in ("dual_l2_logistic", "dual_l2_svm", "ridge_primal"):
        p = kind + "_"
        s = oracle.decision_scores(ex, z[p + "w"])
        np.testing.assert_allclose(s, z[p + "scores"], rtol=1e-12, atol=1e-14)
        if kind.startswith("dual_"):
            y = np.where(d["ex_labels"] > 0, 1.0, 0.0)
            prob = oracle.sigmoid(s)
            assert oracle.log_loss(prob, y) == pytest.approx(float(z[p + "logloss"]),
                                                             rel=1e-12)
            assert oracle.accuracy(prob, y) == float(z[p + "accuracy"])
