"""Generate golden parity fixtures by running the REFERENCE implementation.

This script is the pin for `oracle/`: it imports the reference package
`hierglm` (pure Python/NumPy, read-only under /root/reference/pkg) and records
its outputs on small seeded inputs into `tests/golden/*.npz`. The fixtures are
committed; the GPU box never sees /root/reference.

Run from the repo root (only in the build container):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every block cites the reference function whose output it freezes.
"""

from __future__ import annotations

import io
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg"
sys.path[:0] = [REF + "/src", REF]
sys.dont_write_bytecode = True

from hierglm import data as rdata  # noqa: E402
from hierglm import engine as rengine  # noqa: E402
from hierglm import modelio as rmodelio  # noqa: E402
from hierglm import objectives as robj  # noqa: E402
from hierglm import pipeline as rpipe  # noqa: E402
from hierglm import solver as rsolver  # noqa: E402
from hierglm import cli as rcli  # noqa: E402
from tests import synth as rsynth  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
KINDS = robj.KINDS


def _save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def _mat(prefix, m):
    out = {prefix + "n_rows": np.int64(m.n_rows), prefix + "indptr": m.indptr,
           prefix + "rows": m.rows, prefix + "vals": m.vals}
    if m.labels is not None:
        out[prefix + "labels"] = m.labels
    return out


def instance(kind, n, d, nnz, lam, seed):
    """Reference synth instance (tests/synth.py:32-61) for any of the 4 kinds."""
    if kind.startswith("dual_"):
        m, spec, _ = rsynth.dual_instance(kind, n, d, nnz, lam, seed)
    else:
        m, spec, _ = rsynth.primal_instance(kind, d, n, nnz, lam, seed)
    return m, spec


# --------------------------------------------------------------------------
# PRNG: solver.py:41-89, pipeline.py:29-78
# --------------------------------------------------------------------------
def gen_prng():
    seeds = np.array([0, 1, 13, 42, 2 ** 63 + 5, 0xDEADBEEFCAFEF00D], dtype=np.uint64)
    idx = np.array([0, 1, 7, 1000, 2 ** 40], dtype=np.uint64)
    ds1 = np.array([[rsolver.derive_seed(int(s), int(i)) for i in idx] for s in seeds],
                   dtype=np.uint64)
    ds2 = np.array([[rsolver.derive_seed(int(s), int(i), int(j)) for j in (0, 3, 99)]
                    for s in seeds for i in (0, 5)], dtype=np.uint64)
    xs = []
    for s in seeds:
        st = int(s) or 1
        row = []
        for _ in range(5):
            st = rsolver.xorshift64_step(st)
            row.append(st)
        xs.append(row)
    xs = np.array(xs, dtype=np.uint64)
    sm = np.array([rsolver.splitmix64(int(s)) for s in seeds], dtype=np.uint64)
    # permutation streams: two consecutive permutes from one generator
    perm_cases = []
    arrays = {}
    for c, (seed, n) in enumerate([(1, 1), (123, 100), (9, 50), (rsolver.derive_seed(13, 0), 10),
                                   (rsolver.derive_seed(5, 3), 4097), (0, 33),
                                   (777, 20000)]):
        gen = rsolver.PermutationGenerator(seed)
        s0 = gen.state
        keys = rsolver.PermutationGenerator(seed).keys(n)
        p1 = gen.permute(n)
        s1 = gen.state
        p2 = gen.permute(n)
        s2 = gen.state
        perm_cases.append((seed, n))
        arrays[f"perm{c}_keys"] = keys
        arrays[f"perm{c}_p1"] = p1
        arrays[f"perm{c}_p2"] = p2
        arrays[f"perm{c}_states"] = np.array([s0, s1, s2], dtype=np.uint64)
    arrays["perm_cases"] = np.array(perm_cases, dtype=np.uint64)
    gk = []
    for c, (seed, n) in enumerate([(7, 5), (42, 1), (42, 100), (42, 4096), (42, 5000),
                                   (42, 9001), (rsolver.derive_seed(3, 2, 1), 12345)]):
        arrays[f"gk{c}"] = rpipe.generate_keys(seed, n)
        arrays[f"gk{c}_perm"] = rpipe.keys_to_permutation(arrays[f"gk{c}"])
        gk.append((seed, n))
    arrays["gk_cases"] = np.array(gk, dtype=np.uint64)
    _save("prng", derive1_seeds=seeds, derive1_idx=idx, derive1=ds1, derive2=ds2,
          xorshift=xs, splitmix=sm, **arrays)


# --------------------------------------------------------------------------
# coordinate_update KATs: solver.py:152-187
# --------------------------------------------------------------------------
def gen_coord():
    rng = np.random.default_rng(4)
    rows_all = []
    for kind in KINDS:
        spec = robj.ObjectiveSpec(kind, 0.7, 4, 4, target=np.zeros(4))
        for trial in range(200):
            nnz = int(rng.integers(0, 5))
            rows = np.sort(rng.choice(4, size=nnz, replace=False)).astype(np.int32)
            vals = rng.standard_normal(nnz)
            view = rng.standard_normal(4) * 2
            sq = float(vals @ vals)
            quad = float(rng.uniform(0.1, 3.0))
            if kind == "dual_l2_logistic":
                t = float(rng.uniform(1e-6, 1 - 1e-6)) if trial % 7 else 1e-12
            elif kind == "dual_l2_svm":
                t = float(rng.choice([0.0, 1.0, rng.uniform(0, 1)]))
            else:
                t = float(rng.standard_normal())
            vrow = np.zeros(4)
            vrow[:nnz] = vals
            rrow = np.full(4, -1, np.int32)
            rrow[:nnz] = rows
            step = rsolver.coordinate_update(spec, rows, vals, sq, t, view, quad)
            ga = float(np.dot(vals, view[rows])) if nnz else 0.0
            rows_all.append((KINDS.index(kind), nnz, *rrow, *vrow, *view, sq, t, quad,
                             0.7, ga, step))
    _save("coord", table=np.array(rows_all, dtype=np.float64))


# --------------------------------------------------------------------------
# damped_solve: solver.py:250-305 (sequential, n_threads=1)
# --------------------------------------------------------------------------
SOLVE_CASES = [
    # kind, n coords, d, nnz/col, lam, seed, sigma, epochs, gen seed
    ("dual_l2_logistic", 120, 40, 5, 1.0, 3, 1.0, 3, 11),
    ("dual_l2_logistic", 300, 60, 6, 0.3, 4, 2.0, 2, 12),
    ("dual_l2_svm", 150, 50, 4, 1.0, 5, 1.0, 3, 13),
    ("dual_l2_svm", 90, 200, 7, 0.5, 6, 4.0, 2, 14),
    ("ridge_primal", 40, 120, 8, 0.5, 7, 1.0, 3, 15),
    ("ridge_primal", 25, 300, 30, 2.0, 8, 3.0, 4, 16),
    ("lasso_primal", 40, 120, 8, 0.5, 9, 1.0, 3, 17),
    ("lasso_primal", 60, 80, 10, 0.05, 10, 2.0, 5, 18),
]


def gen_solve():
    arrays = {}
    for c, (kind, n, d, nnz, lam, seed, sigma, epochs, gseed) in enumerate(SOLVE_CASES):
        m, spec = instance(kind, n, d, nnz, lam, seed)
        rng = np.random.default_rng(seed + 100)
        alpha = spec.init_alpha()
        if kind == "dual_l2_logistic":
            alpha = np.clip(alpha + rng.uniform(-0.3, 0.3, len(alpha)), 0.01, 0.99)
        elif kind == "dual_l2_svm":
            alpha = rng.uniform(0, 1, len(alpha)) * (rng.random(len(alpha)) < 0.5)
        else:
            alpha = rng.standard_normal(len(alpha)) * 0.1
        v = m.matvec(alpha)
        sub = rsolver.LocalSubproblem(spec=spec, lin=robj.f_grad(spec, v),
                                      quad=sigma * spec.beta, const=robj.f_eval(spec, v),
                                      base=alpha.copy(), data=m,
                                      col_ids=np.arange(m.n_cols))
        gen = rsolver.PermutationGenerator(gseed)
        state = rsolver.DampingState()
        res = rsolver.damped_solve(sub, gen, epochs, n_threads=1, damping=state)
        p = f"c{c}_"
        arrays.update(_mat(p, m))
        arrays[p + "kind"] = np.int64(KINDS.index(kind))
        arrays[p + "lam"] = np.float64(lam)
        arrays[p + "target"] = spec.target if spec.target is not None else np.zeros(0)
        arrays[p + "lin"] = sub.lin
        arrays[p + "quad"] = np.float64(sub.quad)
        arrays[p + "const"] = np.float64(sub.const)
        arrays[p + "base"] = sub.base
        arrays[p + "gen_seed"] = np.uint64(gseed)
        arrays[p + "epochs"] = np.int64(epochs)
        arrays[p + "delta"] = res.delta_alpha
        arrays[p + "dv"] = res.delta_v
        arrays[p + "values"] = np.array(res.epoch_values)
        arrays[p + "initial"] = np.float64(res.initial_subproblem_value)
        arrays[p + "final"] = np.float64(res.final_subproblem_value)
        arrays[p + "epochs_run"] = np.int64(res.epochs_run)
        arrays[p + "retries"] = np.int64(res.retries)
        arrays[p + "gen_state"] = np.uint64(gen.state)
        arrays[p + "damping"] = np.float64(state.delta)
        arrays[p + "sqnorms"] = m.col_sqnorms()
        w = rng.standard_normal(m.n_rows)
        x = rng.standard_normal(m.n_cols)
        arrays[p + "mv_x"] = x
        arrays[p + "mv"] = m.matvec(x)
        arrays[p + "rmv_w"] = w
        arrays[p + "rmv"] = m.rmatvec(w)
        # objective math at alpha (objectives.py:129-234)
        arrays[p + "alpha"] = alpha
        arrays[p + "fv"] = np.float64(robj.f_eval(spec, v))
        arrays[p + "gsum"] = np.float64(robj.g_sum(spec, alpha))
        arrays[p + "primal"] = np.float64(robj.primal_objective(spec, m, alpha))
        arrays[p + "gap"] = np.float64(robj.duality_gap(spec, m, alpha, v)
                                       if kind != "lasso_primal" else np.nan)
    arrays["n_cases"] = np.int64(len(SOLVE_CASES))
    _save("solve", **arrays)


# --------------------------------------------------------------------------
# Engine traces: engine.py:169-423
# --------------------------------------------------------------------------
ENGINE_CASES = [
    # kind, n, d, nnz, lam, seed, nodes, devices, t2, epochs, rounds, cfg seed, strategy
    ("dual_l2_logistic", 500, 100, 5, 1.0, 909, 2, 2, 1, 2, 8, 13, "contiguous"),
    ("dual_l2_logistic", 500, 100, 5, 1.0, 909, 4, 1, 1, 2, 8, 13, "contiguous"),
    ("dual_l2_logistic", 200, 50, 5, 1.0, 14, 2, 2, 4, 1, 8, 2, "contiguous"),
    ("dual_l2_logistic", 100, 30, 4, 0.5, 21, 1, 1, 1, 3, 6, 0, "contiguous"),
    ("dual_l2_svm", 150, 60, 4, 1.0, 13, 2, 2, 2, 1, 6, 1, "contiguous"),
    ("dual_l2_svm", 240, 30, 3, 0.7, 16, 3, 1, 1, 2, 6, 9, "balanced-by-nnz"),
    ("ridge_primal", 60, 200, 8, 0.5, 31, 2, 1, 1, 2, 6, 4, "contiguous"),
    ("ridge_primal", 50, 150, 10, 1.0, 32, 1, 3, 2, 1, 6, 5, "contiguous"),
    ("lasso_primal", 60, 200, 8, 0.5, 33, 2, 2, 1, 2, 6, 6, "contiguous"),
    ("lasso_primal", 80, 120, 6, 0.1, 34, 1, 1, 1, 1, 6, 7, "contiguous"),
]


def gen_engine():
    arrays = {}
    for c, (kind, n, d, nnz, lam, seed, K, L, t2, ep, R, cs, strat) in enumerate(ENGINE_CASES):
        m, spec = instance(kind, n, d, nnz, lam, seed)
        cfg = rengine.HierarchyConfig(nodes=K, devices=L, t1=R, t2=t2, seed=cs, epochs=ep,
                                      partition_strategy=strat)
        res = rengine.train(m, spec, cfg, rengine.StoppingCriteria(max_rounds=R))
        p = f"c{c}_"
        arrays.update(_mat(p, m))
        arrays[p + "kind"] = np.int64(KINDS.index(kind))
        arrays[p + "lam"] = np.float64(lam)
        arrays[p + "target"] = spec.target if spec.target is not None else np.zeros(0)
        arrays[p + "cfg"] = np.array([K, L, t2, ep, R, cs], dtype=np.int64)
        arrays[p + "balanced"] = np.int64(strat != "contiguous")
        arrays[p + "objective"] = res.trace.objectives()
        arrays[p + "gap"] = np.array([np.nan if r.gap is None else r.gap
                                      for r in res.trace.rows])
        arrays[p + "alpha"] = res.model.alpha
        arrays[p + "v"] = res.v
    arrays["n_cases"] = np.int64(len(ENGINE_CASES))
    _save("engine", **arrays)


# --------------------------------------------------------------------------
# Data layer: data.py:42-304, cli.py:146-185
# --------------------------------------------------------------------------
def gen_data():
    arrays = {}
    rng = np.random.default_rng(77)
    m = rsynth.sparse_columns(37, 53, 6, rng, normalize=False)
    t = m.transpose()
    arrays.update(_mat("m_", m))
    arrays.update(_mat("t_", t))
    cols = np.array([5, 0, 52, 17, 17, 3], dtype=np.int64)
    s = m.select_columns(cols)
    arrays["sel_cols"] = cols
    arrays.update(_mat("s_", s))
    scales = rng.standard_normal(53)
    arrays["scales"] = scales
    arrays.update(_mat("sc_", m.scale_columns(scales)))
    arrays["sqnorms"] = m.col_sqnorms()
    # empty columns inside
    # validate=False: the reference _validate (data.py:80) raises IndexError when the
    # last column is empty; the golden freezes the arithmetic, not that quirk
    m2 = rdata.SparseColumnMatrix(5, [0, 0, 2, 2, 3, 3], [1, 4, 0], [1.5, -2.0, 0.25],
                                  validate=False)
    arrays.update(_mat("e_", m2))
    arrays.update(_mat("et_", m2.transpose()))
    arrays["e_sqnorms"] = m2.col_sqnorms()
    arrays["e_mv"] = m2.matvec(np.arange(5, dtype=np.float64))
    arrays["e_rmv"] = m2.rmatvec(np.array([1.0, -1.0, 2.0, 0.5, 3.0]))
    # partitions
    parts = []
    nnz_skew = np.concatenate([np.full(10, 100), np.ones(90, dtype=np.int64)])
    for n, K, L, strat in [(10, 2, 2, "contiguous"), (7, 1, 1, "contiguous"),
                           (100, 2, 3, "contiguous"), (100, 2, 2, "balanced-by-nnz"),
                           (100, 1, 8, "balanced-by-nnz"), (1000003, 4, 2, "contiguous")]:
        ps = rdata.partition_columns(n, K, L, strategy=strat,
                                     col_nnz=nnz_skew if strat != "contiguous" else None)
        bounds = [int(p.cols[0]) for p in ps] + [int(ps[-1].cols[-1]) + 1]
        parts.append((n, K, L, strat != "contiguous", *bounds[:1], len(bounds)))
        arrays[f"part_{n}_{K}_{L}_{int(strat != 'contiguous')}"] = np.array(bounds, np.int64)
        assert all(np.array_equal(p.cols, np.arange(bounds[i], bounds[i + 1]))
                   for i, p in enumerate(ps))
    arrays["nnz_skew"] = nnz_skew
    # layout contract on the bundled dataset (cli.py:146-185)
    with open(REF + "/data/tiny_binary.svm") as fh:
        ex, labels = rdata.parse_svmlight(fh)
    arrays.update(_mat("ex_", ex))
    arrays["ex_labels"] = labels
    for kind in ("dual_l2_logistic", "ridge_primal"):
        mat, spec, y01, _ = rcli.load_training_data(REF + "/data/tiny_binary.svm",
                                                    "svmlight", kind, 1.0)
        arrays.update(_mat(("dual_" if kind.startswith("dual") else "primal_"), mat))
    # chunk store bytes (data.py:329-359) with labels + row vector
    m3 = rsynth.sparse_columns(9, 23, 3, rng, normalize=False)
    m3 = rdata.SparseColumnMatrix(m3.n_rows, m3.indptr, m3.rows, m3.vals,
                                  labels=rng.standard_normal(23))
    with tempfile.TemporaryDirectory() as td:
        rdata.write_chunks(m3, 5, td + "/a.chunks", row_vector=rng.standard_normal(9))
        arrays["chunk_bytes"] = np.frombuffer(open(td + "/a.chunks", "rb").read(), np.uint8)
        spec = robj.ObjectiveSpec("dual_l2_logistic", 0.5, 23, 9)
        rmodelio.save_model(td + "/m.bin", spec, np.linspace(0.1, 0.9, 23), np.arange(9.0))
        arrays["model_bytes"] = np.frombuffer(open(td + "/m.bin", "rb").read(), np.uint8)
    arrays.update(_mat("ch_", m3))
    _save("data", **arrays)


# --------------------------------------------------------------------------
# Prediction / metrics: modelio.py:57-99 via a trained model on tiny_binary
# --------------------------------------------------------------------------
def gen_predict():
    arrays = {}
    path = REF + "/data/tiny_binary.svm"
    for kind in ("dual_l2_logistic", "dual_l2_svm", "ridge_primal"):
        mat, spec, y01, _ = rcli.load_training_data(path, "svmlight", kind, 0.5)
        res = rengine.train(mat, spec, rengine.HierarchyConfig(t1=5, seed=3, epochs=2),
                            rengine.StoppingCriteria(max_rounds=5))
        model = {"kind": kind, "lam": 0.5, "alpha": res.model.alpha, "v": res.v}
        w = rmodelio.primal_weights(model)
        with open(path) as fh:
            ex, labels = rdata.parse_svmlight(fh)
        scores = rmodelio.decision_scores(ex, w)
        p = kind + "_"
        arrays[p + "w"] = w
        arrays[p + "scores"] = scores
        arrays[p + "alpha"] = res.model.alpha
        arrays[p + "v"] = res.v
        arrays[p + "objective"] = res.trace.objectives()
        if kind.startswith("dual_"):
            prob = rmodelio.sigmoid(scores)
            y = rmodelio.normalize_binary_labels(labels)
            arrays[p + "prob"] = prob
            arrays[p + "logloss"] = np.float64(rmodelio.log_loss(prob, y))
            arrays[p + "accuracy"] = np.float64(rmodelio.accuracy(prob, y))
        else:
            arrays[p + "mse"] = np.float64(rmodelio.mean_squared_error(scores, labels))
    _save("predict", **arrays)


# --------------------------------------------------------------------------
# Chunked device runner (pipeline.py:298-340): pipelined == sequential bits
# --------------------------------------------------------------------------
def gen_chunked():
    arrays = {}
    m, spec, _ = rsynth.dual_instance("dual_l2_logistic", 96, 24, 4, 1.0, 5)
    with tempfile.TemporaryDirectory() as td:
        store = rdata.write_chunks(m, 16, td + "/t.chunks")
        store = rdata.open_chunks(td + "/t.chunks")
        runner = rpipe.chunked_device_runner(store, seed=3, epochs=2, pipelined=True)
        eng = rengine.Engine(m, spec, rengine.HierarchyConfig(t1=3, seed=3, epochs=2),
                             chunk_runner=runner)
        res = eng.train(rengine.StoppingCriteria(max_rounds=3))
    arrays.update(_mat("m_", m))
    arrays["chunk_size"] = np.int64(16)
    arrays["objective"] = res.trace.objectives()
    arrays["alpha"] = res.model.alpha
    arrays["v"] = res.v
    _save("chunked", **arrays)


def gen_ingest():
    """rdata.parse_svmlight (data.py:190-239) on the shared seeded texts
    (tests/svm_texts.py): sha256 of (n_rows, indptr, rows, vals, labels), or
    the exception class and message it raised."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "svm_texts", os.path.join(os.path.dirname(OUT), "svm_texts.py"))
    svm_texts = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(svm_texts)
    names, digests = [], []
    for name, text in svm_texts.cases().items():
        names.append(name)
        try:
            m, y = rdata.parse_svmlight(text)
            digests.append(svm_texts.digest(m, y))
        except Exception as exc:          # the reference's error is the golden
            digests.append(svm_texts.error_key(exc))
    _save("ingest", names=np.array(names), digests=np.array(digests))


if __name__ == "__main__":
    if len(sys.argv) > 1:            # regenerate selected fixtures only
        for name in sys.argv[1:]:
            globals()["gen_" + name]()
        sys.exit(0)
    gen_ingest()
    gen_prng()
    gen_coord()
    gen_solve()
    gen_engine()
    gen_data()
    gen_predict()
    gen_chunked()
