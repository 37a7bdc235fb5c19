"""The level-scheduled deterministic epoch (scd_seq_lvl, csrc/scd.cu): the
same bits as the one-warp sequential walk (scd_seq_csc, kept behind
GLM_SEQ_KERNEL=csc), and the reference's damped_solve (oracle, pinned by the
golden fixtures) at the full C2 size within the north star's 1e-6 relative
objective bar."""

import os
import sys
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_1803_06333_b200 as g  # noqa: E402


def _ragged(n, d, seed, max_nnz=60, long_every=0):
    """Columns of 0..max_nnz distinct rows (some empty); every `long_every`-th
    column has 150 rows (the > 96-entry tail path)."""
    rng = np.random.default_rng(seed)
    counts = rng.integers(0, min(max_nnz, d) + 1, size=n)
    if long_every:
        counts[::long_every] = 150
    indptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    rows = np.concatenate([np.sort(rng.choice(d, size=c, replace=False)) for c in counts]) \
        .astype(np.int32)
    vals = rng.standard_normal(len(rows))
    return g.SparseColumnMatrix(d, indptr, rows, vals)


def _solve(m, kind, lam, epochs, seed, env):
    spec = g.ObjectiveSpec(kind, lam, m.n_cols, m.n_rows)
    om = oracle.OMatrix(m.n_rows, m.indptr, m.rows, m.vals)
    alpha = spec.init_alpha()
    v = oracle.matvec(om, alpha)
    k = 0 if kind == "dual_l2_logistic" else 1
    lin = oracle.f_grad(k, lam, None, v)
    fv = oracle.f_eval(k, lam, None, v)
    sub = g.LocalSubproblem(spec=spec, lin=lin, quad=1.0 / lam, const=fv, base=alpha, data=m,
                            col_ids=np.arange(m.n_cols))
    old = os.environ.pop("GLM_SEQ_KERNEL", None)
    if env:
        os.environ["GLM_SEQ_KERNEL"] = env
    try:
        gen = g.PermutationGenerator(g.derive_seed(seed, 0))
        res = g.damped_solve(sub, gen, epochs, n_threads=1)
    finally:
        os.environ.pop("GLM_SEQ_KERNEL", None)
        if old is not None:
            os.environ["GLM_SEQ_KERNEL"] = old
    return res, gen.state, (k, lin, fv, alpha, om)


@pytest.mark.parametrize("n,d,long_every,kind", [
    (20_000, 3_000, 0, "dual_l2_logistic"),      # view in shared memory
    (60_000, 40_000, 37, "dual_l2_logistic"),    # view in L2, tail columns
    (50_000, 100_000, 0, "dual_l2_svm"),         # C2's d
    (3_000, 200, 0, "dual_l2_svm"),              # dense conflicts: many levels per window
    (1_000, 40, 0, "dual_l2_logistic"),          # up to 40 of 40 rows: > 15 levels per window
])
def test_level_kernel_bit_identical_to_one_warp_walk(n, d, long_every, kind):
    """The level-scheduled kernel (default) and GLM_SEQ_KERNEL=csc (the
    one-warp walk): identical bits."""
    m = _ragged(n, d, seed=n + d, long_every=long_every)
    cs, s_cs, _ = _solve(m, kind, 1.0, 3, 5, "csc")
    for env in (None,):
        lv, s_lv, _ = _solve(m, kind, 1.0, 3, 5, env)
        assert s_lv == s_cs and lv.epochs_run == cs.epochs_run and lv.retries == cs.retries
        assert np.asarray(lv.delta_alpha).tobytes() == np.asarray(cs.delta_alpha).tobytes(), env
        assert np.asarray(lv.delta_v).tobytes() == np.asarray(cs.delta_v).tobytes(), env
        assert list(lv.epoch_values) == list(cs.epoch_values), env


def test_full_c2_deterministic_epoch_vs_reference_oracle():
    """bench.py's C2 arrays (1M examples x 100k features, 40 nnz): two
    deterministic epochs against the oracle's damped_solve — epoch values,
    final objective within 1e-6 relative (north star; measured ~1e-13),
    delta_alpha within 1e-6 absolute, the generator state exact."""
    import bench
    indptr, rows, vals, _ = bench.gen_columns(0, bench.N_EX // bench.BLOCK)
    m = g.SparseColumnMatrix(bench.D_FEAT, indptr, rows, vals, validate=False)
    t0 = time.perf_counter()
    res, state, (k, lin, fv, alpha, om) = _solve(m, "dual_l2_logistic", bench.LAM, 2, 0, None)
    t_gpu = time.perf_counter() - t0
    want = oracle.damped_solve(k, bench.LAM, om, lin, 1.0 / bench.LAM, fv, alpha,
                               g.derive_seed(0, 0), 2)
    assert res.epochs_run == want["epochs_run"] and state == want["gen_state"]
    np.testing.assert_allclose(res.epoch_values, want["values"], rtol=1e-6)
    assert abs(res.final_subproblem_value - want["final"]) <= 1e-6 * abs(want["final"])
    assert np.max(np.abs(np.asarray(res.delta_alpha) - want["delta"])) < 1e-6
    print(f"C2 deterministic solve (2 epochs + setup): {t_gpu:.3f} s")
