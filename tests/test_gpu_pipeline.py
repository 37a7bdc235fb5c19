"""GPU parity of the out-of-core streaming pipeline (csrc/stream.cu) vs the
reference's chunked_device_runner (pipeline.py:298-340): the reference's own
golden trace, the CPU oracle's chunked epoch at larger sizes, and the
property that streaming (device budget < data) gives the same bits as a
resident run and as a sequential in-memory schedule."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_1803_06333_b200 as g  # noqa: E402
from paper_1803_06333_b200 import _lib  # noqa: E402
from paper_1803_06333_b200 import pipeline as P  # noqa: E402


def _golden_matrix(z):
    return g.SparseColumnMatrix(int(z["m_n_rows"]), z["m_indptr"], z["m_rows"], z["m_vals"],
                                validate=False)


def _synth(n, d, k, seed, labels=True):
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.integers(0, d - k + 1, size=(n, k)), axis=1) + np.arange(k)
    vals = rng.standard_normal((n, k))
    vals /= np.linalg.norm(vals, axis=1, keepdims=True)
    if labels:
        vals *= np.where(rng.standard_normal(n) >= 0, 1.0, -1.0)[:, None]
    indptr = np.arange(0, n * k + 1, k, dtype=np.int64)
    return g.SparseColumnMatrix(d, indptr, rows.reshape(-1).astype(np.int32), vals.reshape(-1))


def _train(m, spec, runner, rounds, epochs, seed):
    eng = g.Engine(m, spec, g.HierarchyConfig(t1=rounds, seed=seed, epochs=epochs),
                   chunk_runner=runner)
    return eng.train(g.StoppingCriteria(max_rounds=rounds))


def test_chunked_runner_matches_reference_golden(golden, tmp_path):
    """The reference's chunk store + Engine(chunk_runner=chunked_device_runner)
    trace (tests/golden/make_golden.py gen_chunked)."""
    z = golden("chunked")
    m = _golden_matrix(z)
    spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, m.n_cols, m.n_rows)
    g.write_chunks(m, int(z["chunk_size"]), tmp_path / "t.chunks")
    store = g.open_chunks(tmp_path / "t.chunks")
    for budget in (None, 1):          # all resident / every chunk streamed
        runner = P.chunked_device_runner(store, seed=3, epochs=2, pipelined=True,
                                         device_budget=budget)
        assert (runner.partition.n_resident == runner.partition.n_chunks) == (budget is None)
        res = _train(m, spec, runner, 3, 2, 3)
        np.testing.assert_allclose(res.trace.objectives(), z["objective"], rtol=1e-12)
        np.testing.assert_allclose(res.model.alpha, z["alpha"], atol=1e-9)
        np.testing.assert_allclose(res.v, z["v"], atol=1e-9)
        runner.partition.close()


@pytest.mark.parametrize("kind", ["dual_l2_logistic", "dual_l2_svm"])
def test_chunked_vs_oracle_streamed(kind):
    """A 7-chunk partition (ragged last chunk) streamed through 2 device slots
    vs the oracle's chunked epochs (pipeline.py:158-197)."""
    m = _synth(20_000, 3_000, 12, 4)
    om = oracle.OMatrix(m.n_rows, m.indptr, m.rows, m.vals)
    k = 0 if kind == "dual_l2_logistic" else 1
    spec = g.ObjectiveSpec(kind, 1.0, m.n_cols, m.n_rows)
    chunk = 3_100
    part = P.StreamingPartition(m, chunk_size=chunk, device_budget=1)
    assert part.n_resident == 0 and part.n_chunks == 7
    runner = P.chunked_device_runner(part, seed=11, epochs=2)
    res = _train(m, spec, runner, 3, 2, 11)
    want = oracle.train_chunked(om, k, 1.0, chunk, epochs=2, seed=11, rounds=3)
    np.testing.assert_allclose(res.trace.objectives(), want["objective"], rtol=1e-10)
    np.testing.assert_allclose(res.model.alpha, want["alpha"], atol=1e-7)
    part.close()


def test_streamed_equals_resident_bits_host_and_file(tmp_path):
    """Residency / source (pinned DMA, staged pageable, GLMCHUNK file) never
    changes the result: sequential mode is bit-identical across all of them."""
    m = _synth(9_000, 1_500, 10, 7)
    spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, m.n_cols, m.n_rows)
    g.write_chunks(m, 1_000, tmp_path / "s.chunks")
    store = g.open_chunks(tmp_path / "s.chunks")
    outs = []
    for src, budget, pin, dio in [("host", None, False, False), ("host", 1, False, False),
                                  ("host", 1, True, False), ("file", 1, False, False),
                                  ("file", 600_000, False, False), ("file", 1, False, True)]:
        kw = dict(direct_io=True, io_threads=4) if dio else {}
        part = P.StreamingPartition(store if src == "file" else m, chunk_size=1_000,
                                    device_budget=budget, pin_host=pin, **kw)
        if budget == 600_000:
            assert 0 < part.n_resident < part.n_chunks      # resident prefix + streaming
        runner = P.chunked_device_runner(part, seed=5, epochs=3)
        res = _train(m, spec, runner, 2, 3, 5)
        outs.append((res.trace.objectives(), res.model.alpha))
        part.close()
    for obj, alpha in outs[1:]:
        np.testing.assert_array_equal(obj, outs[0][0])
        np.testing.assert_array_equal(alpha, outs[0][1])


def test_file_stream_direct_io_and_striped_reads(tmp_path):
    """Chunk bodies of 12 MB read from a GLMCHUNK file with O_DIRECT (aligned
    supersets into the pinned staging buffers; buffered where the file system
    refuses it) and with 4 concurrent stripes: the same bits as the buffered
    single-thread reader and as the resident run."""
    m = _synth(400_000, 20_000, 10, 11)
    spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, m.n_cols, m.n_rows)
    g.write_chunks(m, 100_000, tmp_path / "big.chunks")
    store = g.open_chunks(tmp_path / "big.chunks")
    outs = []
    for budget, kw in [(None, {}), (1, {}), (1, dict(io_threads=4)),
                       (1, dict(direct_io=True, io_threads=4)), (1, dict(direct_io=True))]:
        part = P.StreamingPartition(store, device_budget=budget, **kw)
        if budget == 1:
            assert part.n_resident == 0
        runner = P.chunked_device_runner(part, seed=3, epochs=2)
        res = _train(m, spec, runner, 1, 2, 2)
        outs.append((res.trace.objectives(), res.model.alpha, part.direct_io))
        part.close()
    for obj, alpha, _ in outs[1:]:
        np.testing.assert_array_equal(obj, outs[0][0])
        np.testing.assert_array_equal(alpha, outs[0][1])
    print("O_DIRECT active:", outs[3][2])


def test_host_buffers_runner_drop_in():
    """The reference-facing call shape: numpy LocalSubproblem, the reference's
    damping object mutated in place, SubtaskResult with numpy arrays; delta_v
    equals B delta (test_solver.py:160-169)."""
    m = _synth(6_000, 800, 8, 9)
    om = oracle.OMatrix(m.n_rows, m.indptr, m.rows, m.vals)
    spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, m.n_cols, m.n_rows)
    alpha = spec.init_alpha()
    v = oracle.matvec(om, alpha)
    lin = oracle.f_grad(0, 1.0, None, v)
    fv = oracle.f_eval(0, 1.0, None, v)
    sub = g.LocalSubproblem(spec=spec, lin=lin, quad=1.0, const=fv, base=alpha, data=m,
                            col_ids=np.arange(m.n_cols))
    part = P.StreamingPartition(m, chunk_size=1_500, device_budget=1)
    runner = P.chunked_device_runner(part, seed=2, epochs=3)

    class Dev:
        damping = g.DampingState()

    res = runner(sub, Dev(), None)
    assert isinstance(res.delta_alpha, np.ndarray) and res.epochs_run == 3
    dv = oracle.matvec(om, res.delta_alpha)
    assert np.max(np.abs(res.delta_v - dv)) < 1e-9 * max(1.0, np.max(np.abs(dv)))
    # oracle: the same three chunked epochs
    delta = np.zeros(m.n_cols)
    view = lin.copy()
    damping = 1.0
    offsets = np.array([0, 1500, 3000, 4500, 6000], dtype=np.int64)
    vals = []
    for e in range(3):
        st, val, damping = oracle.chunked_epoch(0, 1.0, om, lin, 1.0, fv, alpha, offsets, 2, e,
                                                delta, view, damping)
        assert st == 0
        vals.append(val)
    np.testing.assert_allclose(res.epoch_values, vals, rtol=1e-11)
    np.testing.assert_allclose(res.delta_alpha, delta, atol=1e-9)
    assert np.all(np.diff(res.epoch_values) <= 0)
    part.close()


def test_pipelined_epoch_context_in_place():
    """pipelined_epoch(store, ctx) continues from ctx.delta / ctx.view
    (pipeline.py:200-242) and two single-epoch calls equal one 2-epoch solve."""
    m = _synth(4_000, 600, 6, 13)
    spec = g.ObjectiveSpec("dual_l2_svm", 1.0, m.n_cols, m.n_rows)
    lin = np.zeros(m.n_rows)
    sub = g.LocalSubproblem(spec=spec, lin=lin, quad=1.0, const=0.0, base=spec.init_alpha(),
                            data=m, col_ids=np.arange(m.n_cols))
    part = P.StreamingPartition(m, chunk_size=700, device_budget=1)
    ctx = P.ChunkedSolveContext(sub=sub, delta=np.zeros(m.n_cols), view=lin.copy(),
                                chunk_offsets=list(part.offsets[:-1]), seed=4)
    damp = g.DampingState()
    v1, sched = P.pipelined_epoch(part, ctx, damping=damp)
    ctx.epoch_index = 1
    v2, _ = P.pipelined_epoch(part, ctx, damping=damp)
    assert len(sched.steps) == part.n_chunks
    sched.assert_buffer_safety()
    st, delta, values, info, scal, dmp = part.solve(spec, lin, 1.0, 0.0, sub.base, seed=4,
                                                    epoch_index=0, epochs=2)
    assert st == 0
    np.testing.assert_allclose([v1, v2], values, rtol=1e-12)
    np.testing.assert_allclose(ctx.delta, delta[:m.n_cols], atol=1e-12)
    part.close()


def test_async_stream_with_resumed_chunks():
    """Asynchronous chunk passes on a narrow shared vector (heavy conflicts)
    with one attempt enqueued per chunk: chunks that need retries are resumed
    by the host loop; the accepted values never increase and Delta v = B delta."""
    m = _synth(30_000, 64, 16, 21)
    om = oracle.OMatrix(m.n_rows, m.indptr, m.rows, m.vals)
    spec = g.ObjectiveSpec("dual_l2_logistic", 0.05, m.n_cols, m.n_rows)
    alpha = spec.init_alpha()
    v = oracle.matvec(om, alpha)
    lin = oracle.f_grad(0, 0.05, None, v)
    part = P.StreamingPartition(m, chunk_size=5_000, device_budget=1)
    dv = np.zeros(m.n_rows)
    st, delta, values, info, scal, dmp = part.solve(
        spec, lin, 20.0, 0.0, alpha, seed=1, epoch_index=0, epochs=4, mode=_lib.MODE_ASYNC,
        dv_out=dv, attempts_per_chunk=1, max_inflight=4096)
    assert st == 0 and info[0] == 4
    assert np.all(np.diff(np.concatenate([[scal[0]], values])) <= 1e-12 * abs(scal[0]))
    exact = oracle.matvec(om, delta[:m.n_cols])
    assert np.max(np.abs(dv - exact)) < 1e-8 * max(1.0, np.max(np.abs(exact)))
    part.close()


def test_empty_and_single_chunk_edges():
    m = _synth(10, 40, 4, 3)
    spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, m.n_cols, m.n_rows)
    om = oracle.OMatrix(m.n_rows, m.indptr, m.rows, m.vals)
    for offsets in ([0, 10], [0, 0, 4, 4, 10]):      # one chunk / with empty chunks
        part = P.StreamingPartition(m, chunk_offsets=offsets, device_budget=1)
        lin = oracle.f_grad(0, 1.0, None, oracle.matvec(om, spec.init_alpha()))
        st, delta, values, info, scal, dmp = part.solve(spec, lin, 1.0, 0.0, spec.init_alpha(),
                                                        seed=0, epoch_index=0, epochs=2)
        assert st == 0 and len(values) == 2 and values[1] <= values[0] <= scal[0]
        part.close()


@pytest.mark.parametrize("kind,k", [("ridge_primal", 2), ("lasso_primal", 3)])
def test_chunked_primal_kinds_vs_oracle(kind, k):
    """Primal kinds stream feature columns (the GLMCHUNK row vector is the
    target b, cli.py:182-185): streamed chunked epochs vs the oracle's."""
    rng = np.random.default_rng(17)
    m = _synth(3_000, 4_000, 20, 17, labels=False)          # columns = features
    om = oracle.OMatrix(m.n_rows, m.indptr, m.rows, m.vals)
    b = rng.standard_normal(m.n_rows)
    spec = g.ObjectiveSpec(kind, 0.5, m.n_rows, m.n_cols, target=b)
    part = P.StreamingPartition(m, chunk_size=700, device_budget=1)
    runner = P.chunked_device_runner(part, seed=6, epochs=2)
    res = _train(m, spec, runner, 3, 2, 6)
    want = oracle.train_chunked(om, k, 0.5, 700, target=b, epochs=2, seed=6, rounds=3)
    np.testing.assert_allclose(res.trace.objectives(), want["objective"], rtol=1e-10)
    np.testing.assert_allclose(res.model.alpha, want["alpha"], atol=1e-8)
    part.close()
