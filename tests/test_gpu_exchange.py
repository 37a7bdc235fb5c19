"""The fused Delta v exchange + round start (csrc/peer.cu) against the
unfused engine round (solve -> all-reduce -> v += total -> outer model ->
begin): identical bits in deterministic mode, on one GPU and — when the box
has two — across two processes over NVLink peer memory vs the deterministic
NCCL reducer (all-gather + ascending-rank fold = canonical_sum)."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_1803_06333_b200 as g  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _synth(n, d, k, seed):
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.integers(0, d - k + 1, size=(n, k)), axis=1) + np.arange(k)
    vals = rng.standard_normal((n, k))
    vals /= np.linalg.norm(vals, axis=1, keepdims=True)
    vals *= np.where(rng.standard_normal(n) >= 0, 1.0, -1.0)[:, None]
    indptr = np.arange(0, n * k + 1, k, dtype=np.int64)
    return g.SparseColumnMatrix(d, indptr, rows.reshape(-1).astype(np.int32), vals.reshape(-1))


@pytest.mark.parametrize("retry_budget", [4, 0])
@pytest.mark.parametrize("kind", ["dual_l2_logistic", "dual_l2_svm", "ridge_primal",
                                  "lasso_primal", "logistic_primal"])
def test_fused_round_bit_identical_single_gpu(kind, retry_budget):
    """retry_budget 0: one attempt per round, the round ends in glm_round_turn
    (value + finalize + exchange + next round start in one kernel)."""
    from paper_1803_06333_b200.objectives import KINDS
    m = _synth(6_000, 900, 8, 3)
    om = oracle.OMatrix(m.n_rows, m.indptr, m.rows, m.vals)
    if kind in ("ridge_primal", "lasso_primal"):
        tgt = np.random.default_rng(1).standard_normal(m.n_rows)
        spec = g.ObjectiveSpec(kind, 1.0, m.n_rows, m.n_cols, target=tgt)
        k = KINDS.index(kind)
    elif kind == "logistic_primal":
        tgt = np.where(np.random.default_rng(1).standard_normal(m.n_rows) >= 0, 1.0, -1.0)
        spec = g.ObjectiveSpec(kind, 1.0, m.n_rows, m.n_cols, target=tgt)
        k = KINDS.index(kind)
    else:
        tgt = None
        spec = g.ObjectiveSpec(kind, 1.0, m.n_cols, m.n_rows)
        k = 0 if kind == "dual_l2_logistic" else 1
    cfg = g.HierarchyConfig(t1=6, seed=5, epochs=2 if retry_budget else 1)
    runs = []
    for peer in (False, True):
        eng = g.Engine(m, spec, cfg, mode="sequential", sync_solves=False,
                       retry_budget=retry_budget, peer_exchange=peer)
        assert (eng.exchange is not None) == peer
        runs.append(eng.train(g.StoppingCriteria(max_rounds=6)))
    np.testing.assert_array_equal(runs[0].trace.objectives(), runs[1].trace.objectives())
    np.testing.assert_array_equal(runs[0].model.alpha, runs[1].model.alpha)
    np.testing.assert_array_equal(runs[0].v, runs[1].v)
    want = oracle.train(om, k, 1.0, target=tgt, epochs=cfg.epochs, seed=5, rounds=6)
    np.testing.assert_allclose(runs[1].trace.objectives(), want["objective"], rtol=1e-10)


def test_fused_round_long_delta_v_bit_identical():
    """A Delta v of 2^20 + 3 rows: the turn runs two blocks per SM with every
    row pass of P1 and P3 taking several rows per thread — the same bits as
    the unfused rounds, and the oracle's trace (C4's 10M-row regime, small)."""
    m = _synth(3_000, (1 << 20) + 3, 8, 7)
    om = oracle.OMatrix(m.n_rows, m.indptr, m.rows, m.vals)
    spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, m.n_cols, m.n_rows)
    cfg = g.HierarchyConfig(t1=4, seed=8, epochs=1)
    runs = []
    for peer in (False, True):
        eng = g.Engine(m, spec, cfg, mode="sequential", sync_solves=False, retry_budget=0,
                       peer_exchange=peer)
        assert (eng.exchange is not None) == peer
        runs.append(eng.train(g.StoppingCriteria(max_rounds=4)))
        eng.close()
    np.testing.assert_array_equal(runs[0].trace.objectives(), runs[1].trace.objectives())
    np.testing.assert_array_equal(runs[0].model.alpha, runs[1].model.alpha)
    np.testing.assert_array_equal(runs[0].v, runs[1].v)
    want = oracle.train(om, 0, 1.0, epochs=1, seed=8, rounds=4)
    np.testing.assert_allclose(runs[1].trace.objectives(), want["objective"], rtol=1e-10)


def test_fused_round_reset_and_graph_replay():
    """reset() drops the pending Delta v; a captured graph of fused rounds
    replays to the same trajectory as eager rounds."""
    m = _synth(20_000, 2_000, 10, 8)
    spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, m.n_cols, m.n_rows)
    eng = g.Engine(m, spec, g.HierarchyConfig(seed=2, epochs=1), mode="sequential",
                   sync_solves=False, retry_budget=0)
    for _ in range(4):
        eng.outer_round()
    v_eager, a_eager = eng.v, eng.alpha
    eng.reset()
    graph = eng.capture(4)
    eng.reset()
    graph.replay()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(eng.alpha, a_eager)
    np.testing.assert_array_equal(eng.v, v_eager)


def _why(out):
    """The child's own traceback (torchrun's summary follows it on stderr)."""
    err = out.stderr
    i = err.find("Traceback (most recent call last)")
    head = err[i:i + 4000] if i >= 0 else err[-3000:]
    return out.stdout[-1500:] + "\n--- stderr ---\n" + head


def _free_port():
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def _torchrun(*extra, timeout=600, script="mp_exchange_check.py", nproc=2, env=None):
    return subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
         f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1",
         "--master-port", str(_free_port()), os.path.join(ROOT, "tests", script), *extra],
        capture_output=True, text=True, timeout=timeout, cwd=ROOT,
        env=None if env is None else dict(os.environ, **env))


def test_two_process_exchange_matches_nccl():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    out = _torchrun()
    assert out.returncode == 0, _why(out)
    assert "HOST ALLREDUCE OK" in out.stdout, out.stdout[-2000:]
    assert "EXCHANGE OK" in out.stdout, out.stdout[-2000:]
    assert "GRAPH async OK" in out.stdout, out.stdout[-2000:]


@pytest.mark.parametrize("rs", ["0", "1"])
def test_two_process_exchange_same_gpu(rs):
    """Both ranks on cuda:0 (gloo bootstrap, time-sliced contexts): the IPC
    mappings, the pushed flag words, the parity double buffer and the
    rank-ordered sum of csrc/peer.cu across two processes, bit-identical to the
    deterministic reducer and to the in-process K = 2 engine; then the benched
    kernel configuration (async, cache_flags=1, fused turn) replayed from a
    CUDA graph across the ranks, with v = A alpha afterwards.  rs = 1 runs the
    turn's exchange as reduce-scatter + all-gather over peer memory (the
    default from 3 ranks up): the same bits."""
    out = _torchrun("--same-gpu", env={"GLM_PEER_RS": rs})
    assert out.returncode == 0, _why(out)
    assert "EXCHANGE OK" in out.stdout, out.stdout[-2000:]
    assert "GRAPH sequential OK" in out.stdout and "GRAPH async OK" in out.stdout, \
        out.stdout[-2000:]


@pytest.mark.parametrize("rs", ["0", "1"])
def test_three_process_exchange_same_gpu(rs):
    """Three ranks on cuda:0: an odd world, and with rs = 1 the reduce-scatter
    slices 1024 / 1024 / 952 rows of the 3000-row Delta v (a ragged last slice)
    — bit-identical to the deterministic reducer and the in-process K = 3
    engine."""
    out = _torchrun("--same-gpu", nproc=3, env={"GLM_PEER_RS": rs})
    assert out.returncode == 0, _why(out)
    assert "EXCHANGE OK" in out.stdout, out.stdout[-2000:]
    assert "GRAPH sequential OK" in out.stdout and "GRAPH async OK" in out.stdout, \
        out.stdout[-2000:]


def test_dead_rank_surfaces_as_error():
    """Rank 1 dies mid-training; rank 0's device-side waits hit their deadline
    (3 s here; the reference's DEFAULT_TIMEOUT is 60 s, comm.py:30) and the
    engine raises instead of spinning forever (engine.py:284-288)."""
    out = _torchrun("--same-gpu", "--kill", timeout=300)
    assert "TIMEOUT OK" in out.stdout or "TIMEOUT CUDA" in out.stdout, \
        out.stdout[-3000:] + out.stderr[-3000:]
    assert "NO ERROR" not in out.stdout


def test_hierarchical_ranks_same_gpu():
    """K = 2 nodes x L = 2 devices as four ranks on cuda:0 (gloo groups), t2 = 2
    inner rounds: the per-inner-round node fold and the outer node sum across
    processes equal the in-process two-level engine bit for bit."""
    out = _torchrun("--same-gpu", "--nodes", "2", "--devices", "2", "--t2", "2",
                    script="mp_hier_check.py", nproc=4)
    assert out.returncode == 0, _why(out)
    assert "HIER OK" in out.stdout, out.stdout[-2000:]


def test_hierarchical_ranks_multi_gpu():
    n = torch.cuda.device_count()
    if n < 4:
        pytest.skip("needs 4 GPUs")
    out = _torchrun("--nodes", "2", "--devices", "2", "--t2", "3", script="mp_hier_check.py",
                    nproc=4)
    assert out.returncode == 0, _why(out)
    assert "HIER OK" in out.stdout, out.stdout[-2000:]
