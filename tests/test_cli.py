"""CLI contract (cli.py:27-300 of the reference): exit codes on CPU; train /
predict / eval / chunk artefacts on the GPU against the reference's own
trained model on its bundled dataset (tests/golden/predict.npz)."""

import io

import numpy as np
import pytest

from paper_1803_06333_b200 import cli
from paper_1803_06333_b200.data import SparseColumnMatrix, write_svmlight


def _tiny_svm(golden, path):
    d = golden("data")
    ex = SparseColumnMatrix(int(d["ex_n_rows"]), d["ex_indptr"], d["ex_rows"], d["ex_vals"],
                            validate=False)
    buf = io.StringIO()
    write_svmlight(ex, d["ex_labels"], buf)
    path.write_text(buf.getvalue())
    return path


def test_usage_errors_exit_2(tmp_path, capsys):
    assert cli.main(["train", "--data", str(tmp_path / "missing.svm")]) == cli.EXIT_USAGE
    cfg = tmp_path / "bad.cfg"
    cfg.write_text("lambda 0.5\n")
    assert cli.main(["--config", str(cfg), "train", "--data", "x"]) == cli.EXIT_USAGE
    assert cli.main(["predict", "--model", str(tmp_path / "none.bin"),
                     "--data", "x"]) == cli.EXIT_USAGE
    with pytest.raises(SystemExit):
        cli.main(["train", "--data", "x", "--objective", "kernel"])


@pytest.mark.gpu
def test_train_predict_eval_match_reference(golden, tmp_path, capsys):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    data = _tiny_svm(golden, tmp_path / "tiny.svm")
    z = golden("predict")
    cfg = tmp_path / "run.cfg"
    cfg.write_text("# config file (keys are flag dests; flags win)\nlam = 0.5\nepochs = 2\nseed = 99\n")
    model, trace = tmp_path / "m.bin", tmp_path / "trace.csv"
    rc = cli.main(["--config", str(cfg), "train", "--data", str(data), "--objective",
                   "dual-logistic", "--max-rounds", "5", "--seed", "3", "--model-out",
                   str(model), "--trace-out", str(trace)])
    assert rc == cli.EXIT_OK
    out = capsys.readouterr().out
    assert out.startswith("rounds=5 objective=") and "logloss=" in out
    rows = np.loadtxt(trace, delimiter=",", skiprows=1, usecols=(0, 3))
    np.testing.assert_allclose(rows[:, 1], z["dual_l2_logistic_objective"], rtol=1e-10)
    scores = tmp_path / "scores.csv"
    assert cli.main(["predict", "--model", str(model), "--data", str(data), "--scores-out",
                     str(scores)]) == cli.EXIT_OK
    got = np.loadtxt(scores, delimiter=",", skiprows=1)
    assert np.max(np.abs(got[:, 1] - z["dual_l2_logistic_prob"])) < 1e-12
    np.testing.assert_array_equal(got[:, 2], np.where(z["dual_l2_logistic_prob"] >= 0.5, 1, -1))
    assert cli.main(["eval", "--model", str(model), "--data", str(data)]) == cli.EXIT_OK
    line = capsys.readouterr().out.strip().splitlines()[-1]
    ll = float(line.split()[0].split("=")[1])
    assert ll == pytest.approx(float(z["dual_l2_logistic_logloss"]), rel=1e-10)


@pytest.mark.gpu
def test_chunk_then_streamed_training_converges_like_in_memory(golden, tmp_path, capsys):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    data = _tiny_svm(golden, tmp_path / "tiny.svm")
    store = tmp_path / "tiny.chunks"
    assert cli.main(["chunk", "--data", str(data), "--chunk-size", "30", "--out",
                     str(store)]) == cli.EXIT_OK
    assert "chunks=4" in capsys.readouterr().out
    objs = []
    for extra in (["--data", str(data)],
                  ["--data", str(store), "--data-format", "chunks", "--pipeline", "on",
                   "--device-budget-mb", "0.001", "--stage-log-out", str(tmp_path / "s.csv")]):
        trace = tmp_path / "t.csv"
        rc = cli.main(["train", "--lambda", "0.5", "--epochs", "2", "--max-rounds", "60",
                       "--target-gap", "1e-10", "--model-out", str(tmp_path / "m.bin"),
                       "--trace-out", str(trace)] + extra)
        assert rc == cli.EXIT_OK
        objs.append(np.loadtxt(trace, delimiter=",", skiprows=1, usecols=(3,))[-1])
    assert objs[1] == pytest.approx(objs[0], rel=1e-9)
    stages = (tmp_path / "s.csv").read_text().splitlines()
    assert stages[0] == "epoch,chunk,load_ms,rand_ms,train_ms,step_ms"
