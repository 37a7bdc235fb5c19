"""bench.py's output contract, end to end on the GPU: one short run prints one
JSON line with the keys and types the driver reads (metric / value / unit /
n_gpus / steps == --steps / warmup / ms_per_step / higher_is_better / scaling /
vs_baseline / dtype / data / config.workload / e2e with its copy bytes /
gpu_launches / clocks / roofline with traffic and peak), and exits 0; the
reference arm prints its own line with impl = "reference"."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=timeout, cwd=ROOT,
                         env=dict(os.environ, CUDA_VISIBLE_DEVICES="0"))
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _line("--steps", "7", "--warmup", "3", "--no-cpu", "--no-primal", "--no-ttt")
    assert d["metric"] and d["unit"] == "epochs/s" and d["value"] > 0
    assert d["n_gpus"] == 1 and d["steps"] == 7 and d["warmup"] == 3
    assert d["ms_per_step"] == pytest.approx(1000.0 / d["value"], rel=1e-9)
    assert d["higher_is_better"] is True and d["scaling"] in ("strong", "weak")
    assert d["vs_baseline"] is None and d["dtype"] and d["data"] == "synthetic"
    assert "workload" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert isinstance(d["gpu_launches"], int) and d["gpu_launches"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] == "GB/s"
    assert r["peak"] > 0 and r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-9)
    assert r["traffic"] is None or r["traffic"] > 0
    assert d["cpu_baseline"] is None            # --no-cpu


def test_reference_arm_contract():
    d = _line("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "epochs/s"
    c = d["cpu_baseline"]
    assert c["kind"] in ("reference", "port") and c["cores"] >= 1 and c["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def test_bench_line_contract_two_gpus():
    """Under torchrun (one process per GPU): rank 0 alone prints the line,
    n_gpus = 2, every process exits 0."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node=2", "--master-addr", "127.0.0.1", "--master-port",
                          str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps",
                          "6", "--warmup", "3", "--no-ttt"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 6 and d["value"] > 0 and d["e2e"]["value"] > 0
