"""Disk -> HBM streaming of a Criteo-shaped GLMCHUNK file:
the native loader reads chunk bodies with pread into pinned staging and
copies them into the device slots while the previous chunk trains.

Writes an N-example C5-shaped file (bench_configs.criteo_block) to PATH, then
times streamed epochs (1 GB device budget, every chunk streamed) with
  buffered reads (page cache, warm after the write; read-ahead advice),
  O_DIRECT reads (page cache bypassed: the device itself) with 1 and 8 stripes.
One JSON line.   python tools/disk_stream.py [N=8000000] [PATH]
"""
import json
import os
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_1803_06333_b200 as g  # noqa: E402
from paper_1803_06333_b200 import _lib as L  # noqa: E402
from paper_1803_06333_b200 import pipeline as P  # noqa: E402
from bench_configs import criteo_block  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
path = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "c5.chunks")
torch.cuda.set_device(0)
d, k = 1 << 20, 39
nnz = n * k
indptr = np.arange(0, nnz + 1, k, dtype=np.int64)
rows = np.empty(nnz, dtype=np.int32)
vals = np.empty(nnz, dtype=np.float64)
w = np.random.default_rng(55).standard_normal(d)
B = 1_000_000
for lo in range(0, n, B):
    hi = min(n, lo + B)
    r, v = criteo_block(np.random.default_rng([55, lo // B]), hi - lo, d, w)
    rows[lo * k:hi * k] = r.reshape(-1)
    vals[lo * k:hi * k] = v.reshape(-1)
m = g.SparseColumnMatrix(d, indptr, rows, vals, validate=False)
t0 = time.perf_counter()
store = g.write_chunks(m, 1_000_000, path)
t_write = time.perf_counter() - t0
size = os.path.getsize(path)
del rows, vals
fs = subprocess.run(["df", "-T", os.path.dirname(path)], capture_output=True, text=True).stdout
spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, n, d)
lin = torch.zeros(d, dtype=torch.float64, device="cuda")
base = np.full(n, 0.5)
res = {"config": "C5-disk", "examples": n, "file_bytes": size, "write_s": t_write,
       "filesystem": fs.strip().splitlines()[-1] if fs.strip() else None}
for name, kw in (("buffered", {}), ("buffered_8", dict(io_threads=8)),
                 ("o_direct_1", dict(direct_io=True)), ("o_direct_8", dict(direct_io=True, io_threads=8))):
    part = P.StreamingPartition(store, device_budget=1 << 30, **kw)
    times = []
    for e in range(3):
        st, delta, values, info, scal, dmp = part.solve(
            spec, lin, 1.0, 0.0, base, seed=1, epoch_index=e, epochs=1, mode=L.MODE_ASYNC,
            timing=True)
        assert st == 0, st
        times.append(float(scal[2]))
    streamed = size * (part.n_chunks - part.n_resident) / part.n_chunks
    ms = float(np.median(times[1:]))
    res[name] = {"epoch_ms": ms, "disk_to_hbm_GBps": streamed / (ms * 1e-3) / 1e9,
                 "o_direct_active": part.direct_io, "chunks": part.n_chunks,
                 "resident": part.n_resident, "epoch_ms_all": times}
    part.close()
os.remove(path)
print(json.dumps(res), flush=True)
