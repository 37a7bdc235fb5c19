"""Phase timestamps of glm_round_turn on the C2 workload (debug)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1803_06333_b200 as g
from paper_1803_06333_b200 import _lib as L
from paper_1803_06333_b200.data import DeviceMatrix
torch.cuda.set_device(0)
torch.cuda.set_stream(torch.cuda.Stream(priority=-100 if os.environ.get("HIPRI") else 0))
indptr, rows, vals, y = bench.gen_columns(0, bench.N_EX // bench.BLOCK)
dm = DeviceMatrix.from_csc(bench.D_FEAT, indptr, rows, vals)
spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, bench.N_EX, bench.D_FEAT)
eng = g.Engine(dm, spec, g.HierarchyConfig(t1=10**6, seed=0, epochs=1), mode="async",
               sync_solves=False, retry_budget=0, cache_flags=1)
st = torch.zeros(8, dtype=torch.int64, device="cuda")
L.check(L.lib().glm_peer_stamps(eng.exchange.handle, st.data_ptr()), "stamps")
for _ in range(5):
    eng.outer_round()
ph = []
for _ in range(30):
    eng.outer_round()
    torch.cuda.synchronize()
    s = st.cpu().numpy().astype(np.int64)
    ph.append(np.concatenate([np.diff(s[:5]), [s[5] - s[0], s[6] - s[0], s[7] - s[0]]]) / 1e3)
print("us: P1 decide | P2 publish | wait peers | P3 round start | blk0 view loads | blk0 reduced | last block starts ->", np.median(ph, axis=0))
