"""Kernel timeline of fused rounds on the C2 workload (debug, 1 GPU, graph
replay): per round the epoch, the first and last permutation kernel (side
stream) and the round turn, from %globaltimer stamps (glm_debug_timeline)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1803_06333_b200 as g
from paper_1803_06333_b200 import _lib as L
from paper_1803_06333_b200.data import DeviceMatrix
torch.cuda.set_device(0)
# SHARE=k: the 1/k share of the examples one rank owns at k GPUs
indptr, rows, vals, y = bench.gen_columns(0, (bench.N_EX // bench.BLOCK) // int(os.environ.get("SHARE", "1")))
dm = DeviceMatrix.from_csc(bench.D_FEAT, indptr, rows, vals)
spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, bench.N_EX, bench.D_FEAT)
eng = g.Engine(dm, spec, g.HierarchyConfig(t1=10**6, seed=0, epochs=1), mode="async",
               sync_solves=False, retry_budget=0, cache_flags=1)
for _ in range(3):
    eng.outer_round()
eng.reset()
ROUNDS = int(os.environ.get("TL_ROUNDS", "1"))
graph = eng.capture(ROUNDS)       # ROUNDS fused rounds per replay (stamps: first start, last end)
slots = torch.zeros(16, dtype=torch.int64, device="cuda")
init = torch.tensor([2**63 - 1, 0] * 8, dtype=torch.int64, device="cuda")
L.check(L.lib().glm_debug_timeline(slots.data_ptr()), "timeline")
rows_ = []
eng.reset()
for r in range(40):
    slots.copy_(init)
    torch.cuda.synchronize()
    graph.replay()
    torch.cuda.synchronize()
    s = slots.cpu().numpy().astype(np.float64)
    t0 = s[0]
    rows_.append([(s[i] - t0) / 1e3 if s[i] not in (0, 2**63 - 1) else np.nan for i in range(12)])
L.lib().glm_debug_timeline(None)
med = np.nanmedian(np.array(rows_[5:]), axis=0)
names = ["epoch start", "epoch end", "perm first start", "perm first end", "perm last start",
         "perm last end", "turn start", "turn end", "perm scan start", "perm scan end",
         "perm scatter start", "perm scatter end"]
for n, v in zip(names, med):
    print(f"{n:18s} {v:9.2f} us")
if ROUNDS > 1:
    span = med[1] - med[0]
    print(f"{ROUNDS} rounds: first epoch start -> last epoch end {span:.1f} us, "
          f"{span / ROUNDS:.1f} us per round (epoch end -> turn end of the last round "
          f"{med[7] - med[1]:.1f} us)")

