"""Fused duality-gap kernels on the C2 workload (1 GPU): CUDA-event time per
glm_gap_terms call (gap_rows + gap_cols), medians of 50 after warm-up."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1803_06333_b200 as g
from paper_1803_06333_b200.data import DeviceMatrix

torch.cuda.set_device(0)
indptr, rows, vals, y = bench.gen_columns(0, bench.N_EX // bench.BLOCK)
dm = DeviceMatrix.from_csc(bench.D_FEAT, indptr, rows, vals)
spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, bench.N_EX, bench.D_FEAT)
eng = g.Engine(dm, spec, g.HierarchyConfig(t1=10**6, seed=0, epochs=1), mode="async",
               sync_solves=False, retry_budget=0, cache_flags=1)
for _ in range(3):
    eng.outer_round()
out = torch.zeros(4, dtype=torch.float64, device="cuda")
for _ in range(5):
    eng.gap_terms_async(out)
torch.cuda.synchronize()
ts = []
for _ in range(50):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    eng.gap_terms_async(out)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print("gap_terms_ms", round(float(np.median(ts)), 4), "nnz", int(indptr[-1]))
