"""Where the plugin call's time goes (C2, 1 GPU): pinned H2D / D2H of the
call's bytes alone, the whole glm_device_solve call (host buffers), and the
same solve on device-resident inputs.  Host wall clock, medians of 30."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1803_06333_b200 as g
from paper_1803_06333_b200.solver import device_solve_host

torch.cuda.set_device(0)
indptr, rows, vals, y = bench.gen_columns(0, bench.N_EX // bench.BLOCK)
m, d = len(indptr) - 1, bench.D_FEAT


def med(f, n=30):
    for _ in range(3):
        f()
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        t = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return 1e3 * float(np.median(ts))


hb = torch.empty(m + d, dtype=torch.float64, pin_memory=True)
db = torch.empty(m + d, dtype=torch.float64, device="cuda")
print("h2d_ms", round(med(lambda: db.copy_(hb, non_blocking=True)), 4), "bytes", 8 * (m + d))
print("d2h_ms", round(med(lambda: hb.copy_(db, non_blocking=True)), 4), "bytes", 8 * (m + d))
import ctypes
from paper_1803_06333_b200 import _lib
h = ctypes.c_void_p()
_lib.check(_lib.lib().glm_ctx_create(0, _lib.CSC, d, m, indptr.ctypes.data_as(ctypes.c_void_p),
                                     rows.ctypes.data_as(ctypes.c_void_p),
                                     vals.ctypes.data_as(ctypes.c_void_p), ctypes.byref(h)), "ctx")
pin = lambda n: torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
lin, base, dl, dvb = pin(d), pin(m), pin(m), pin(d)
base[:] = 0.5
v0 = np.bincount(rows, weights=0.5 * vals, minlength=d)      # first round: v0 = A alpha0
lin[:] = v0 / bench.LAM
spec = g.ObjectiveSpec("dual_l2_logistic", bench.LAM, bench.N_EX, bench.D_FEAT)
sub = g.LocalSubproblem(spec=spec, lin=lin, quad=1.0 / bench.LAM,
                        const=float(v0 @ v0) / (2.0 * bench.LAM), base=base, data=None,
                        col_ids=np.arange(m))
st = g.derive_seed(0, 0)
print("plugin_call_ms", round(med(lambda: device_solve_host(h, sub, st, 1.0, 1, 1, out=(dl, dvb))), 4))
_lib.lib().glm_ctx_destroy(h)
