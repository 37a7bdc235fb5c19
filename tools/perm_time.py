"""Warm, serial cost of the fused permutation (glm_perm: generate + stable
argsort, the solver's per-epoch permutation) at the per-rank sizes of C2 on
1/2/4/8 GPUs: 50 permutations captured back to back in one CUDA graph,
device-timed.  Also the per-kernel list under ncu (PERM_NCU=1: 3 eager calls)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1803_06333_b200 import _lib as L  # noqa: E402

lib = L.lib()
out = {}
for n in (1_000_000, 500_000, 250_000, 125_000):
    tb = lib.glm_argsort_temp_bytes(n)
    temp = torch.empty(tb, dtype=torch.uint8, device="cuda")
    perm = torch.empty(n, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()

    def call(state):
        L.check(lib.glm_perm(state, n, perm.data_ptr(), temp.data_ptr(), tb,
                             ctypes.c_void_p(s.cuda_stream)), "glm_perm")

    with torch.cuda.stream(s):
        call(12345)
    torch.cuda.synchronize()
    if os.environ.get("PERM_NCU"):
        with torch.cuda.stream(s):
            for i in range(3):
                call(777 + i)
        torch.cuda.synchronize()
        continue
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(50):
            call(1000 + i)
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s)
            g.replay()
            b.record(s)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 50 * 1e3)
    out[n] = round(best, 2)
    print(f"n={n}: {best:.2f} us per permutation (incl. glm_perm's counter memset)", flush=True)
print(json.dumps({"perm_us": out}))
