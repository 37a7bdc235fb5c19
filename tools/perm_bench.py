"""Standalone permutation timing (glm_perm: generate + stable argsort on the
GPU, CUDA events, idle GPU; each call also zeroes its scratch) for a few
sizes.  Prints one JSON line per size."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1803_06333_b200 import _lib as L, _device as D

torch.cuda.set_device(0)
for n in [int(x) for x in (sys.argv[1:] or ["100000", "1000000", "2000000"])]:
    perm = torch.empty(n, dtype=torch.int32, device="cuda")
    nb = L.lib().glm_argsort_temp_bytes(n)
    tmp = torch.empty(nb, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    call = lambda i: L.check(L.lib().glm_perm(12345 + i, n, D.ptr(perm), D.ptr(tmp), nb,
                                              s.cuda_stream), "glm_perm")
    for i in range(5):
        call(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    e0.record()
    for i in range(reps):
        call(i)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"n": n, "us_per_perm": round(e0.elapsed_time(e1) * 1e3 / reps, 2)}))
