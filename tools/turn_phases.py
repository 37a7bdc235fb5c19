"""Phase timestamps of glm_round_turn on the C2 workload (debug); world >= 1
under torchrun; 3-round CUDA graphs replayed like bench.py, stamps of the
last round's turn. Prints, per rank, the median µs of: P1 decide | turn
counter bumped | publish -> every flag seen | P3 round start | publish: system
fence done | flag stores issued | last block starts its P1 fold (the last
three relative to the turn start)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import torch.distributed as dist
import bench
import paper_1803_06333_b200 as g
from paper_1803_06333_b200 import _lib as L
from paper_1803_06333_b200.comm import NcclReducer
from paper_1803_06333_b200.data import DeviceMatrix
world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
# SHARE=k (one process): the 1/k share of the examples one rank owns at k GPUs
per = (bench.N_EX // bench.BLOCK) // (world if world > 1 else int(os.environ.get("SHARE", "1")))
indptr, rows, vals, y = bench.gen_columns(rank * per, (rank + 1) * per)
dm = DeviceMatrix.from_csc(bench.D_FEAT, indptr, rows, vals)
spec = g.ObjectiveSpec("dual_l2_logistic", 1.0, bench.N_EX, bench.D_FEAT)
kw = dict(reducer=NcclReducer(), node_index=rank, n_total=bench.N_EX) if world > 1 else {}
eng = g.Engine(dm, spec, g.HierarchyConfig(nodes=world, t1=10**6, seed=0, epochs=1),
               mode="async", sync_solves=False, retry_budget=0, cache_flags=1, **kw)
st = torch.zeros(8, dtype=torch.int64, device="cuda")
L.check(L.lib().glm_peer_stamps(eng.exchange.handle, st.data_ptr()), "stamps")
for _ in range(5):
    eng.outer_round()
torch.cuda.synchronize()
eng.reset()
graph = eng.capture(3)           # graph replay like bench.py: no host pacing between rounds
ph = []
raw = []
for _ in range(40):
    eng.reset()
    graph.replay()
    torch.cuda.synchronize()
    s = st.cpu().numpy().astype(np.int64)
    raw.append(s.copy())
    ph.append(np.concatenate([np.diff(s[:5]), [s[5] - s[0], s[6] - s[0], s[7] - s[0]]]) / 1e3)
med = torch.tensor(np.median(ph, axis=0), device="cuda")
out = [torch.zeros_like(med) for _ in range(world)]
if world > 1:
    dist.all_gather(out, med)
else:
    out = [med]
if rank == 0:
    for r, o in enumerate(out):
        print(f"rank {r}:", np.round(o.cpu().numpy(), 2), flush=True)
# %globaltimer is not synchronised across GPUs, so the skew is read from the
# local waits (publish -> every flag seen): per replay the last rank to publish
# waits only for the flag latency, the others also for that rank.
if world > 1:
    wt = torch.tensor([(x[3] - x[2]) / 1e3 for x in raw], dtype=torch.float64, device="cuda")
    allw = [torch.zeros_like(wt) for _ in range(world)]
    dist.all_gather(allw, wt)
    if rank == 0:
        W = np.stack([x.cpu().numpy() for x in allw])        # [rank, replay]
        print("wait per replay (us): median of min over ranks (flag latency):",
              round(float(np.median(W.min(0))), 2), "| median of max over ranks:",
              round(float(np.median(W.max(0))), 2))
sys.stdout.flush()
from paper_1803_06333_b200.comm import shutdown  # noqa: E402
shutdown()
