#!/usr/bin/env python
"""Multi-GPU runs of BASELINE configs C3 (dense SVM, examples partitioned) and
C4 (lasso primal, features column-partitioned), one process per GPU:

    python -m torch.distributed.run --nproc-per-node N tools/bench_multi.py c3|c4

Each rank generates only its own partition on its GPU (the same data for any N:
blocks are seeded by their global index), builds the engine with the NVLink
peer exchange, and times async rounds with CUDA events (max over ranks).
Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import time
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import paper_1803_06333_b200 as g  # noqa: E402
from paper_1803_06333_b200 import _lib as L  # noqa: E402
from paper_1803_06333_b200.comm import NcclReducer  # noqa: E402
from paper_1803_06333_b200.data import DeviceMatrix  # noqa: E402

HBM = 6552.3


def max_all(x):
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    if dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def timed(eng, rounds, gap=True):
    ms, rel = [], []
    obj, gp = eng.objective_and_gap()
    rel.append(None if gp is None or obj == 0 else gp / abs(obj))
    for _ in range(rounds):
        if dist.is_initialized():
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.outer_round()
        b.record()
        torch.cuda.synchronize()
        ms.append(max_all(a.elapsed_time(b)))
        eng.check_solves()
        if gap:
            obj, gp = eng.objective_and_gap()
            rel.append(None if gp is None or obj == 0 else gp / abs(obj))
        else:
            rel.append(eng.objective_and_gap()[0])
    return ms, rel


def c3(args, rank, world):
    n, d, lam = args.n, 28, args.lam
    blocks = 8
    per = n // blocks
    lo_b, hi_b = rank * blocks // world, (rank + 1) * blocks // world
    gw = torch.Generator(device="cuda").manual_seed(33)
    w = torch.randn(d, device="cuda", dtype=torch.float64, generator=gw)
    parts = []
    for b in range(lo_b, hi_b):
        gen = torch.Generator(device="cuda").manual_seed(1000 + b)
        X = torch.randn(per, d, device="cuda", dtype=torch.float64, generator=gen)
        X /= X.norm(dim=1, keepdim=True)
        y = torch.where(X @ w + 0.3 * torch.randn(per, device="cuda", dtype=torch.float64,
                                                      generator=gen) >= 0, 1.0, -1.0)
        parts.append((X * y[:, None]).reshape(-1))
    cm = torch.cat(parts).contiguous()
    m_loc = (hi_b - lo_b) * per
    dm = DeviceMatrix(d, m_loc, L.DENSE, cm)
    n_tot = per * blocks
    spec = g.ObjectiveSpec("dual_l2_svm", lam, n_tot, d)
    cfg = g.HierarchyConfig(nodes=world, seed=0, epochs=1)
    kw = dict(reducer=NcclReducer(), node_index=rank, n_total=n_tot) if world > 1 else {}
    eng = g.Engine(dm, spec, cfg, mode="async", sync_solves=False, retry_budget=0, **kw)
    for _ in range(2):
        eng.outer_round()
    eng.reset()
    ms, rel = timed(eng, args.rounds)
    alg = 8 * n_tot * d + 28 * n_tot
    med = float(np.median(ms[1:]))
    return {"config": "C3", "n_gpus": world,
            "workload": f"dual hinge SVM, dense HIGGS-shaped {n_tot}x{d}, lambda={lam}, "
                        f"examples partitioned over {world} GPU(s)",
            "epoch_ms_median": med, "epochs_per_s": 1000.0 / med,
            "coord_updates_per_s": n_tot * 1000.0 / med,
            "hbm_frac_per_gpu": alg / world / (med * 1e-3) / 1e9 / HBM,
            "rel_gap": rel, "round_ms": ms, "exchange": "nvlink-peer" if eng.exchange else "nccl"}


def c4(args, rank, world):
    n_ex, n_feat, per_col, lam = args.n_ex, args.n_feat, args.per_col, args.lam
    blocks = 8
    fb = n_feat // blocks
    lo_b, hi_b = rank * blocks // world, (rank + 1) * blocks // world
    rows_l, vals_l, coef_l = [], [], []
    for b in range(lo_b, hi_b):
        gen = torch.Generator(device="cuda").manual_seed(4000 + b)
        r = torch.randint(0, n_ex - per_col + 1, (fb, per_col), device="cuda", generator=gen,
                          dtype=torch.int64)
        r, _ = torch.sort(r, dim=1)
        rows_l.append((r + torch.arange(per_col, device="cuda")).to(torch.int32).reshape(-1))
        vals_l.append(torch.randn(fb * per_col, device="cuda", dtype=torch.float64,
                                  generator=gen))
        c = torch.randn(fb, device="cuda", dtype=torch.float64, generator=gen)
        c[torch.rand(fb, device="cuda", generator=gen, dtype=torch.float64) < 0.5] = 0.0
        coef_l.append(c)
    m_loc = (hi_b - lo_b) * fb
    rows, vals = torch.cat(rows_l), torch.cat(vals_l)
    indptr = torch.arange(0, m_loc * per_col + 1, per_col, device="cuda", dtype=torch.int64)
    dm = DeviceMatrix(n_ex, m_loc, L.CSC, vals, indptr, rows, nnz=m_loc * per_col)
    b = dm.matvec(torch.cat(coef_l)).clone()          # this partition's share of X coef
    if world > 1:
        dist.all_reduce(b)
    gen = torch.Generator(device="cuda").manual_seed(4999)
    b += 0.1 * torch.randn(n_ex, device="cuda", dtype=torch.float64, generator=gen)
    n_tot = fb * blocks
    spec = g.ObjectiveSpec("lasso_primal", lam, n_ex, n_tot, target=b.cpu().numpy())
    cfg = g.HierarchyConfig(nodes=world, seed=0, epochs=1)
    kw = dict(reducer=NcclReducer(), node_index=rank, n_total=n_tot) if world > 1 else {}
    eng = g.Engine(dm, spec, cfg, mode="async", sync_solves=False, retry_budget=0,
                   cache_flags=3, **kw)    # C4: stream evict-first, view evict-last + L1
    for _ in range(2):
        eng.outer_round()
    eng.reset()
    ms, objs = timed(eng, args.rounds, gap=False)
    breakdown = None
    if args.breakdown:      # per-kernel events of extra rounds + the turn's phase stamps
        wk = next(iter(eng.workers.values()))
        st = torch.zeros(8, dtype=torch.int64, device="cuda")
        if eng.exchange is not None:
            L.check(L.lib().glm_peer_stamps(eng.exchange.handle, st.data_ptr()), "stamps")
        wk.solver.timing_read()
        wk.solver.timing_glue()
        wk.solver.timing(True)
        for _ in range(3):
            eng.outer_round()
        torch.cuda.synchronize()
        k_ms, k_n = wk.solver.timing_read()
        gl_ms, gl_n = wk.solver.timing_glue()
        wk.solver.timing(False)
        s_ = st.cpu().numpy().astype(np.int64)
        breakdown = {"perm_ms": k_ms[0] / max(k_n, 1), "epoch_ms": k_ms[1] / max(k_n, 1),
                     "turn_ms": gl_ms[2] / max(gl_n[2], 1),
                     "turn_phases_us": (np.diff(s_[:5]) / 1e3).round(2).tolist()
                     if eng.exchange is not None else None}
        if eng.exchange is not None:
            L.lib().glm_peer_stamps(eng.exchange.handle, None)
    nnz = n_tot * per_col
    alg = 12 * nnz + 36 * n_tot
    med = float(np.median(ms[1:]))
    return {"config": "C4", "n_gpus": world,
            "workload": f"lasso (primal), sparse {n_ex}x{n_tot}, {per_col} nnz/feature, "
                        f"lambda={lam}, features partitioned over {world} GPU(s)",
            "epoch_ms_median": med, "epochs_per_s": 1000.0 / med,
            "coord_updates_per_s": n_tot * 1000.0 / med,
            "hbm_frac_per_gpu": alg / world / (med * 1e-3) / 1e9 / HBM,
            "objective": objs, "round_ms": ms,
            "exchange": "nvlink-peer" if eng.exchange else "nccl",
            "exchange_bytes_per_rank_per_round": 8 * n_ex, "breakdown": breakdown}


def c5(args, rank, world):
    """Every rank streams its own Criteo-shaped partition (pinned host memory ->
    two device slots, csrc/stream.cu) and the ranks run CoCoA rounds with the
    Delta v all-reduce (NCCL): the out-of-core configuration at N GPUs."""
    from bench_configs import criteo_block
    from paper_1803_06333_b200 import pipeline as P
    n_per, d, k, lam = args.n_per, 1 << 20, 39, args.lam
    nnz = n_per * k
    indptr = torch.arange(0, nnz + 1, k, dtype=torch.int64).pin_memory().numpy()
    rows = torch.empty(nnz, dtype=torch.int32).pin_memory().numpy()
    vals = torch.empty(nnz, dtype=torch.float64).pin_memory().numpy()
    w = np.random.default_rng(55).standard_normal(d)
    B = 1_000_000
    for lo in range(0, n_per, B):
        hi = min(n_per, lo + B)
        blk = (rank * n_per + lo) // B                     # global block id: same data for any N
        r, v = criteo_block(np.random.default_rng([55, blk]), hi - lo, d, w)
        rows[lo * k:hi * k] = r.reshape(-1)
        vals[lo * k:hi * k] = v.reshape(-1)
    m = g.SparseColumnMatrix(d, indptr, rows, vals, validate=False)
    part = P.StreamingPartition(m, chunk_size=args.chunk,
                                device_budget=int(args.budget_gb * 2 ** 30))
    spec = g.ObjectiveSpec("dual_l2_logistic", lam, n_per * world, d)
    alpha = torch.full((n_per,), 0.5, dtype=torch.float64, device="cuda")
    v = torch.zeros(d, dtype=torch.float64, device="cuda")
    dv = torch.empty(d, dtype=torch.float64, device="cuda")
    delta = torch.empty(n_per, dtype=torch.float64, device="cuda")
    def one_round(rnd):
        lin = v / lam
        st, _, values, info, scal, dmp = part.solve(
            spec, lin, world / lam, 0.0, alpha, seed=1, epoch_index=rnd, epochs=1,
            mode=L.MODE_ASYNC, delta=delta, dv_out=dv)
        assert st == 0, st
        if world > 1:
            dist.all_reduce(dv)
        v.add_(dv)
        alpha.add_(delta)

    one_round(0)                                      # warm
    # The loader streams the next solve's first chunks while the caller folds
    # and exchanges, so per-round events would miss that part of the copy
    # traffic: time the whole loop of rounds on the host clock, synchronised
    # on both sides, max over ranks.
    if dist.is_initialized():
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for rnd in range(1, args.rounds + 1):
        one_round(rnd)
    torch.cuda.synchronize()
    total_ms = max_all((time.perf_counter() - t0) * 1e3)
    ms = [total_ms / args.rounds] * (args.rounds + 1)
    # the pinned host -> device copy peak of this box (1 GiB, best of 5)
    hbuf = torch.empty(1 << 27, dtype=torch.float64).pin_memory()
    dbuf = torch.empty(1 << 27, dtype=torch.float64, device="cuda")
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dbuf.copy_(hbuf, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    h2d_peak = (8 << 27) / (best * 1e-3) / 1e9
    del hbuf, dbuf
    med = float(np.median(ms[1:]))
    streamed = (8 * (n_per + 1) + 12 * nnz) * (part.n_chunks - part.n_resident) / part.n_chunks
    part.close()
    return {"config": "C5", "n_gpus": world,
            "workload": f"dual L2 logistic, Criteo-shaped {n_per * world} examples "
                        f"({n_per} per GPU) x 2^20 hashed features, 39 nnz, streamed "
                        f"(device budget {args.budget_gb} GB per GPU), lambda={lam}",
            "round_ms_median": med, "epochs_per_s": 1000.0 / med,
            "examples_per_s": n_per * world * 1000.0 / med,
            "stream_GBps_per_gpu": streamed / (med * 1e-3) / 1e9,
            "pinned_h2d_peak_GBps": h2d_peak,
            "stream_frac_of_h2d_peak": streamed / (med * 1e-3) / 1e9 / h2d_peak,
            "timer": "host clock around all rounds (loads between rounds included), "
                     "max over ranks",
            "round_ms": ms}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=("c3", "c4", "c5"))
    ap.add_argument("--n-per", type=int, default=8_000_000)
    ap.add_argument("--chunk", type=int, default=1_000_000)
    ap.add_argument("--budget-gb", type=float, default=1.0)
    ap.add_argument("--rounds", type=int, default=10)
    ap.add_argument("--n", type=int, default=11_000_000)
    ap.add_argument("--lam", type=float, default=None)
    ap.add_argument("--n-ex", type=int, default=10_000_000)
    ap.add_argument("--n-feat", type=int, default=1_000_000)
    ap.add_argument("--per-col", type=int, default=400)
    ap.add_argument("--out", default=None, help="append the JSON line to this file")
    ap.add_argument("--breakdown", action="store_true",
                    help="C4: per-kernel times and the turn's phase stamps of 3 extra rounds")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    print(f"[multi r{rank}] start {args.config} world {world}", file=sys.stderr, flush=True)
    if args.config == "c3":
        args.lam = args.lam or 100.0
        res = c3(args, rank, world)
    elif args.config == "c4":
        args.lam = args.lam or 50.0
        res = c4(args, rank, world)
    else:
        args.lam = args.lam or 1.0
        res = c5(args, rank, world)
    if rank == 0:
        line = json.dumps(res)
        print(line, flush=True)
        if args.out:
            with open(args.out, "a") as fh:
                fh.write(line + "\n")
    sys.stdout.flush()
    from paper_1803_06333_b200.comm import shutdown
    shutdown()


if __name__ == "__main__":
    main()
