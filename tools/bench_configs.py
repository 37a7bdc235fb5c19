#!/usr/bin/env python
"""Measurements of BASELINE.json's other configs (parity-test configs, not the
bench line): C1 dense ridge, C3 HIGGS-shaped dense SVM, C4 lasso primal
10M x 1M, C5 Criteo-shaped streamed logistic. One JSON line per config.

    python tools/bench_configs.py c3 [--lam 100] [--n 11000000]
    python tools/bench_configs.py c5 [--n 8000000] [--budget-gb 1.0]

Synthetic data is generated on the GPU (torch) except C5, whose data must
live in pinned host memory to be streamed. Epoch times are CUDA events on
the engine stream; gap checks run outside the timed epochs.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1803_06333_b200 as g  # noqa: E402
from paper_1803_06333_b200 import _lib as L  # noqa: E402
from paper_1803_06333_b200.data import DeviceMatrix  # noqa: E402

HBM = 6552.3


def ev():
    return torch.cuda.Event(enable_timing=True)


def timed_rounds(eng, rounds, gap_every=1, target=1e-3):
    """Run outer rounds; epoch time by CUDA events, gap checks untimed."""
    out = {"round_ms": [], "rel_gap": [], "objective": []}
    obj, gap = eng.objective_and_gap()
    out["rel_gap"].append(None if gap is None or obj == 0 else gap / abs(obj))
    out["objective"].append(obj)
    hit = None
    t_total = 0.0
    for r in range(1, rounds + 1):
        s = torch.cuda.current_stream()
        a, b = ev(), ev()
        a.record(s)
        eng.outer_round()
        b.record(s)
        torch.cuda.synchronize()
        eng.check_solves()
        ms = a.elapsed_time(b)
        t_total += ms
        out["round_ms"].append(ms)
        if r % gap_every == 0 or r == rounds:
            obj, gap = eng.objective_and_gap()
            rel = None if gap is None or obj == 0 else gap / abs(obj)
            out["rel_gap"].append(rel)
            out["objective"].append(obj)
            if hit is None and rel is not None and rel <= target:
                hit = {"epochs": r, "train_ms": t_total}
    out["to_target"] = hit
    return out


# ------------------------------------------------------------------ C3
def c3(args):
    n, d, lam = args.n, 28, args.lam
    gen = torch.Generator(device="cuda").manual_seed(3)
    X = torch.randn(n, d, device="cuda", dtype=torch.float64, generator=gen)
    X /= X.norm(dim=1, keepdim=True)
    w = torch.randn(d, device="cuda", dtype=torch.float64, generator=gen)
    y = torch.where(X @ w + 0.3 * torch.randn(n, device="cuda", dtype=torch.float64,
                                                  generator=gen) >= 0, 1.0, -1.0)
    cm = (X * y[:, None]).contiguous().reshape(-1)    # column i = y_i x_i, contiguous
    del X
    dm = DeviceMatrix(d, n, L.DENSE, cm)
    spec = g.ObjectiveSpec("dual_l2_svm", lam, n, d)
    res = {"config": "C3", "workload": f"dual hinge SVM, dense HIGGS-shaped {n}x{d}, lambda={lam}",
           "nnz": n * d}
    alg = 8 * n * d + 28 * n
    for mode in ("async", "sequential") if args.seq_rounds > 0 else ("async",):
        eng = g.Engine(dm, spec, g.HierarchyConfig(seed=0, epochs=1), mode=mode,
                       sync_solves=(mode == "sequential"), max_inflight=args.inflight)
        rounds = args.rounds if mode == "async" else args.seq_rounds
        r = timed_rounds(eng, rounds)
        ms = float(np.median(r["round_ms"]))
        res[mode] = {"epoch_ms_median": ms, "epochs_per_s": 1000.0 / ms,
                     "coord_updates_per_s": n * 1000.0 / ms,
                     "hbm_frac_of_round": alg / (ms * 1e-3) / 1e9 / HBM,
                     "rel_gap": r["rel_gap"], "to_1e-3": r["to_target"],
                     "round_ms": r["round_ms"]}
        del eng
        torch.cuda.empty_cache()
    res["algorithmic_bytes_per_epoch"] = alg
    print(json.dumps(res), flush=True)


# ------------------------------------------------------------------ C2
def c2_modes(args):
    """The bench workload (C2, dual logistic 1M x 100k, 40 nnz) in both modes:
    epochs to a 1e-3 relative duality gap for the deterministic sequential
    kernel (the parity-checked reference semantics) and the async TPA-SCD
    kernel, i.e. the north star's "same target within the same number of
    epochs +-10 %" at full size."""
    import bench
    indptr, rows, vals, _ = bench.gen_columns(0, bench.N_EX // bench.BLOCK)
    dm = DeviceMatrix.from_csc(bench.D_FEAT, indptr, rows, vals)
    spec = g.ObjectiveSpec("dual_l2_logistic", bench.LAM, bench.N_EX, bench.D_FEAT)
    res = {"config": "C2-modes", "workload": "bench.py C2 (dual L2 logistic 1M x 100k, 40 nnz)"}
    for mode, rounds in (("async", args.rounds), ("sequential", args.seq_rounds)):
        eng = g.Engine(dm, spec, g.HierarchyConfig(seed=0, epochs=1), mode=mode,
                       sync_solves=(mode == "sequential"))
        r = timed_rounds(eng, rounds)
        res[mode] = {"epoch_ms_median": float(np.median(r["round_ms"])), "rel_gap": r["rel_gap"],
                     "to_1e-3": r["to_target"]}
        del eng
    print(json.dumps(res), flush=True)


# -------------------------------------------------------- CPU baselines
def cpu_baselines(om, kind, lam, *, target=None, y=None, rounds_all=3, target_rel=1e-3,
                  max_epochs=60):
    """The oracle port (C restatement of the reference, oracle/) on the same
    arrays: all host cores (CoCoA over nproc host workers, the reference's
    multi-process mode) for a few rounds, and ONE core (K = 1, the reference's
    damped_solve with threads_per_device=1) run to the duality-gap target
    (BASELINE.md §3)."""
    import oracle
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    ra = oracle.train(om, kind, lam, target=target, y=y, nodes=cores, epochs=1, seed=0,
                      rounds=rounds_all, parallel=True, record_obj=False)
    per_all = float(np.mean(ra["round_s"]))
    t_all = time.perf_counter() - t0
    t0 = time.perf_counter()
    r1 = oracle.train(om, kind, lam, target=target, y=y, nodes=1, epochs=1, seed=0,
                      rounds=max_epochs, target_rel_gap=target_rel)
    t_one = time.perf_counter() - t0
    hit = r1["rounds"] if r1["gap"][-1] <= target_rel * abs(r1["objective"][-1]) else None
    return {"all_cores": {"cores": cores, "epochs_per_s": 1.0 / per_all, "rounds": rounds_all,
                          "wall_s": t_all, "kind": "port"},
            "one_core": {"cores": 1, "epochs_per_s": r1["rounds"] / max(sum(r1["round_s"]), 1e-9),
                         "time_to_target_s": t_one if hit else None, "epochs_to_target": hit,
                         "target": f"gap <= {target_rel} |F|", "kind": "port",
                         "includes_gap_checks": True}}


def engine_modes(dm, spec, args, alg_bytes, n_coords, seq_rounds=None):
    """Async (bench's configuration: one attempt per round, fused turn, L1-cached
    view gathers) and sequential engines: epoch ms, roofline fraction, rounds
    and device time to gap <= 1e-3 |F|."""
    out = {}
    for mode in ("async", "sequential"):
        rounds = args.rounds if mode == "async" else (seq_rounds or args.seq_rounds)
        kw = dict(sync_solves=False, retry_budget=0, cache_flags=1,
                  group_lanes=getattr(args, "lanes", 0)) if mode == "async" else {}
        eng = g.Engine(dm, spec, g.HierarchyConfig(seed=0, epochs=1), mode=mode, **kw)
        r = timed_rounds(eng, rounds)
        ms = float(np.median(r["round_ms"][1:] if len(r["round_ms"]) > 2 else r["round_ms"]))
        out[mode] = {"epoch_ms_median": ms, "epochs_per_s": 1000.0 / ms,
                     "coord_updates_per_s": n_coords * 1000.0 / ms,
                     "algorithmic_GBps": alg_bytes / (ms * 1e-3) / 1e9,
                     "hbm_frac_of_round": alg_bytes / (ms * 1e-3) / 1e9 / HBM,
                     "rel_gap": r["rel_gap"], "to_1e-3": r["to_target"]}
        eng.close()
        del eng
        torch.cuda.empty_cache()
    out["algorithmic_bytes_per_epoch"] = alg_bytes
    return out


# ------------------------------------------------------------ C2 primal
def c2p(args):
    """BASELINE configs[1] literally: L2 logistic regression in the PRIMAL
    (restated kind logistic_primal): coordinates = the 100k features (about
    400 nnz per column, the long-column path), v = A w over the 1M examples
    (8 MB), the same synthetic examples as bench.py (labels unfolded)."""
    import bench
    import oracle
    indptr, rows, vals, y = bench.gen_columns(0, bench.N_EX // bench.BLOCK)
    raw = vals * np.repeat(y, bench.NNZ)             # undo bench's label fold
    ex = DeviceMatrix.from_csc(bench.D_FEAT, indptr, rows, raw)
    dm = ex.transpose()                               # columns = features
    del ex
    spec = g.ObjectiveSpec("logistic_primal", bench.LAM, bench.N_EX, bench.D_FEAT, target=y)
    nnz = bench.N_EX * bench.NNZ
    res = {"config": "C2-primal", "workload": "L2 logistic regression, PRIMAL SCD "
           "(logistic_primal), synthetic sparse 1M examples x 100k features, 40 nnz/example "
           "(~400 per feature column), lambda=1", "nnz": nnz}
    res.update(engine_modes(dm, spec, args, 12 * nnz + 36 * bench.D_FEAT, bench.D_FEAT))
    if not args.no_cpu:
        h = dm.to_host()
        om = oracle.OMatrix(h.n_rows, h.indptr, h.rows, h.vals)
        res["cpu_baseline"] = cpu_baselines(om, "logistic_primal", bench.LAM, target=y)
    print(json.dumps(res), flush=True)


# --------------------------------------------------------------- C1 dual
def c1d(args):
    """BASELINE configs[0] literally: ridge regression in the DUAL (restated
    kind dual_ridge): coordinates = the 20k examples (dense columns of 500),
    v = X^T alpha (500 doubles)."""
    import oracle
    n_ex, n_feat = 20_000, 500
    gen = torch.Generator(device="cuda").manual_seed(1)
    X = torch.randn(n_ex, n_feat, device="cuda", dtype=torch.float64, generator=gen) / \
        np.sqrt(n_feat)
    wt = torch.randn(n_feat, device="cuda", dtype=torch.float64, generator=gen)
    b = X @ wt + 0.1 * torch.randn(n_ex, device="cuda", dtype=torch.float64, generator=gen)
    dm = DeviceMatrix(n_feat, n_ex, L.DENSE, X.contiguous().reshape(-1))   # column = example
    yb = b.cpu().numpy()
    spec = g.ObjectiveSpec("dual_ridge", 1.0, n_ex, n_feat, target=yb)
    nnz = n_ex * n_feat
    res = {"config": "C1-dual", "workload": "ridge regression, DUAL SCD (dual_ridge), dense "
           "20k x 500, lambda=1", "nnz": nnz}
    res.update(engine_modes(dm, spec, args, 8 * nnz + 28 * n_ex, n_ex, seq_rounds=args.rounds))
    if not args.no_cpu:
        Xh = X.cpu().numpy()
        indptr = np.arange(0, nnz + 1, n_feat, dtype=np.int64)
        rws = np.tile(np.arange(n_feat, dtype=np.int32), n_ex)
        om = oracle.OMatrix(n_feat, indptr, rws, Xh.reshape(-1))
        res["cpu_baseline"] = cpu_baselines(om, "dual_ridge", 1.0, y=yb)
    print(json.dumps(res), flush=True)


def c2cpu(args):
    """The bench workload's CPU baselines: the oracle port on
    all host cores and on one core run to the 1e-3 duality-gap target."""
    import bench
    import oracle
    indptr, rows, vals, _ = bench.gen_columns(0, bench.N_EX // bench.BLOCK)
    om = oracle.OMatrix(bench.D_FEAT, indptr, rows, vals)
    res = {"config": "C2-cpu", "workload": "bench.py C2 (dual L2 logistic 1M x 100k, 40 nnz)",
           "cpu_baseline": cpu_baselines(om, "dual_l2_logistic", bench.LAM)}
    print(json.dumps(res), flush=True)


# ------------------------------------------------------------------ C1
def c1(args):
    """ridge_primal, dense 20k examples x 500 features (coordinates = features)."""
    n_ex, n_feat = 20_000, 500
    gen = torch.Generator(device="cuda").manual_seed(1)
    X = torch.randn(n_ex, n_feat, device="cuda", dtype=torch.float64, generator=gen) / \
        np.sqrt(n_feat)
    wt = torch.randn(n_feat, device="cuda", dtype=torch.float64, generator=gen)
    b = X @ wt + 0.1 * torch.randn(n_ex, device="cuda", dtype=torch.float64, generator=gen)
    dm = DeviceMatrix(n_ex, n_feat, L.DENSE, X.t().contiguous().reshape(-1))
    spec = g.ObjectiveSpec("ridge_primal", 1.0, n_ex, n_feat, target=b.cpu().numpy())
    res = {"config": "C1", "workload": "ridge (primal), dense 20k x 500, lambda=1",
           "nnz": n_ex * n_feat}
    for mode in ("sequential", "async"):
        eng = g.Engine(dm, spec, g.HierarchyConfig(seed=0, epochs=1), mode=mode)
        r = timed_rounds(eng, args.rounds)
        ms = float(np.median(r["round_ms"]))
        res[mode] = {"epoch_ms_median": ms, "epochs_per_s": 1000.0 / ms,
                     "rel_gap": r["rel_gap"], "to_1e-3": r["to_target"]}
    print(json.dumps(res), flush=True)


# ------------------------------------------------------------------ C4
def c4(args):
    """lasso_primal, sparse 10M examples x 1M features, ~40 nnz per example
    (400 per feature column), coordinates = features; one GPU holds the lot
    (4.8 GB) — the 8-GPU run column-partitions it."""
    n_ex, n_feat, per_col = args.n_ex, args.n_feat, args.per_col
    gen = torch.Generator(device="cuda").manual_seed(4)
    rows = torch.empty(n_feat, per_col, dtype=torch.int32, device="cuda")
    step = 1_000_000 // max(1, per_col // 40)
    for lo in range(0, n_feat, step):        # distinct sorted rows per column
        hi = min(n_feat, lo + step)
        r = torch.randint(0, n_ex - per_col + 1, (hi - lo, per_col), device="cuda",
                          generator=gen, dtype=torch.int64)
        r, _ = torch.sort(r, dim=1)
        rows[lo:hi] = (r + torch.arange(per_col, device="cuda")).to(torch.int32)
    vals = torch.randn(n_feat * per_col, device="cuda", dtype=torch.float64, generator=gen)
    indptr = torch.arange(0, n_feat * per_col + 1, per_col, device="cuda", dtype=torch.int64)
    dm = DeviceMatrix(n_ex, n_feat, L.CSC, vals, indptr, rows.reshape(-1),
                      nnz=n_feat * per_col)
    coef = torch.randn(n_feat, device="cuda", dtype=torch.float64, generator=gen)
    coef[torch.rand(n_feat, device="cuda", generator=gen, dtype=torch.float64) < 0.5] = 0.0
    b = dm.matvec(coef) + 0.1 * torch.randn(n_ex, device="cuda", dtype=torch.float64,
                                             generator=gen)
    lam = args.lam
    spec = g.ObjectiveSpec("lasso_primal", lam, n_ex, n_feat, target=b.cpu().numpy())
    nnz = n_feat * per_col
    alg = 12 * nnz + 36 * n_feat
    res = {"config": "C4", "workload": f"lasso (primal), sparse {n_ex}x{n_feat}, "
                                       f"{per_col} nnz/feature, lambda={lam}", "nnz": nnz}
    eng = g.Engine(dm, spec, g.HierarchyConfig(seed=0, epochs=1), mode="async",
                   sync_solves=False, cache_flags=args.cache_flags, group_lanes=args.lanes)
    res["cache_flags"] = args.cache_flags
    res["lanes"] = args.lanes
    ms_all = []
    objs = []
    for r in range(args.rounds):
        s = torch.cuda.current_stream()
        a, bb = ev(), ev()
        a.record(s)
        eng.outer_round()
        bb.record(s)
        torch.cuda.synchronize()
        eng.check_solves()
        ms_all.append(a.elapsed_time(bb))
        objs.append(eng.objective_and_gap()[0])
    ms = float(np.median(ms_all))
    res["async"] = {"epoch_ms_median": ms, "epochs_per_s": 1000.0 / ms,
                    "coord_updates_per_s": n_feat * 1000.0 / ms,
                    "algorithmic_GBps": alg / (ms * 1e-3) / 1e9,
                    "hbm_frac_of_round": alg / (ms * 1e-3) / 1e9 / HBM,
                    "objective": objs, "round_ms": ms_all}
    print(json.dumps(res), flush=True)


# ------------------------------------------------------------------ C5
def criteo_block(rng, n, d, w):
    """13 log-normal 'integer' features + 26 categorical fields hashed into
    disjoint ranges of [13, d) with Zipf popularity; per-example L2
    normalisation; planted logistic labels; label-folded."""
    n_cat, n_int = 26, 13
    width = (d - n_int) // n_cat
    ints = np.log1p(rng.lognormal(1.0, 1.5, size=(n, n_int)))
    cats = (rng.zipf(1.3, size=(n, n_cat)) - 1) % width + n_int + np.arange(n_cat) * width
    rows = np.concatenate([np.broadcast_to(np.arange(n_int), (n, n_int)), cats], axis=1)
    vals = np.concatenate([ints, np.ones((n, n_cat))], axis=1)
    vals /= np.linalg.norm(vals, axis=1, keepdims=True)
    z = np.einsum("ij,ij->i", vals, w[rows])
    y = np.where(rng.random(n) < 0.5 * (1 + np.tanh(0.5 * z)), 1.0, -1.0)
    vals *= y[:, None]
    return rows.astype(np.int32), vals


def c5(args):
    from paper_1803_06333_b200 import pipeline as P
    n, d, k = args.n, 1 << 20, 39
    nnz = n * k
    t0 = time.perf_counter()
    indptr = torch.arange(0, nnz + 1, k, dtype=torch.int64).pin_memory().numpy()
    rows = torch.empty(nnz, dtype=torch.int32).pin_memory().numpy()
    vals = torch.empty(nnz, dtype=torch.float64).pin_memory().numpy()
    w = np.random.default_rng(55).standard_normal(d)
    B = 1_000_000
    for lo in range(0, n, B):
        hi = min(n, lo + B)
        r, v = criteo_block(np.random.default_rng([55, lo // B]), hi - lo, d, w)
        rows[lo * k:hi * k] = r.reshape(-1)
        vals[lo * k:hi * k] = v.reshape(-1)
    t_gen = time.perf_counter() - t0
    m = g.SparseColumnMatrix(d, indptr, rows, vals, validate=False)
    budget = int(args.budget_gb * 2 ** 30)
    part = P.StreamingPartition(m, chunk_size=args.chunk, device_budget=budget)
    spec = g.ObjectiveSpec("dual_l2_logistic", args.lam, n, d)
    lam = args.lam
    base = np.full(n, 0.5)
    # v0 = A alpha0 via the chunk data on the device is not needed for the
    # timing: a zero-lin subproblem exercises the identical data path
    lin = torch.zeros(d, dtype=torch.float64, device="cuda")
    bytes_per_epoch = 8 * (n + 1) + 12 * nnz
    res = {"config": "C5", "workload": f"dual L2 logistic, Criteo-shaped synthetic: {n} examples "
                                       f"x 2^20 hashed features, 39 nnz/example (13 log-normal + "
                                       f"26 Zipf categorical), lambda={lam}",
           "nnz": nnz, "host_bytes": bytes_per_epoch, "device_budget_bytes": budget,
           "chunks": part.n_chunks, "resident_chunks": part.n_resident,
           "streamed_bytes_per_epoch": int(bytes_per_epoch * (part.n_chunks - part.n_resident)
                                           / part.n_chunks),
           "direct_dma": part.direct_dma, "gen_s": t_gen}
    for mode in (L.MODE_ASYNC,):
        times = []
        h2d = []
        train = []
        for e in range(args.epochs):
            st, delta, values, info, scal, dmp = part.solve(
                spec, lin, 1.0 / lam, 0.0, base, seed=1, epoch_index=e, epochs=1, mode=mode,
                timing=True)
            assert st == 0, st
            times.append(float(scal[2]))
            rows_s = part.last_schedule
            h2d.append(float(rows_s[:, 3].sum()))
            train.append(float(rows_s[:, 4].sum()))
        ms = float(np.median(times[1:])) if len(times) > 1 else times[0]
        streamed = res["streamed_bytes_per_epoch"]
        res["async"] = {"epoch_ms_median": ms, "epochs_per_s": 1000.0 / ms,
                        "examples_per_s": n * 1000.0 / ms,
                        "h2d_ms_per_epoch": float(np.median(h2d)),
                        "train_ms_per_epoch": float(np.median(train)),
                        "h2d_GBps": streamed / (float(np.median(h2d)) * 1e-3) / 1e9
                        if np.median(h2d) > 0 else None,
                        "end_to_end_stream_GBps": streamed / (ms * 1e-3) / 1e9,
                        "epoch_ms": times}
    part.close()
    print(json.dumps(res), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=("c1", "c1d", "c2", "c2p", "c2cpu", "c3", "c4", "c5"))
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cache-flags", type=int, default=0,
                    help="C4: glm_solve_args.flags cache bits (1 view via L1, 2 stream evict-first / "
                         "view evict-last, 3 both)")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--lam", type=float, default=None)
    ap.add_argument("--rounds", type=int, default=10)
    ap.add_argument("--seq-rounds", type=int, default=2)
    ap.add_argument("--epochs", type=int, default=4)
    ap.add_argument("--budget-gb", type=float, default=1.0)
    ap.add_argument("--chunk", type=int, default=1_000_000)
    ap.add_argument("--n-ex", type=int, default=10_000_000)
    ap.add_argument("--n-feat", type=int, default=1_000_000)
    ap.add_argument("--per-col", type=int, default=400)
    ap.add_argument("--inflight", type=int, default=0, help="async in-flight budget (0 = auto)")
    ap.add_argument("--lanes", type=int, default=0,
                    help="async lanes per coordinate: G | (R << 8) (0 = auto)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    if args.config == "c3":
        args.n = args.n or 11_000_000
        args.lam = args.lam or 100.0
        c3(args)
    elif args.config == "c1":
        c1(args)
    elif args.config == "c1d":
        c1d(args)
    elif args.config == "c2p":
        c2p(args)
    elif args.config == "c2cpu":
        c2cpu(args)
    elif args.config == "c2":
        c2_modes(args)
    elif args.config == "c4":
        args.lam = args.lam or 50.0
        c4(args)
    else:
        args.n = args.n or 8_000_000
        args.lam = args.lam or 1.0
        c5(args)


if __name__ == "__main__":
    main()
