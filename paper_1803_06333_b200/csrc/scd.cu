// scd.cu — the TPA-SCD local solver on B200 (sm_100a).
//
// Replaces damped_solve / scd_epoch / run_pass / coordinate_update
// (solver.py:152-305).  One subtask = begin -> G(0) -> attempts -> finalize,
// where each attempt is
//     permutation (prng.cu)  ->  snapshot view  ->  epoch kernel  ->  value+decide
// and the damping control flow of damped_solve (restore / plateau / halve /
// divergence, solver.py:272-298) runs in the last block of the value kernel
// against a device-resident SolveState.  Attempts therefore queue on the
// stream with no host round-trip; once the state says `done` every later
// kernel of the subtask exits at its first instruction.
//
// Epoch kernels:
//  * scd_seq   — GLM_MODE_SEQUENTIAL, the deterministic fixed-permutation
//                mode: one CTA walks the permutation exactly like
//                run_pass(n_threads=1); the view lives in shared memory when
//                it fits (d <= 24k), otherwise in global memory.
//  * scd_async — GLM_MODE_ASYNC (TPA-SCD): a group of G lanes owns one
//                coordinate j = perm[k]; coalesced loads of the column, a
//                gather of the shared view through L2 (ld.global.cg),
//                shuffle reduction, the closed-form / Newton step on lane 0,
//                and red.global.add.f64 scatter of quad*step*a_j into the view.
//                Concurrent groups read stale views by design (solver.py:8-13,
//                SPEC.md:261-262); the damping check discards bad epochs.
//  * scd_seq_narrow / scd_replica — dense columns with d <= 256 (C3): the
//                view in registers (sequential) or a CTA snapshot plus
//                per-warp pending updates published per phase (async).
//
// Solve variants: chunked solves (stream.cu) guard every kernel with the open
// chunk's sequence number; GLM_FLAG_TURN solves leave the value check and
// the finalize to glm_round_turn (peer.cu), which fuses them with the Delta v
// exchange and the next round's start; GLM_FLAG_PREFETCH_PERM generates the
// next solve's permutation on a low-priority side stream (early — while this
// epoch runs — when every solve has exactly one attempt).
//
// Memory: delta is double-buffered (every coordinate is visited exactly once
// per epoch, so the epoch reads delta[dc] and writes delta[dc^1] — accept is a
// buffer flip, reject costs nothing); the view is snapshotted per attempt
// (d doubles) and a reject flips the working/snapshot roles.
// Delta v = B delta is recovered as (view - lin)/quad instead of a second
// SpMV (the reference recomputes it exactly, solver.py:300); the parity tests
// bound the difference (tests/test_gpu_solver.py).

#include <atomic>
#include <cstdio>

#include "solver.cuh"

namespace glm {

constexpr int EPOCH_PARTIALS = 16 * NUM_SMS;    // >= any epoch grid
constexpr int VALUE_MAX_BLOCKS = 8 * NUM_SMS;

struct EpochParams {
    SolveState *st;
    int kind;
    double lam, rho, quad;
    int64_t m, d;
    const int64_t *indptr;
    const int32_t *rows;
    const double *vals;
    const double *sq;
    const longlong2 *meta;  // packed {start | count << 40, |a_j|^2} (CM bit 2) or NULL
    const double *base;
    const double *y;
    double *delta0, *delta1;
    double *view0, *view1;
    const int32_t *perm;
    double *gpart;          // per-block partial sum_j g(base_j + delta_j) of the epoch
    int64_t nnz;
    int64_t seq;            // chunked mode: run only while chunk `seq` is open (-1: always)
    int pdl;                // async: launched as a programmatic dependent (turn rounds)
};

// A kernel of chunk `seq` runs only while that chunk is open and unfinished;
// seq < 0 (in-memory solves) only tests `done`.
__device__ __forceinline__ bool skip_attempt(const SolveState *st, int64_t seq) {
    return st->done || (seq >= 0 && st->seq != seq);
}

__device__ __forceinline__ void flag_error(SolveState *st) {
    atomicCAS(&st->status, GLM_OK, GLM_SOLVER_ERROR);
}

// delta buffers: dc == -1 means "delta is identically zero" (no buffer read);
// an epoch reads buffer dc and writes buffer (dc == 0 ? 1 : 0).
__device__ __forceinline__ const double *delta_cur(const EpochParams &p, int dc) {
    return dc < 0 ? nullptr : (dc ? p.delta1 : p.delta0);
}
__device__ __forceinline__ double *delta_next(const EpochParams &p, int dc) {
    return dc == 0 ? p.delta1 : p.delta0;
}

// Writes the block's partial g-sum (warp shuffles + smem, fixed order).
__device__ __forceinline__ void store_block_gsum(double g, double *gpart, SolveState *st) {
    __shared__ double s_g[32];
    g = warp_sum(g);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s_g[warp] = g;
    __syncthreads();
    if (threadIdx.x < 32) {
        double x = threadIdx.x < (blockDim.x >> 5) ? s_g[threadIdx.x] : 0.0;
        x = warp_sum(x);
        if (threadIdx.x == 0) {
            gpart[blockIdx.x] = x;
            if (blockIdx.x == 0) st->epoch_blocks = gridDim.x;
        }
    }
}

// --------------------------------------------------------------- async
// TPA-SCD: a group of G lanes owns coordinate j = perm[k].  The column is
// loaded once into registers (R elements per lane; longer columns stream the
// tail), gathered against the shared view through L2, reduced with shuffles,
// stepped on the group leader, and scattered with red.global.add.f64.
// Packed coordinate record (glm_solver_prepare): start | count << 40 and the
// bits of |a_j|^2; a count that does not fit 24 bits is the sentinel 2^24-1
// (the kernel then reads indptr).
constexpr int64_t META_CNT_SENTINEL = (1LL << 24) - 1;

// GLM_EPOCH_EARLY_TRIGGER=0|1 (experiments) overrides glm_solver::early_trigger
static int epoch_early_trigger(const glm_solver *s) {
    static const int v = [] {
        const char *e = getenv("GLM_EPOCH_EARLY_TRIGGER");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    return v >= 0 ? v : (s->early_trigger ? 1 : 0);
}

// 104 registers (2 CTAs of 256 threads: 53 K of the SM's 64 K) leave room for
// one 256-thread CTA of <= 48 registers next to the epoch on every SM — the
// side-stream permutation of the next round (prng.cu region kernels) then runs
// under the epoch instead of taking SM slots from the next turn and epoch.
// Measured (bench.py C2, one 4-GPU box, 2 runs each; 121 registers before):
// 1924 -> 1994 / 3816 -> 3947 / 6760 -> 7003 epochs/s at 1 / 2 / 4 GPUs, C4
// 194 -> 198.  No spills in the sparse instantiations (GLM_EPOCH_MAXNREG
// overrides for experiments).
#ifndef GLM_EPOCH_MAXNREG
#define GLM_EPOCH_MAXNREG 104
#endif
template <int G, int R, bool DENSE, int CM>
__global__ void __maxnreg__(GLM_EPOCH_MAXNREG) scd_async(EpochParams p) {
    SolveState *st = p.st;
    pdl_wait();
    // pdl 2: the round turn may be scheduled at once — its blocks take SM
    // slots as this grid's CTAs retire (one full wave, so none is displaced)
    // and wait in griddepcontrol.wait for this grid to complete
    if (p.pdl == 2) pdl_trigger();
    if (skip_attempt(st, p.seq)) return;
    tl_start(TL_EPOCH);
    // CM bit 0: gather the view through L1 (ld.ca); bit 1: stream the column
    // with L1::no_allocate + L2 evict_first, view traffic evict_last.
    const uint64_t pol_col = (CM & 2) ? policy_evict_first() : 0;
    const uint64_t pol_view = (CM & 2) ? policy_evict_last() : 0;
    auto ld_view = [&](const double *a) -> double {
        if (CM == 0) return ld_cg(a);
        if (CM == 1) return __ldca(a);
        if (CM == 2) return ld_cg_hint(a, pol_view);
        return ld_ca_hint(a, pol_view);
    };
    auto ld_val = [&](const double *a) -> double {
        return (CM & 2) ? ld_stream_f64(a, pol_col) : __ldg(a);
    };
    auto ld_row = [&](const int32_t *a) -> int {
        return (CM & 2) ? ld_stream_i32(a, pol_col) : __ldg(a);
    };
    auto scatter = [&](double *a, double v) {
        if (CM & 2) red_add_hint(a, v, pol_view);
        else red_add(a, v);
    };
    const int dc = st->dc;
    const double damping = st->damping;
    const double *__restrict__ dcur = delta_cur(p, dc);
    double *__restrict__ dnext = delta_next(p, dc);
    double *view = st->vw ? p.view1 : p.view0;
    constexpr int GPW = 32 / G;
    const int lane = threadIdx.x & 31;
    const int sub = lane / G, gl = lane % G;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int kind = p.kind;
    double gacc = 0.0;
    for (int64_t kb = warp * GPW; kb < p.m; kb += nwarps * GPW) {
        const int64_t k = kb + sub;
        const bool valid = k < p.m;
        const int j = valid ? __ldg(p.perm + k) : 0;
        int64_t lo = 0, hi = 0;
        double sj = 0.0;
        if (valid) {
            if (DENSE) {
                lo = (int64_t)j * p.d;
                hi = lo + p.d;
            } else if (CM & 4) {           // one 16-byte record: bounds and |a_j|^2
                const longlong2 rec = __ldg(p.meta + j);
                const int64_t cnt = (int64_t)((unsigned long long)rec.x >> 40);
                lo = rec.x & ((1LL << 40) - 1);
                hi = lo + cnt;
                if (cnt == META_CNT_SENTINEL) {
                    lo = __ldg(p.indptr + j);
                    hi = __ldg(p.indptr + j + 1);
                }
                sj = __longlong_as_double(rec.y);
            } else {
                lo = __ldg(p.indptr + j);
                hi = __ldg(p.indptr + j + 1);
            }
        }
        // group leader prefetches the coordinate's metadata under the gather
        double bj = 0.0, dj = 0.0, yj = 0.0;
        if (valid && gl == 0) {
            bj = __ldg(p.base + j);
            dj = dcur ? dcur[j] : 0.0;
            if (!(CM & 4)) sj = __ldg(p.sq + j);
            if (p.y) yj = __ldg(p.y + j);
        }
        int rr[R];
        double vv[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int64_t q = lo + gl + i * G;
            const bool in = q < hi;
            rr[i] = in ? (DENSE ? (int)(q - lo) : ld_row(p.rows + q)) : 0;
            vv[i] = in ? ld_val(p.vals + q) : 0.0;
        }
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < R; ++i)
            if (lo + gl + i * G < hi) acc += vv[i] * ld_view(view + rr[i]);
        for (int64_t q = lo + gl + R * G; q < hi; q += G) {
            const int r = DENSE ? (int)(q - lo) : ld_row(p.rows + q);
            acc += ld_val(p.vals + q) * ld_view(view + r);
        }
        const double ga = group_sum<G>(acc);
        double step = 0.0;
        if (valid && gl == 0) {
            const double t = bj + dj;
            double raw = 0.0;
            if (!coord_step(kind, p.lam, p.rho, yj, ga, p.quad * sj, t, raw)) {
                flag_error(st);
                raw = 0.0;
            }
            step = damping * raw;
            const double dn = step != 0.0 ? dj + step : dj;
            dnext[j] = dn;
            gacc += g_one(kind, p.lam, p.rho, yj, bj + dn);
        }
        step = __shfl_sync(0xffffffffu, step, sub * G);
        if (step != 0.0) {
            const double f = p.quad * step;
#pragma unroll
            for (int i = 0; i < R; ++i)
                if (lo + gl + i * G < hi) scatter(view + rr[i], f * vv[i]);
            for (int64_t q = lo + gl + R * G; q < hi; q += G) {
                const int r = DENSE ? (int)(q - lo) : ld_row(p.rows + q);
                scatter(view + r, f * ld_val(p.vals + q));
            }
        }
    }
    store_block_gsum(gacc, p.gpart, st);
    pdl_trigger();
    tl_end(TL_EPOCH);
}


// ------------------------------------------------------ narrow dense
// Dense columns with d <= 32*R rows (C3: HIGGS-shaped, d = 28).  Lane l of a
// warp owns rows l, l+32, ... of the column and of the view, so a coordinate
// is R coalesced loads, R FMAs, one butterfly all-reduce (every lane ends
// with the same bits, so every lane takes the same step) and R FMAs — no
// shared-vector traffic on the critical path.  The next coordinate's column
// and metadata are loaded while the current one is stepped.

template <int R>
struct NarrowCol {
    double a[R];
    double b, dj, s, y;
    int j;
};

template <int R>
__device__ __forceinline__ void narrow_load_j(const EpochParams &p, const double *dcur, int j,
                                              NarrowCol<R> &c) {
    const int lane = threadIdx.x & 31;
    c.j = j;
    const double *col = p.vals + (int64_t)j * p.d;
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int r = lane + 32 * i;
        c.a[i] = r < p.d ? __ldg(col + r) : 0.0;
    }
    c.b = __ldg(p.base + j);
    c.dj = dcur ? dcur[j] : 0.0;
    c.s = __ldg(p.sq + j);
    c.y = p.y ? __ldg(p.y + j) : 0.0;
}

template <int R>
__device__ __forceinline__ void narrow_load(const EpochParams &p, const double *dcur, int64_t k,
                                            NarrowCol<R> &c) {
    narrow_load_j<R>(p, dcur, __ldg(p.perm + k), c);
}

__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic mode (run_pass n_threads=1, solver.py:202-211): one warp, the
// view in registers.
template <int R>
__global__ void __launch_bounds__(32) scd_seq_narrow(EpochParams p) {
    SolveState *st = p.st;
    if (skip_attempt(st, p.seq)) return;
    const int dc = st->dc;
    const double damping = st->damping;
    const double *dcur = delta_cur(p, dc);
    double *dnext = delta_next(p, dc);
    double *view = st->vw ? p.view1 : p.view0;
    const int lane = threadIdx.x;
    double v[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int r = lane + 32 * i;
        v[i] = r < p.d ? view[r] : 0.0;
    }
    const int kind = p.kind;
    double gacc = 0.0;
    // two-stage pipeline: permutation entry k + 2 and column k + 1 in flight
    NarrowCol<R> nx;
    int jn = 0;
    if (p.m > 0) narrow_load<R>(p, dcur, 0, nx);
    if (p.m > 1) jn = __ldg(p.perm + 1);
    for (int64_t k = 0; k < p.m; ++k) {
        const NarrowCol<R> c = nx;
        if (k + 1 < p.m) narrow_load_j<R>(p, dcur, jn, nx);
        if (k + 2 < p.m) jn = __ldg(p.perm + k + 2);
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < R; ++i) acc += c.a[i] * v[i];
        const double ga = warp_allsum(acc);
        double raw = 0.0;
        if (!coord_step(kind, p.lam, p.rho, c.y, ga, p.quad * c.s, c.b + c.dj, raw)) {
            if (lane == 0) flag_error(st);
            raw = 0.0;
        }
        const double step = damping * raw;
        const double dn = step != 0.0 ? c.dj + step : c.dj;
        if (lane == 0) {
            dnext[c.j] = dn;
            gacc += g_one(kind, p.lam, p.rho, c.y, c.b + dn);
        }
        if (step != 0.0) {
            const double f = p.quad * step;
#pragma unroll
            for (int i = 0; i < R; ++i) v[i] += f * c.a[i];
        }
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int r = lane + 32 * i;
        if (r < p.d) view[r] = v[i];
    }
    if (lane == 0) {
        p.gpart[0] = gacc;
        st->epoch_blocks = 1;
    }
}

// Asynchronous mode (TPA-SCD) for narrow dense data: a global red.add per
// row per coordinate would serialise every coordinate on the same d L2
// addresses, so each warp keeps its own pending Delta view in registers and
// reads view = (CTA snapshot of the shared view) + (its own pending).  Every
// `per_phase` coordinates per warp the CTA folds the warps' pendings, adds
// them to the shared view with one atom.add per row, and refreshes its
// snapshot from the values the atomics returned.  Staleness is bounded by
// grid x warps x per_phase coordinates (the in-flight budget); the damping
// check of the value kernel guards the epoch as for scd_async.
// The shared view lives, for the kernel's duration, in `vpad` with one row
// per 1 KB (PAD_STRIDE doubles) so the d rows hash to d different L2 slices
// (address bits 10+); contiguous, all CTAs' atomics would queue on the one
// or two slices holding the view's 224 bytes.
constexpr int PAD_STRIDE = 128;
constexpr int NARROW_MAX_ROWS = 1024;   // dense views kept in registers (32 per lane)

__global__ void narrow_pad_kernel(const SolveState *st, const double *view0, const double *view1,
                                  double *vpad, int64_t d, int64_t seq) {
    if (skip_attempt(st, seq)) return;
    const double *view = st->vw ? view1 : view0;
    for (int64_t r = threadIdx.x; r < d; r += blockDim.x) vpad[r * PAD_STRIDE] = view[r];
}

template <int R>
__global__ void __launch_bounds__(256) scd_replica(EpochParams p, int per_phase, double *vpad) {
    SolveState *st = p.st;
    if (skip_attempt(st, p.seq)) return;
    __shared__ double snap[32 * R];
    __shared__ double fold[32 * R];
    __shared__ int s_last;
    const int dc = st->dc;
    const double damping = st->damping;
    const double *dcur = delta_cur(p, dc);
    double *dnext = delta_next(p, dc);
    double *view = st->vw ? p.view1 : p.view0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarp = blockDim.x >> 5;
    for (int r = threadIdx.x; r < 32 * R; r += blockDim.x) {
        snap[r] = r < p.d ? ld_cg(vpad + (int64_t)r * PAD_STRIDE) : 0.0;
        fold[r] = 0.0;
    }
    __syncthreads();
    const int kind = p.kind;
    double gacc = 0.0;
    double pend[R];
#pragma unroll
    for (int i = 0; i < R; ++i) pend[i] = 0.0;
    const int64_t per_cta = (int64_t)nwarp * per_phase;
    const int64_t stride = (int64_t)gridDim.x * per_cta;
    // rows threadIdx.x + 256 q (q < RPT) of the view: their last publish
    constexpr int RPT = (32 * R + 255) / 256;
    double prev_old[RPT], prev_x[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) prev_old[q] = prev_x[q] = 0.0;
    bool have_prev = false;
    // This warp's coordinates: position t -> k(t) = base + (t / P) * stride +
    // t % P.  Two-stage software pipeline: the permutation entry of t + 2 and
    // the column of t + 1 are in flight while t is stepped (the column load
    // depends on the permutation load, so one stage alone would leave both
    // latencies on the critical path of a short phase).
    // position -> coordinate index, advanced without divisions: inside a
    // phase k + 1, at its end the same slot of the next phase (k - i + stride)
    struct Pos {
        int64_t k;
        int i;
    };
    auto adv = [&](Pos q) -> Pos {
        return q.i + 1 < per_phase ? Pos{q.k + 1, q.i + 1} : Pos{q.k - q.i + stride, 0};
    };
    Pos p0{(int64_t)blockIdx.x * per_cta + (int64_t)warp * per_phase, 0};
    Pos p1 = adv(p0), p2 = adv(p1);
    NarrowCol<R> cur;
    int jn = 0;
    if (p0.k < p.m) narrow_load<R>(p, dcur, p0.k, cur);
    if (p1.k < p.m) jn = __ldg(p.perm + p1.k);
    for (int64_t k0 = (int64_t)blockIdx.x * per_cta; k0 < p.m; k0 += stride) {
        for (int ii = 0; ii < per_phase; ++ii) {
            if (p0.k >= p.m) break;
            const NarrowCol<R> c = cur;
            if (p1.k < p.m) narrow_load_j<R>(p, dcur, jn, cur);
            if (p2.k < p.m) jn = __ldg(p.perm + p2.k);
            p0 = p1;
            p1 = p2;
            p2 = adv(p2);
            double acc = 0.0;
#pragma unroll
            for (int i = 0; i < R; ++i) acc += c.a[i] * (snap[lane + 32 * i] + pend[i]);
            const double ga = warp_allsum(acc);
            double raw = 0.0;
            if (!coord_step(kind, p.lam, p.rho, c.y, ga, p.quad * c.s, c.b + c.dj, raw)) {
                if (lane == 0) flag_error(st);
                raw = 0.0;
            }
            const double step = damping * raw;
            const double dn = step != 0.0 ? c.dj + step : c.dj;
            if (lane == 0) {
                dnext[c.j] = dn;
                gacc += g_one(kind, p.lam, p.rho, c.y, c.b + dn);
            }
            if (step != 0.0) {
                const double f = p.quad * step;
#pragma unroll
                for (int i = 0; i < R; ++i) pend[i] += f * c.a[i];
            }
        }
        // phase end: fold the warps' pendings and publish them.  The publish's
        // returned value is consumed one phase later (thread r owns row r), so
        // the atomic round trip overlaps the next phase's coordinates; the
        // snapshot gets the CTA's own contributions at once and the other
        // CTAs' one phase late.
#pragma unroll
        for (int i = 0; i < R; ++i)
            if (pend[i] != 0.0) atomicAdd(&fold[lane + 32 * i], pend[i]);
        __syncthreads();
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int r = threadIdx.x + 256 * q;
            if (r < p.d) {
                const double x = fold[r];
                fold[r] = 0.0;
                snap[r] = have_prev ? prev_old[q] + prev_x[q] + x : snap[r] + x;
                prev_old[q] = atomicAdd(vpad + (int64_t)r * PAD_STRIDE, x);
                prev_x[q] = x;
            }
        }
        have_prev = true;
#pragma unroll
        for (int i = 0; i < R; ++i) pend[i] = 0.0;
        __syncthreads();
    }
    // the last CTA to finish writes the shared view back
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&st->block_counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        for (int r = threadIdx.x; r < p.d; r += blockDim.x)
            view[r] = ld_cg(vpad + (int64_t)r * PAD_STRIDE);
        __syncthreads();
        if (threadIdx.x == 0) st->block_counter = 0;
    }
    store_block_gsum(gacc, p.gpart, st);
}

// ----------------------------------------------------------- sequential
// One CTA of BS threads walks the permutation in order (run_pass with
// n_threads=1, solver.py:202-211).  Deterministic: fixed per-thread strides
// and a fixed reduction tree.
template <int BS, bool SMEM, bool DENSE>
__global__ void __launch_bounds__(BS) scd_seq(EpochParams p) {
    SolveState *st = p.st;
    if (skip_attempt(st, p.seq)) return;
    extern __shared__ double sview[];
    __shared__ double sred[32];
    __shared__ double sstep;
    const int dc = st->dc;
    const double damping = st->damping;
    const double *dcur = delta_cur(p, dc);
    double *dnext = delta_next(p, dc);
    double *gview = st->vw ? p.view1 : p.view0;
    double *V = SMEM ? sview : gview;
    const int t = threadIdx.x;
    if (SMEM) {
        for (int64_t r = t; r < p.d; r += BS) sview[r] = gview[r];
        __syncthreads();
    }
    const int kind = p.kind;
    double gacc = 0.0;
    for (int64_t k = 0; k < p.m; ++k) {
        const int j = p.perm[k];
        int64_t lo, hi;
        if (DENSE) {
            lo = (int64_t)j * p.d;
            hi = lo + p.d;
        } else {
            lo = p.indptr[j];
            hi = p.indptr[j + 1];
        }
        double acc = 0.0;
        for (int64_t q = lo + t; q < hi; q += BS) {
            const int r = DENSE ? (int)(q - lo) : p.rows[q];
            acc += p.vals[q] * V[r];
        }
        acc = warp_sum(acc);
        if (BS > 32) {
            if ((t & 31) == 0) sred[t >> 5] = acc;
            __syncthreads();
            if (t < 32) {
                double x = t < BS / 32 ? sred[t] : 0.0;
                acc = warp_sum(x);
            }
        }
        if (t == 0) {
            const double dj = dcur ? dcur[j] : 0.0;
            const double yj = p.y ? p.y[j] : 0.0;
            const double tt = p.base[j] + dj;
            double raw = 0.0;
            if (!coord_step(kind, p.lam, p.rho, yj, acc, p.quad * p.sq[j], tt, raw)) {
                flag_error(st);
                raw = 0.0;
            }
            const double step = damping * raw;
            const double dn = step != 0.0 ? dj + step : dj;
            dnext[j] = dn;
            gacc += g_one(kind, p.lam, p.rho, yj, p.base[j] + dn);
            sstep = step;
        }
        if (BS > 32) __syncthreads(); else __syncwarp();
        const double step = sstep;
        if (step != 0.0) {
            const double f = p.quad * step;
            for (int64_t q = lo + t; q < hi; q += BS) {
                const int r = DENSE ? (int)(q - lo) : p.rows[q];
                V[r] += f * p.vals[q];
            }
        }
        if (BS > 32) __syncthreads(); else __syncwarp();
    }
    if (SMEM) {
        for (int64_t r = t; r < p.d; r += BS) gview[r] = sview[r];
    }
    if (t == 0) {
        p.gpart[0] = gacc;
        st->epoch_blocks = 1;
    }
}

// Deterministic CSC epoch for short columns (<= 32 R entries in registers):
// one warp, with the permutation entry of k + 3, the column bounds of k + 2
// and the column + metadata of k + 1 in flight while k is stepped, and the
// scatter written from the gathered values (no re-load).  Same arithmetic,
// in the same order, as scd_seq<32>.
template <int R, bool SMEM>
__global__ void __launch_bounds__(32) scd_seq_csc(EpochParams p) {
    SolveState *st = p.st;
    if (skip_attempt(st, p.seq)) return;
    extern __shared__ double sview[];
    const int dc = st->dc;
    const double damping = st->damping;
    const double *dcur = delta_cur(p, dc);
    double *dnext = delta_next(p, dc);
    double *gview = st->vw ? p.view1 : p.view0;
    double *V = SMEM ? sview : gview;
    const int lane = threadIdx.x;
    if (SMEM) {
        for (int64_t r = lane; r < p.d; r += 32) sview[r] = gview[r];
        __syncwarp();
    }
    struct Col {
        int j;
        int64_t lo, hi;
        int rows[R];
        double vals[R];
        double b, dj, s, y;
    };
    auto load_col = [&](int j, int64_t lo, int64_t hi, Col &c) {
        c.j = j;
        c.lo = lo;
        c.hi = hi;
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int64_t q = lo + lane + 32 * i;
            const bool in = q < hi;
            c.rows[i] = in ? __ldg(p.rows + q) : 0;
            c.vals[i] = in ? __ldg(p.vals + q) : 0.0;
        }
        c.b = __ldg(p.base + j);
        c.dj = dcur ? dcur[j] : 0.0;
        c.s = __ldg(p.sq + j);
        c.y = p.y ? __ldg(p.y + j) : 0.0;
    };
    const int64_t m = p.m;
    Col cur;
    int jA = 0, jB = 0;
    int64_t loA = 0, hiA = 0;
    if (m > 0) {
        const int j0 = __ldg(p.perm);
        load_col(j0, __ldg(p.indptr + j0), __ldg(p.indptr + j0 + 1), cur);
    }
    if (m > 1) {
        jA = __ldg(p.perm + 1);
        loA = __ldg(p.indptr + jA);
        hiA = __ldg(p.indptr + jA + 1);
    }
    if (m > 2) jB = __ldg(p.perm + 2);
    const int kind = p.kind;
    double gacc = 0.0;
    for (int64_t k = 0; k < m; ++k) {
        const Col c = cur;
        int64_t loB = 0, hiB = 0;
        int jC = 0;
        if (k + 1 < m) load_col(jA, loA, hiA, cur);
        if (k + 2 < m) {
            loB = __ldg(p.indptr + jB);
            hiB = __ldg(p.indptr + jB + 1);
        }
        if (k + 3 < m) jC = __ldg(p.perm + k + 3);
        double g[R];
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < R; ++i) {
            g[i] = c.lo + lane + 32 * i < c.hi ? V[c.rows[i]] : 0.0;
            if (c.lo + lane + 32 * i < c.hi) acc += c.vals[i] * g[i];
        }
        for (int64_t q = c.lo + lane + 32 * R; q < c.hi; q += 32) acc += p.vals[q] * V[p.rows[q]];
        acc = warp_sum(acc);
        double raw = 0.0;
        if (!coord_step(kind, p.lam, p.rho, c.y, acc, p.quad * c.s, c.b + c.dj, raw)) {
            if (lane == 0) flag_error(st);
            raw = 0.0;
        }
        const double step = damping * raw;
        const double dn = step != 0.0 ? c.dj + step : c.dj;
        if (lane == 0) {
            dnext[c.j] = dn;
            gacc += g_one(kind, p.lam, p.rho, c.y, c.b + dn);
        }
        if (step != 0.0) {
            const double f = p.quad * step;
#pragma unroll
            for (int i = 0; i < R; ++i)
                if (c.lo + lane + 32 * i < c.hi) V[c.rows[i]] = g[i] + f * c.vals[i];
            for (int64_t q = c.lo + lane + 32 * R; q < c.hi; q += 32) V[p.rows[q]] += f * p.vals[q];
        }
        __syncwarp();
        jA = jB;
        loA = loB;
        hiA = hiB;
        jB = jC;
    }
    if (SMEM) {
        for (int64_t r = lane; r < p.d; r += 32) gview[r] = sview[r];
    }
    if (lane == 0) {
        p.gpart[0] = gacc;
        st->epoch_blocks = 1;
    }
}

// ------------------------------------------- sequential, level-scheduled
// The deterministic epoch with the same bits as scd_seq_csc, but with many
// coordinates in flight.  Coordinates whose columns share no row commute
// exactly: the later one's gather does not see the earlier one's scatter.  So
// a window of consecutive permutation entries is cut into levels — a
// coordinate's level is one more than the highest level of an EARLIER window
// entry it shares a row with — and the levels run one after another, each
// level's coordinates concurrently.  Every coordinate then gathers exactly
// the view the sequential walk would have shown it, and every row receives
// the same writes in the same order, so view, delta and the epoch's g-sum
// (summed afterwards in permutation order) are bit-identical to scd_seq_csc.
//
// Warp 0 plans window w+1 (permutation entries, column bounds, rows staged
// through shared memory with cp.async, levels from a shared row -> level+1
// table, cleared again right after the window is planned) while warps
// 1..NW execute window w.
constexpr int LVL_THREADS = 512;
constexpr int LVL_WORKERS = LVL_THREADS / 32 - 1;
constexpr int LVL_WINDOW = 256;
constexpr int LVL_MAX = 31;                      // levels 0..30 per window
constexpr int LVL_STAGE = 64;                    // staged rows per planned column
constexpr int64_t LVL_TAB_MAX = 128 * 1024;      // rows with an in-smem level table
constexpr int64_t LVL_SMEM_VIEW_MAX = 8 * 1024;  // doubles kept in shared memory
constexpr size_t LVL_STAGE_BYTES = sizeof(uint32_t) * LVL_WINDOW * LVL_STAGE;

struct LvlPlan {
    int64_t lo[LVL_WINDOW];
    int j[LVL_WINDOW];
    int cnt[LVL_WINDOW];
    double gterm[LVL_WINDOW];    // b + delta of the entry, then g(b + delta)
    double gy[LVL_WINDOW];       // the entry's y (dual_ridge)
    uint16_t order[LVL_WINDOW];
    uint8_t lvl[LVL_WINDOW];
    uint16_t lstart[LVL_MAX + 1];
    int n, nlev;
    int64_t k0;
};

__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}
__device__ __forceinline__ void workers_sync() {
    asm volatile("bar.sync 1, %0;" ::"r"(LVL_WORKERS * 32) : "memory");
}

// Warp 0: plan the window of permutation entries starting at k0.  The
// window's permutation entries and column bounds are loaded with every load
// in flight, its rows (up to LVL_STAGE per column) staged into shared memory
// with cp.async, then the entries get their levels one after another from
// the row -> level+1 table, which is cleared again from the staged rows.
// GLM_LVL_DEBUG=1: the kernel prints where its time went (cycles of warp 0
// planning, per planning phase, and of worker warp 1 executing; windows, levels)
__device__ int lvl_debug = 0;
__device__ unsigned long long lvl_phase[6];

__device__ void lvl_plan(const EpochParams &p, LvlPlan &P, int64_t k0, uint8_t *tab,
                         uint32_t (*stage)[LVL_STAGE]) {
    const int lane = threadIdx.x & 31;
    long long tp = clock64();
    auto mark = [&](int i) {
        if (lvl_debug && lane == 0) {
            const long long t = clock64();
            lvl_phase[i] += (unsigned long long)(t - tp);
            tp = t;
        }
    };
    const int64_t rem = p.m - k0;
    const int nmax = rem < LVL_WINDOW ? (int)rem : LVL_WINDOW;
    constexpr int U = LVL_WINDOW / 32;
    int jj[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int c = u * 32 + lane;
        jj[u] = c < nmax ? __ldg(p.perm + k0 + c) : 0;
    }
    int64_t lo[U], hi[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int c = u * 32 + lane;
        lo[u] = c < nmax ? __ldg(p.indptr + jj[u]) : 0;
        hi[u] = c < nmax ? __ldg(p.indptr + jj[u] + 1) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int c = u * 32 + lane;
        if (c < nmax) {
            P.j[c] = jj[u];
            P.lo[c] = lo[u];
            P.cnt[c] = (int)(hi[u] - lo[u]);
        }
    }
    // stage the rows: lane l copies the columns l, l + 32, ... (bounds in registers)
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int c = u * 32 + lane;
        const int64_t cu = hi[u] - lo[u];
        const int ci = c < nmax ? (cu < LVL_STAGE ? (int)cu : LVL_STAGE) : 0;
        for (int q = 0; q < ci; ++q) cp_async4(&stage[c][q], p.rows + lo[u] + q);
    }
    mark(0);
    cp_async_wait_all();
    __syncwarp();
    mark(1);
    // levels, one entry after another: the chain per entry is the table
    // reads, one redux.sync max and the table writes (the entry's staged rows
    // are read into registers one entry ahead)
    int n = 0, maxlev = -1;
    int r0n = 0, r1n = 0, cin = 0;
    auto rows_of = [&](int c, int &r0, int &r1, int &ci) {
        ci = P.cnt[c];
        r0 = lane < ci ? (int)stage[c][lane] : -1;
        r1 = lane + 32 < ci && lane + 32 < LVL_STAGE ? (int)stage[c][lane + 32] : -1;
    };
    bool longcols = false;
    if (nmax > 0) rows_of(0, r0n, r1n, cin);
    for (int c = 0; c < nmax; ++c) {
        const int r0 = r0n, r1 = r1n, ci = cin;
        if (c + 1 < nmax) rows_of(c + 1, r0n, r1n, cin);
        int lv = -1;
        if (r0 >= 0) lv = (int)tab[r0] - 1;
        if (r1 >= 0) lv = max(lv, (int)tab[r1] - 1);
        if (ci > LVL_STAGE) {              // rows past the staged ones (rare)
            longcols = true;
            for (int q = LVL_STAGE + lane; q < ci; q += 32)
                lv = max(lv, (int)tab[__ldg(p.rows + P.lo[c] + q)] - 1);
        }
        const int level = __reduce_max_sync(0xffffffffu, lv) + 1;
        if (level >= LVL_MAX) break;       // the window closes before this entry
        if (r0 >= 0) tab[r0] = (uint8_t)(level + 1);
        if (r1 >= 0) tab[r1] = (uint8_t)(level + 1);
        if (ci > LVL_STAGE)
            for (int q = LVL_STAGE + lane; q < ci; q += 32)
                tab[__ldg(p.rows + P.lo[c] + q)] = (uint8_t)(level + 1);
        if (lane == 0) P.lvl[c] = (uint8_t)level;
        maxlev = max(maxlev, level);
        n = c + 1;
        __syncwarp();
    }
    __syncwarp();
    mark(2);
    // the table only serves dependencies inside a window: clear this one's
    // rows (eight entries' staged rows read before any is cleared)
    for (int c0 = 0; c0 < n; c0 += 8) {
        int ra[8], rb[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int c = c0 + u;
            const int ci = c < n ? P.cnt[c] : 0;
            ra[u] = lane < ci ? (int)stage[c][lane] : -1;
            rb[u] = lane + 32 < ci && lane + 32 < LVL_STAGE ? (int)stage[c][lane + 32] : -1;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (ra[u] >= 0) tab[ra[u]] = 0;
            if (rb[u] >= 0) tab[rb[u]] = 0;
        }
    }
    if (__any_sync(0xffffffffu, longcols))
        for (int c = 0; c < n; ++c)
            for (int q = LVL_STAGE + lane; q < P.cnt[c]; q += 32) tab[__ldg(p.rows + P.lo[c] + q)] = 0;
    __syncwarp();
    mark(3);
    if (lane == 0) {
        P.n = n;
        P.nlev = maxlev + 1;
        P.k0 = k0;
    }
    __syncwarp();
    mark(4);
}

// One executing warp: the stable counting sort of the planned window's
// entries by level (order, lstart) — off the planner's critical path.
__device__ void lvl_sort(LvlPlan &P) {
    const int lane = threadIdx.x & 31;
    const int n = P.n, nlev = P.nlev;
    int base = 0;
    for (int L = 0; L < nlev; ++L) {
        if (lane == 0) P.lstart[L] = (uint16_t)base;
        for (int c0 = 0; c0 < n; c0 += 32) {
            const int c = c0 + lane;
            const bool hit = c < n && P.lvl[c] == L;
            const unsigned bal = __ballot_sync(0xffffffffu, hit);
            if (hit) P.order[base + __popc(bal & ((1u << lane) - 1))] = (uint16_t)c;
            base += __popc(bal);
        }
    }
    if (lane == 0) P.lstart[nlev] = (uint16_t)base;
    __syncwarp();
}


template <bool SMEM>
__global__ void __launch_bounds__(LVL_THREADS) scd_seq_lvl(EpochParams p) {
    SolveState *st = p.st;
    if (skip_attempt(st, p.seq)) return;
    extern __shared__ __align__(16) unsigned char lvl_smem[];
    __shared__ LvlPlan plans[2];
    // dynamic: [staged rows of the planned window][view (SMEM)][row table]
    uint32_t(*stage)[LVL_STAGE] = reinterpret_cast<uint32_t(*)[LVL_STAGE]>(lvl_smem);
    double *sview = reinterpret_cast<double *>(lvl_smem + LVL_STAGE_BYTES);
    uint8_t *tab = lvl_smem + LVL_STAGE_BYTES + (SMEM ? sizeof(double) * ((p.d + 1) & ~1LL) : 0);
    const int dc = st->dc;
    const double damping = st->damping;
    const double *dcur = delta_cur(p, dc);
    double *dnext = delta_next(p, dc);
    double *gview = st->vw ? p.view1 : p.view0;
    double *V = SMEM ? sview : gview;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t r = threadIdx.x; r < p.d; r += blockDim.x) {
        if (SMEM) sview[r] = gview[r];
        tab[r] = 0;
    }
    __syncthreads();
    if (warp == 0) lvl_plan(p, plans[0], 0, tab, stage);
    __syncthreads();
    const int kind = p.kind;
    double gacc = 0.0;
    struct Col {
        int j, cnt, slot;
        int64_t lo;
        int rows[3];
        double vals[3];
        double b, dj, s, y;
    };
    long long dbg_busy = 0, dbg_levels = 0, dbg_windows = 0;
    const long long dbg_t0 = clock64();
    for (int w = 0;; ++w) {
        LvlPlan &P = plans[w & 1];
        const int n = P.n;
        const long long dbg_w0 = clock64();
        if (n == 0) break;
        if (warp == 0) {
            const int64_t k1 = P.k0 + n;
            if (k1 < p.m) lvl_plan(p, plans[(w + 1) & 1], k1, tab, stage);
            else if (lane == 0) plans[(w + 1) & 1].n = 0;
        } else {
            const int me = warp - 1;
            const int tw = me * 32 + lane;
            if (me == 0) lvl_sort(P);           // order / lstart of this window
            workers_sync();
            auto load = [&](int e, Col &c) {
                const int slot = P.order[e];
                c.slot = slot;
                c.j = P.j[slot];
                c.lo = P.lo[slot];
                c.cnt = P.cnt[slot];
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    const bool in = lane + 32 * i < c.cnt;
                    c.rows[i] = in ? __ldg(p.rows + c.lo + lane + 32 * i) : 0;
                    c.vals[i] = in ? __ldg(p.vals + c.lo + lane + 32 * i) : 0.0;
                }
                c.b = __ldg(p.base + c.j);
                c.dj = dcur ? dcur[c.j] : 0.0;
                c.s = __ldg(p.sq + c.j);
                c.y = p.y ? __ldg(p.y + c.j) : 0.0;
            };
            // this worker's entries, level after level; the next one's column
            // (independent of the view) is loaded before the current one steps
            const int nlev = P.nlev;
            int L = 0;
            int e = P.lstart[0] + me;
            auto advance = [&](int &e_, int &L_) {      // next own entry, possibly a later level
                while (L_ < nlev && e_ >= P.lstart[L_ + 1]) {
                    ++L_;
                    if (L_ < nlev) e_ = P.lstart[L_] + me;
                }
            };
            advance(e, L);
            Col nx;
            if (L < nlev) load(e, nx);
            int cur_level = 0;
            while (L < nlev) {
                while (cur_level < L) {      // levels this worker has nothing in
                    workers_sync();
                    ++cur_level;
                }
                const Col c = nx;
                int e2 = e + LVL_WORKERS, L2 = L;
                advance(e2, L2);
                if (L2 < nlev) load(e2, nx);
                double g[3];
                double acc = 0.0;
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    g[i] = lane + 32 * i < c.cnt ? V[c.rows[i]] : 0.0;
                    if (lane + 32 * i < c.cnt) acc += c.vals[i] * g[i];
                }
                for (int q = lane + 96; q < c.cnt; q += 32) acc += p.vals[c.lo + q] * V[p.rows[c.lo + q]];
                acc = warp_sum(acc);
                double raw = 0.0;
                if (!coord_step(kind, p.lam, p.rho, c.y, acc, p.quad * c.s, c.b + c.dj, raw)) {
                    if (lane == 0) flag_error(st);
                    raw = 0.0;
                }
                const double step = damping * raw;
                const double dn = step != 0.0 ? c.dj + step : c.dj;
                if (step != 0.0) {          // the scatter first: the next level waits on it
                    const double f = p.quad * step;
#pragma unroll
                    for (int i = 0; i < 3; ++i)
                        if (lane + 32 * i < c.cnt) V[c.rows[i]] = g[i] + f * c.vals[i];
                    for (int q = lane + 96; q < c.cnt; q += 32) V[p.rows[c.lo + q]] += f * p.vals[c.lo + q];
                }
                if (lane == 0) {
                    dnext[c.j] = dn;
                    P.gterm[c.slot] = c.b + dn;     // g() applied by warp 0 after the window
                    P.gy[c.slot] = c.y;
                }
                __syncwarp();
                e = e2;
                L = L2;
            }
            while (cur_level < nlev) {       // the barriers of the remaining levels
                workers_sync();
                ++cur_level;
            }
            dbg_levels += nlev;
            // g(b + delta) of the window's entries in parallel, then summed in
            // permutation order (scd_seq_csc's sum: the same bits)
            const long long tg = clock64();
            for (int c = tw; c < n; c += LVL_WORKERS * 32)
                P.gterm[c] = g_one(kind, p.lam, p.rho, P.gy[c], P.gterm[c]);
            workers_sync();
            if (tw == 0) {
                for (int c = 0; c < n; ++c) gacc += P.gterm[c];
                if (lvl_debug) lvl_phase[5] += (unsigned long long)(clock64() - tg);
            }
        }
        dbg_busy += clock64() - dbg_w0;
        ++dbg_windows;
        __syncthreads();
    }
    if (lvl_debug && lane == 0 && warp <= 1)
        printf("scd_seq_lvl warp %d: busy %lld of %lld cycles, %lld windows, %lld levels\n", warp,
               dbg_busy, clock64() - dbg_t0, dbg_windows, dbg_levels);
    if (lvl_debug && threadIdx.x == 0)
        printf("scd_seq_lvl planner phases (cycles): loads+stage issue %llu, stage wait %llu, "
               "levels %llu, clear %llu, bookkeeping %llu; workers' g-sum %llu\n", lvl_phase[0], lvl_phase[1],
               lvl_phase[2], lvl_phase[3], lvl_phase[4], lvl_phase[5]);
    __syncthreads();
    if (SMEM)
        for (int64_t r = threadIdx.x; r < p.d; r += blockDim.x) gview[r] = sview[r];
    if (warp == 1 && lane == 0) {      // the workers' first thread holds the g-sum
        p.gpart[0] = gacc;
        st->epoch_blocks = 1;
    }
}

// ------------------------------------------------------- value + decide
// damped_solve's control flow after an attempt (solver.py:272-298; per chunk
// _train_chunk, pipeline.py:180-193) for the new value G (one thread).
__device__ __forceinline__ void decide_attempt(SolveState *st, double G, double gnew,
                                               double nonfinite, int chunked) {
    st->attempts += 1;
    if (nonfinite > 0.0) {         // solver.py:279-280
        st->status = GLM_SOLVER_ERROR;
        st->done = 1;
        return;
    }
    if (st->status != GLM_OK) {    // coordinate-level error (solver.py:160-161, 185-186)
        st->done = 1;
        return;
    }
    const double value = st->value;
    if (G > value) {
        st->vw ^= 1;               // restore the snapshot view; delta[dc] untouched
        if (G - value <= PLATEAU_REL * (1.0 + fabs(value))) {
            st->plateaued = 1;
            st->done = 1;
            return;
        }
        st->retries += 1;
        st->damping *= 0.5;
        if (st->damping < DAMPING_FLOOR) {
            st->status = GLM_DIVERGENCE;
            st->done = 1;
        }
        return;
    }
    st->value = G;
    st->gsum_acc = gnew;
    st->dc = st->dc == 0 ? 1 : 0;  // the buffer the epoch wrote
    if (!chunked && st->epochs_run < MAX_EPOCH_VALUES) st->epoch_values[st->epochs_run] = G;
    st->epochs_run += 1;
    if (st->epochs_run >= st->epochs_target) st->done = 1;
}

struct ValueParams {
    SolveState *st;
    int mode;   // 0: initial G; 1: after an attempt; 2: chunk g-sum of the accepted state
    int kind;
    double lam, rho, quad;
    const double *cnst;
    int64_t m, d;
    const double *lin, *base, *y;
    const double *dfull;    // modes 0/2: delta added to base (NULL = 0)
    int view_terms;         // mode 0: include (lin.u + u.u/2)/quad, u = view - lin
    int chunked;            // mode 1: G uses gsum_acc - gsum_old + the chunk's new g-sum
    int64_t seq;
    double *view0, *view1;
    double *partials;       // [blocks][3]
    const double *gpart;    // epoch partial g-sums
};

// G(delta) = const + lin.w + quad/2 |w|^2 + sum g(base + delta) with
// quad*w = view - lin, i.e. (lin.u + u.u/2)/quad for u = view - lin
// (LocalSubproblem.value_given_w, solver.py:132-135).  The g-sum of an
// attempt comes from the epoch kernel's block partials; G(0) sums g(base).
// Chunked mode (pipeline.py:158-197): the g-sum of an attempt over chunk c is
// the accepted total minus the chunk's accepted share (mode 2) plus the
// chunk's new share; an accepted chunk pass ends the chunk.
__global__ void __launch_bounds__(VALUE_THREADS) value_kernel(ValueParams p) {
    SolveState *st = p.st;
    if (skip_attempt(st, p.seq)) return;
    __shared__ double sm[96];
    __shared__ int s_last;
    const double *V = st->vw ? p.view1 : p.view0;
    double acc[3] = {0.0, 0.0, 0.0};   // g-sum | view terms | non-finite count
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    if (p.mode == 1 || (p.mode == 0 && p.view_terms)) {
        for (int64_t r = tid; r < p.d; r += nth) {
            const double v = V[r], l = p.lin[r];
            if (!isfinite(v)) acc[2] += 1.0;
            const double u = v - l;
            acc[1] += l * u + 0.5 * u * u;
        }
    }
    if (p.mode != 1) {
        for (int64_t j = tid; j < p.m; j += nth)
            acc[0] += g_one(p.kind, p.lam, p.rho, p.y ? p.y[j] : 0.0,
                            p.dfull ? p.base[j] + p.dfull[j] : p.base[j]);
    }
    block_sum<3>(acc, sm);
    if (threadIdx.x == 0) {
        p.partials[blockIdx.x * 3 + 0] = acc[0];
        p.partials[blockIdx.x * 3 + 1] = acc[1];
        p.partials[blockIdx.x * 3 + 2] = acc[2];
        __threadfence();
        const unsigned ticket = atomicAdd(&st->block_counter, 1u);
        s_last = ticket == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    double tot[3] = {0.0, 0.0, 0.0};
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
        tot[0] += __ldcg(p.partials + b * 3 + 0);
        tot[1] += __ldcg(p.partials + b * 3 + 1);
        tot[2] += __ldcg(p.partials + b * 3 + 2);
    }
    double gs[1] = {0.0};
    if (p.mode == 1) {
        const int eb = st->epoch_blocks;
        for (int b = threadIdx.x; b < eb; b += blockDim.x) gs[0] += __ldcg(p.gpart + b);
    }
    block_sum<3>(tot, sm);
    block_sum<1>(gs, sm);
    if (threadIdx.x != 0) return;
    st->block_counter = 0;
    if (p.mode == 2) {
        st->gsum_old = tot[0];
        return;
    }
    if (p.mode == 0) {
        const double G0 = *p.cnst + (p.view_terms ? tot[1] / p.quad : 0.0) + tot[0];
        st->value = G0;
        st->initial = G0;
        st->gsum_acc = tot[0];
        return;
    }
    const double gnew = p.chunked ? (st->gsum_acc - st->gsum_old) + gs[0] : gs[0];
    decide_attempt(st, *p.cnst + tot[1] / p.quad + gnew, gnew, tot[2], p.chunked);
}

// ---------------------------------------------------------- begin / end
// Resets the solve state, writes view0 = view1 = lin (the first attempt's
// snapshot), and — when the caller guarantees base == the previous solve's
// base + delta (an in-place fold) — takes G(0) = const + the cached g-sum.
__global__ void begin_kernel(SolveState *st, double *view0, double *view1, const double *lin,
                             int64_t d, int epochs, int reset_damping, const double *cnst,
                             int reuse_gsum) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = tid; r < d; r += nth) {
        const double l = lin[r];
        view0[r] = l;
        view1[r] = l;
    }
    if (tid == 0) {
        if (reuse_gsum) {
            const double G0 = *cnst + st->gsum_acc;
            st->value = G0;
            st->initial = G0;
        }
        st->gen_state = st->gen_next;
        if (reset_damping) st->damping = 1.0;
        st->epochs_target = epochs;
        st->epochs_run = 0;
        st->retries = 0;
        st->plateaued = 0;
        st->attempts = 0;
        st->status = GLM_OK;
        st->done = 0;
        st->dc = -1;
        st->vw = 0;
        st->block_counter = 0;
        st->epoch_blocks = 0;
    }
}

__global__ void snapshot_kernel(const SolveState *st, double *view0, double *view1, int64_t d,
                                int64_t seq) {
    if (skip_attempt(st, seq)) return;
    const double *src = st->vw ? view1 : view0;
    double *dst = st->vw ? view0 : view1;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = tid; r < d; r += nth) dst[r] = src[r];
}

// Outputs (overwrite or accumulate) + the generator state after the solve.
__global__ void finalize_kernel(SolveState *st, const double *delta0, const double *delta1,
                                const double *view0, const double *view1, const double *lin,
                                double quad, int64_t m, int64_t d, double *delta_out,
                                double *dv_out, int accumulate, int box, int next_known = 0,
                                uint64_t next_state = 0) {
    const int dc = st->dc;
    const double *dl = dc < 0 ? nullptr : (dc ? delta1 : delta0);
    const double *V = st->vw ? view1 : view0;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    if (delta_out) {
        if (accumulate) {
            // folding into alpha: a coordinate clipped to a bound of the SVM box
            // lands there up to the rounding of base + delta (the reference can
            // step an ulp outside and then fails its own check_alpha,
            // objectives.py:110-112); keep the folded alpha in the box
            if (dl && box)
                for (int64_t j = tid; j < m; j += nth)
                    delta_out[j] = fmin(1.0, fmax(0.0, delta_out[j] + dl[j]));
            else if (dl)
                for (int64_t j = tid; j < m; j += nth) delta_out[j] += dl[j];
        } else {
            for (int64_t j = tid; j < m; j += nth) delta_out[j] = dl ? dl[j] : 0.0;
        }
    }
    if (dv_out) {
        if (accumulate)
            for (int64_t r = tid; r < d; r += nth) dv_out[r] += (V[r] - lin[r]) / quad;
        else
            for (int64_t r = tid; r < d; r += nth) dv_out[r] = (V[r] - lin[r]) / quad;
    }
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        const uint64_t g = next_known ? next_state
                                      : warp_jump(st->gen_state, (uint64_t)st->attempts * (uint64_t)m);
        if (threadIdx.x == 0) st->gen_next = g;
    }
}

__global__ void empty_solve_kernel(SolveState *st) {
    for (int i = 0; i < st->epochs_target && i < MAX_EPOCH_VALUES; ++i)
        st->epoch_values[i] = st->value;
    st->epochs_run = st->epochs_target;
    st->done = 1;
}

__global__ void empty_chunk_kernel(SolveState *st, int64_t seq) {
    if (st->seq != seq || st->done) return;
    st->epochs_run = 1;
    st->done = 1;
}

__global__ void set_state_kernel(SolveState *st, uint64_t gen, double damping) {
    st->gen_next = gen;
    st->damping = damping;
    st->block_counter = 0;
    st->done = 1;
}

// ------------------------------------------------------------- launchers
static int grid_stride_blocks(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b < 1) b = 1;
    if (b > 8 * NUM_SMS) b = 8 * NUM_SMS;
    return (int)b;
}

template <int G, int R, bool DENSE, int CM>
static int launch_async_t(const EpochParams &p, int max_inflight, cudaStream_t s) {
    // identical for every B200; atomic because the reference calls the
    // device solve from one thread per device (engine.py:259-263)
    static std::atomic<int> occ{0};
    int blocks_per_sm = occ.load(std::memory_order_relaxed);
    if (!blocks_per_sm) {
        GLM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &blocks_per_sm, scd_async<G, R, DENSE, CM>, 256, 0));
        if (blocks_per_sm < 1) blocks_per_sm = 1;
        occ.store(blocks_per_sm, std::memory_order_relaxed);
    }
    // Staleness control: at most max_inflight coordinates in flight (default
    // n/32, i.e. ~3% of the partition) — the GPU analogue of the reference's
    // thread count (solver.py:213-239).  Large partitions fill the GPU.
    int64_t groups = max_inflight;
    if (groups <= 0) {   // feature-conflict budget: ~16 * d / nnz coordinates in flight
        const double avg = DENSE ? (double)p.d : (double)p.nnz / (double)(p.m > 0 ? p.m : 1);
        groups = (int64_t)(16.0 * (double)p.d / (avg > 1.0 ? avg : 1.0));
        if (groups < 32) groups = 32;
    }
    if (groups > p.m) groups = p.m;
    if (groups < 32 / G) groups = 32 / G;
    const int64_t need_blocks = (groups * G + 255) / 256;
    int64_t cap = (int64_t)blocks_per_sm * NUM_SMS;
    if (cap < NUM_SMS) cap = NUM_SMS;
    if (cap > EPOCH_PARTIALS) cap = EPOCH_PARTIALS;
    const int grid = (int)(need_blocks < cap ? (need_blocks < 1 ? 1 : need_blocks) : cap);
    count_launch();
    GLM_CUDA_TRY(launch_pdl(p.pdl != 0, scd_async<G, R, DENSE, CM>, dim3(grid), dim3(256), 0, s,
                            p));
    return GLM_OK;
}

// lanes = G | (R << 8): G lanes per coordinate holding R column elements
// each in registers (R = 0: the default for G)
template <bool DENSE, int CM>
static int launch_async_cm(const EpochParams &p, int lanes, int max_inflight, cudaStream_t s) {
    const int G = lanes & 0xff, R = lanes >> 8;
    switch (G) {
    case 4:
        if (R >= 10) return launch_async_t<4, 10, DENSE, CM>(p, max_inflight, s);
        return launch_async_t<4, 4, DENSE, CM>(p, max_inflight, s);
    case 8:
        if (R > 0 && R <= 5) return launch_async_t<8, 5, DENSE, CM>(p, max_inflight, s);
        return launch_async_t<8, 8, DENSE, CM>(p, max_inflight, s);
    case 16: return launch_async_t<16, 4, DENSE, CM>(p, max_inflight, s);
    default: return launch_async_t<32, 4, DENSE, CM>(p, max_inflight, s);
    }
}

template <bool DENSE>
static int launch_async(const EpochParams &p, int lanes, int max_inflight, int flags,
                        cudaStream_t s) {
    if (!DENSE && p.meta) {          // a prepared partition: packed records
        switch (flags & 3) {
        case 1: return launch_async_cm<DENSE, 5>(p, lanes, max_inflight, s);
        case 2: return launch_async_cm<DENSE, 6>(p, lanes, max_inflight, s);
        case 3: return launch_async_cm<DENSE, 7>(p, lanes, max_inflight, s);
        default: return launch_async_cm<DENSE, 4>(p, lanes, max_inflight, s);
        }
    }
    switch (flags & 3) {
    case 1: return launch_async_cm<DENSE, 1>(p, lanes, max_inflight, s);
    case 2: return launch_async_cm<DENSE, 2>(p, lanes, max_inflight, s);
    case 3: return launch_async_cm<DENSE, 3>(p, lanes, max_inflight, s);
    default: return launch_async_cm<DENSE, 0>(p, lanes, max_inflight, s);
    }
}

__global__ void meta_build_kernel(const int64_t *indptr, const double *sq, int64_t m,
                                  longlong2 *meta) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = indptr[j], cnt = indptr[j + 1] - lo;
        const bool fits = cnt < META_CNT_SENTINEL && lo >= 0 && lo < (1LL << 40);
        longlong2 r;
        r.x = fits ? (lo | (cnt << 40)) : (META_CNT_SENTINEL << 40);
        r.y = __double_as_longlong(sq[j]);
        meta[j] = r;
    }
}


// Narrow dense launch: R = rows per lane.  The async grid follows the
// in-flight budget: warps x per_phase x CTAs <= budget (budget 0 = auto:
// 32 * d / nnz-per-column / (quad * mean |a|^2), the coupling-scaled
// feature-conflict budget; at least one warp per SM).
static int narrow_rows(int64_t d) {
    if (d <= 32) return 1;
    if (d <= 64) return 2;
    if (d <= 128) return 4;
    if (d <= 256) return 8;
    if (d <= 512) return 16;      // C1 dual: 500 rows, 16 registers per lane
    if (d <= NARROW_MAX_ROWS) return 32;
    return 0;
}

template <int R>
static int launch_narrow_t(const EpochParams &p, bool async, int64_t budget, double *vpad,
                           cudaStream_t s) {
    count_launch();
    if (!async) {
        scd_seq_narrow<R><<<1, 32, 0, s>>>(p);
        GLM_CUDA_TRY(cudaGetLastError());
        return GLM_OK;
    }
    static std::atomic<int> occ{0};
    int blocks_per_sm = occ.load(std::memory_order_relaxed);
    if (!blocks_per_sm) {
        GLM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm,
                                                                   scd_replica<R>, 256, 0));
        if (blocks_per_sm < 1) blocks_per_sm = 1;
        occ.store(blocks_per_sm, std::memory_order_relaxed);
    }
    constexpr int W = 8;
    int64_t cap = (int64_t)blocks_per_sm * NUM_SMS;
    if (cap > EPOCH_PARTIALS) cap = EPOCH_PARTIALS;
    int64_t grid = budget / W;
    if (grid < 1) grid = 1;
    if (grid > cap) grid = cap;
    const int64_t need = (p.m + W - 1) / W;      // at least one coordinate per warp
    if (grid > need) grid = need < 1 ? 1 : need;
    int64_t per = budget / (grid * W);
    if (per < 1) per = 1;
    if (per > 64) per = 64;
    narrow_pad_kernel<<<1, 256, 0, s>>>(p.st, p.view0, p.view1, vpad, p.d, p.seq);
    count_launch();
    scd_replica<R><<<(int)grid, 32 * W, 0, s>>>(p, (int)per, vpad);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

static int launch_narrow(const EpochParams &p, bool async, int64_t budget, double *vpad,
                         cudaStream_t s) {
    switch (narrow_rows(p.d)) {
    case 1: return launch_narrow_t<1>(p, async, budget, vpad, s);
    case 2: return launch_narrow_t<2>(p, async, budget, vpad, s);
    case 4: return launch_narrow_t<4>(p, async, budget, vpad, s);
    case 8: return launch_narrow_t<8>(p, async, budget, vpad, s);
    case 16: return launch_narrow_t<16>(p, async, budget, vpad, s);
    default: return launch_narrow_t<32>(p, async, budget, vpad, s);
    }
}

__global__ void mean_kernel(const double *x, int64_t n, double *out) {
    __shared__ double sm[32];
    double acc[1] = {0.0};
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc[0] += x[i];
    block_sum<1>(acc, sm);
    if (threadIdx.x == 0) out[0] = n > 0 ? acc[0] / (double)n : 1.0;
}

// mean |a_j|^2 of a partition (cached per sqnorm array; one sync the first time)
static int mean_sqnorm(glm_solver *s, const double *sq, int64_t m, cudaStream_t stream,
                       double *out) {
    if (s->sq_src == sq && s->sq_n == m) {
        *out = s->sq_mean;
        return GLM_OK;
    }
    count_launch();
    mean_kernel<<<1, 1024, 0, stream>>>(sq, m, s->scratch);
    GLM_CUDA_TRY(cudaGetLastError());
    double h = 1.0;
    GLM_CUDA_TRY(cudaMemcpyAsync(&h, s->scratch, sizeof(double), cudaMemcpyDeviceToHost, stream));
    GLM_CUDA_TRY(cudaStreamSynchronize(stream));
    s->sq_src = sq;
    s->sq_n = m;
    s->sq_mean = h > 0.0 ? h : 1.0;
    *out = s->sq_mean;
    return GLM_OK;
}

static int64_t narrow_budget(const EpochParams &p, double sq_mean, int max_inflight) {
    if (max_inflight > 0) return max_inflight;
    const double c = p.quad * sq_mean;
    double b = 32.0 / (c > 1e-300 ? c : 1e-300);
    if (b < 32.0) b = 32.0;
    if (b > 1e9) b = 1e9;
    return (int64_t)b;
}

constexpr int64_t SMEM_VIEW_MAX = 24 * 1024;   // doubles (192 KB)

// GLM_SEQ_KERNEL=csc keeps the one-warp walk (A/B checks of the level-
// scheduled kernel, which must produce the same bits)
static bool seq_csc_forced() {
    const char *e = getenv("GLM_SEQ_KERNEL");
    return e && strcmp(e, "csc") == 0;
}

template <int BS, bool DENSE>
static int launch_seq_t(const EpochParams &p, cudaStream_t s) {
    if (BS == 32 && !DENSE && p.d <= LVL_TAB_MAX && !seq_csc_forced()) {
        static std::atomic<int> dbg_set{-1};
        if (dbg_set.load(std::memory_order_relaxed) < 0) {
            const char *e = getenv("GLM_LVL_DEBUG");
            int dbg = e && e[0] == '1';
            if (dbg) GLM_CUDA_TRY(cudaMemcpyToSymbol(lvl_debug, &dbg, sizeof(int)));
            dbg_set.store(dbg, std::memory_order_relaxed);
        }
        const bool sv = p.d <= LVL_SMEM_VIEW_MAX;
        const size_t tab = (size_t)((p.d + 16) & ~15LL);
        const size_t bytes =
            LVL_STAGE_BYTES + tab + (sv ? sizeof(double) * (size_t)((p.d + 1) & ~1LL) : 0);
        count_launch();
        if (sv) {
            GLM_CUDA_TRY(cudaFuncSetAttribute(scd_seq_lvl<true>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)bytes));
            scd_seq_lvl<true><<<1, LVL_THREADS, bytes, s>>>(p);
        } else {
            GLM_CUDA_TRY(cudaFuncSetAttribute(scd_seq_lvl<false>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)bytes));
            scd_seq_lvl<false><<<1, LVL_THREADS, bytes, s>>>(p);
        }
        GLM_CUDA_TRY(cudaGetLastError());
        return GLM_OK;
    }
    if (BS == 32 && !DENSE) {   // short CSC columns: the pipelined one-warp kernel
        if (p.d <= SMEM_VIEW_MAX) {
            size_t bytes = sizeof(double) * (size_t)(p.d > 0 ? p.d : 1);
            GLM_CUDA_TRY(cudaFuncSetAttribute(scd_seq_csc<3, true>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)(SMEM_VIEW_MAX * sizeof(double))));
            count_launch();
            scd_seq_csc<3, true><<<1, 32, bytes, s>>>(p);
        } else {
            count_launch();
            scd_seq_csc<3, false><<<1, 32, 0, s>>>(p);
        }
        GLM_CUDA_TRY(cudaGetLastError());
        return GLM_OK;
    }
    if (p.d <= SMEM_VIEW_MAX) {
        size_t bytes = sizeof(double) * (size_t)(p.d > 0 ? p.d : 1);
        GLM_CUDA_TRY(cudaFuncSetAttribute(scd_seq<BS, true, DENSE>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(SMEM_VIEW_MAX * sizeof(double))));
        count_launch();
        scd_seq<BS, true, DENSE><<<1, BS, bytes, s>>>(p);
    } else {
        count_launch();
        scd_seq<BS, false, DENSE><<<1, BS, 0, s>>>(p);
    }
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

static int auto_lanes(double avg_nnz, bool dense, int64_t d) {   // lanes x registers cover the column
    if (avg_nnz <= 16) return 4;
    if (avg_nnz <= 40) return 4 | (10 << 8);   // C2 / C5: 4 lanes x 10 registers (tools/sweep_c2.py)
    if (avg_nnz <= 64) return 8;
    // sparse columns of a few hundred rows into an L2-resident view: more
    // coordinates in flight beat more lanes per coordinate (C2 primal, 400 nnz
    // per feature into a 1M-row view: 32 lanes 0.63-0.67 ms, 16 x 4 0.55-0.56,
    // 8 x 5 0.53 per epoch); a view beyond L2 wants 32 lanes (C4, 10M rows:
    // 32 lanes 5.03 ms, 16 x 4 5.21; tools/gpu_c2p2.sh)
    if (!dense && avg_nnz <= 1024 && d <= ((int64_t)1 << 22)) return 8 | (5 << 8);
    return 32;
}

// Timing events: inside a CUDA-graph capture they become event-record nodes
// that timestamp every replay (cudaEventRecordExternal).
static cudaError_t event_record(cudaEvent_t ev, cudaStream_t stream) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaError_t e = cudaStreamIsCapturing(stream, &cs);
    if (e != cudaSuccess) return e;
    if (cs == cudaStreamCaptureStatusActive)
        return cudaEventRecordWithFlags(ev, stream, cudaEventRecordExternal);
    return cudaEventRecord(ev, stream);
}

int glue_begin(glm_solver *s, int kind, cudaStream_t stream) {
    std::array<cudaEvent_t, 2> ev{};
    if (!s->glue_pool.empty()) {
        ev = s->glue_pool.back();
        s->glue_pool.pop_back();
    } else {
        for (int i = 0; i < 2; ++i) GLM_CUDA_TRY(cudaEventCreate(&ev[i]));
    }
    GLM_CUDA_TRY(event_record(ev[0], stream));
    s->glue_events.push_back({kind, ev});
    return GLM_OK;
}

int glue_end(glm_solver *s, cudaStream_t stream) {
    GLM_CUDA_TRY(event_record(s->glue_events.back().second[1], stream));
    return GLM_OK;
}

// The prefetch branch (side stream) must rejoin `stream` before the solver's
// scratch is reused or a graph capture ends.
// A join retires the prefetch: its event may have been recorded inside a graph
// capture and must not be waited on again outside it.
int join_prefetch(glm_solver *s, cudaStream_t stream) {
    if (s->prefetched) GLM_CUDA_TRY(cudaStreamWaitEvent(stream, s->ev_join, 0));
    s->prefetched = false;
    return GLM_OK;
}

static int ensure_side_stream(glm_solver *s) {
    if (!s->side) {
        // the permutation prefetch runs at the lowest priority so the
        // caller's round kernels (epoch, turn) get free SMs first
        int lo = 0, hi = 0;
        GLM_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        GLM_CUDA_TRY(cudaStreamCreateWithPriority(&s->side, cudaStreamNonBlocking, lo));
        GLM_CUDA_TRY(cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming));
        GLM_CUDA_TRY(cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming));
    }
    return GLM_OK;
}

int prefetch_first_perm(glm_solver *s, int64_t m, cudaStream_t stream) {
    if (!s->host_known || m <= 0 || m > s->max_coords || s->prefetched) return GLM_OK;
    int rc = ensure_device_tables();
    if (rc || (rc = ensure_side_stream(s))) return rc;
    GLM_CUDA_TRY(cudaEventRecord(s->ev_fork, stream));
    GLM_CUDA_TRY(cudaStreamWaitEvent(s->side, s->ev_fork, 0));
    const PermScratch ps = carve_perm_scratch(s->perm_mem, s->max_coords, m);
    int32_t *P = s->perm_cur ? s->perm_b : s->perm;
    if ((rc = stream_perm(nullptr, s->host_gen, 0, m, P, ps, s->side))) return rc;
    GLM_CUDA_TRY(cudaEventRecord(s->ev_join, s->side));
    s->prefetched = true;
    s->prefetch_m = m;
    s->prefetch_alt = false;
    return GLM_OK;
}

int set_state(glm_solver *s, uint64_t gen_state, double damping, cudaStream_t stream) {
    int rc = join_prefetch(s, stream);
    if (rc) return rc;
    s->prefetched = false;               // the stream state changes
    s->host_known = true;
    s->host_gen = gen_state ? gen_state : 0x9E3779B97F4A7C15ULL;
    count_launch();
    set_state_kernel<<<1, 1, 0, stream>>>(s->st, gen_state ? gen_state : 0x9E3779B97F4A7C15ULL,
                                          damping);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

int read_result(glm_solver *s, glm_solve_result *res, double *epoch_values, int cap,
                cudaStream_t stream) {
    GLM_CUDA_TRY(cudaMemcpyAsync(s->st_host, s->st, sizeof(SolveState), cudaMemcpyDeviceToHost,
                                 stream));
    GLM_CUDA_TRY(cudaStreamSynchronize(stream));
    fill_result(s, res, epoch_values, cap);
    return GLM_OK;
}

void fill_result(const glm_solver *s, glm_solve_result *res, double *epoch_values, int cap) {
    const SolveState &h = *s->st_host;
    if (res) {
        res->status = h.status;
        res->epochs_run = h.epochs_run;
        res->retries = h.retries;
        res->plateaued = h.plateaued;
        res->attempts = h.attempts;
        res->done = h.done;
        res->damping = h.damping;
        res->initial_value = h.initial;
        res->final_value = h.value;
        res->gen_state = h.gen_next;
    }
    if (epoch_values) {
        int n = h.epochs_run < cap ? h.epochs_run : cap;
        n = n < MAX_EPOCH_VALUES ? n : MAX_EPOCH_VALUES;
        for (int i = 0; i < n; ++i) epoch_values[i] = h.epoch_values[i];
    }
}

int solve(glm_solver *s, const glm_matrix *A, const glm_solve_args *a, double *delta_out,
          double *dv_out, glm_solve_result *res, cudaStream_t stream, const HostCopies *hc) {
    if (!A || !a) return glm_set_error(GLM_USAGE, "null matrix or args");
    if (a->epochs < 1) return glm_set_error(GLM_USAGE, "t_epochs must be >= 1");
    const int64_t m = A->n_cols, d = A->n_rows;
    if (m > s->max_coords || d > s->max_rows)
        return glm_set_error(GLM_USAGE, "partition larger than the solver was created for");
    if (m >= (1LL << 31)) return glm_set_error(GLM_USAGE, "partition exceeds 2^31 coordinates");
    if (a->kind < 0 || a->kind > GLM_HINGE_PRIMAL)
        return glm_set_error(GLM_USAGE, "unknown objective kind");
    if (!(a->quad > 0.0)) return glm_set_error(GLM_USAGE, "quad must be positive");
    if (a->kind == GLM_DUAL_RIDGE && !a->coord_target)
        return glm_set_error(GLM_USAGE, "dual_ridge needs per-coordinate targets");
    int rc = ensure_device_tables();
    if (rc) return rc;
    const bool dense = A->layout == GLM_DENSE;

    EpochParams ep;
    ep.st = s->st;
    ep.kind = a->kind;
    ep.lam = a->lam;
    ep.rho = a->l1_ratio;
    ep.quad = a->quad;
    ep.m = m;
    ep.d = d;
    ep.indptr = A->indptr;
    ep.rows = A->rows;
    ep.vals = A->vals;
    ep.sq = A->sqnorms;
    // packed records when this partition was prepared (glm_solver_prepare)
    ep.meta = (!dense && s->meta && s->meta_indptr == A->indptr && s->meta_sq == A->sqnorms &&
               s->meta_m == m) ? s->meta : nullptr;
    ep.base = a->base;
    ep.y = a->coord_target;
    ep.delta0 = s->delta[0];
    ep.delta1 = s->delta[1];
    ep.view0 = s->view[0];
    ep.view1 = s->view[1];
    ep.perm = s->perm;
    ep.gpart = s->gpart;
    ep.nnz = A->nnz;
    ep.seq = -1;

    ValueParams vp{};
    vp.st = s->st;
    vp.kind = a->kind;
    vp.lam = a->lam;
    vp.rho = a->l1_ratio;
    vp.quad = a->quad;
    vp.cnst = a->cnst;
    vp.m = m;
    vp.d = d;
    vp.lin = a->lin;
    vp.base = a->base;
    vp.y = a->coord_target;
    vp.view0 = s->view[0];
    vp.view1 = s->view[1];
    vp.partials = s->partials;
    vp.gpart = s->gpart;
    vp.seq = -1;

    const double avg = dense ? (double)d : (m > 0 ? (double)A->nnz / (double)m : 0.0);
    const int lanes = a->group_lanes > 0 ? a->group_lanes : auto_lanes(avg, dense, d);
    const int seq_bs = avg <= 96.0 ? 32 : 256;
    // the per-attempt value pass over the view: ~4 rows per thread keeps the
    // block partials (and the last block's fold) short
    auto value_grid_view = [](int64_t n) {
        int64_t b = (n + 4 * VALUE_THREADS - 1) / (4 * VALUE_THREADS);
        if (b < 1) b = 1;
        if (b > 2 * NUM_SMS) b = 2 * NUM_SMS;
        return (int)b;
    };
    auto value_grid = [](int64_t n) {
        int64_t b = (n + VALUE_THREADS - 1) / VALUE_THREADS;
        if (b < 1) b = 1;
        if (b > VALUE_MAX_BLOCKS) b = VALUE_MAX_BLOCKS;
        return (int)b;
    };

    const bool narrow = dense && narrow_rows(d) > 0;
    int64_t nbudget = 0;
    if (narrow && a->mode != GLM_MODE_SEQUENTIAL && m > 0) {
        double sqm = 1.0;
        if ((rc = mean_sqnorm(s, A->sqnorms, m, stream, &sqm))) return rc;
        nbudget = narrow_budget(ep, sqm, a->max_inflight);
    }
    const int reuse = (a->flags & GLM_FLAG_REUSE_GSUM) ? 1 : 0;
    // GLM_FLAG_SKIP_BEGIN: glm_round_start already reset the state, wrote the
    // views and took G(0) from the cached g-sum (peer.cu)
    const bool skip_begin = (a->flags & GLM_FLAG_SKIP_BEGIN) && reuse;
    if (!skip_begin) {
        count_launch();
        begin_kernel<<<grid_stride_blocks(d), 256, 0, stream>>>(s->st, s->view[0], s->view[1],
                                                                a->lin, d, a->epochs,
                                                                a->reset_damping, a->cnst, reuse);
    }
    if (!reuse) {
        vp.mode = 0;
        count_launch();
        value_kernel<<<value_grid(m), VALUE_THREADS, 0, stream>>>(vp);
        GLM_CUDA_TRY(cudaGetLastError());
    }
    vp.mode = 1;

    const PermScratch ps = carve_perm_scratch(s->perm_mem, s->max_coords, m);
    // a permutation prefetched by the previous solve (GLM_FLAG_PREFETCH_PERM)
    // is this solve's attempt 0 when it was generated for the same m
    bool have_perm0 = false;
    if (s->prefetched) {
        GLM_CUDA_TRY(cudaStreamWaitEvent(stream, s->ev_join, 0));
        have_perm0 = s->prefetch_m == m;
        if (have_perm0 && s->prefetch_alt) s->perm_cur ^= 1;
        s->prefetched = false;
    }
    int32_t *P = s->perm_cur ? s->perm_b : s->perm;
    int32_t *P_alt = s->perm_cur ? s->perm : s->perm_b;
    ep.perm = P;
    // Early prefetch: with one attempt per solve the generator advances by
    // exactly m keys, so the host knows the next solve's start state and its
    // permutation can be generated on the side stream into the other buffer
    // while this solve's epoch runs (overlapping value / finalize / the round
    // start instead of sitting between them and the next epoch).
    static const int fork_mode = [] {        // experiments: 0 before / 1 after the epoch, 2 off
        const char *e = getenv("GLM_PERM_FORK");
        return e ? e[0] - '0' : 0;
    }();
    const bool early = (a->flags & GLM_FLAG_PREFETCH_PERM) && s->host_known &&
                       a->max_attempts == 1 && a->epochs == 1 && m > 0 && fork_mode != 2;
    // GLM_FLAG_TURN: one attempt, and glm_round_turn follows on this stream
    const bool turn = (a->flags & GLM_FLAG_TURN) && a->max_attempts == 1 && a->epochs == 1 &&
                      m > 0;
    ep.pdl = turn ? 1 + epoch_early_trigger(s) : 0;   // follows the previous round's turn
    const uint64_t next_state = early ? host_jump(s->host_gen, (uint64_t)m) : 0;
    auto ensure_side = [&]() -> int { return ensure_side_stream(s); };
    int launched = 0;
    auto attempt = [&]() -> int {
        // optional CUDA-event bracket: [perm | snapshot+epoch | value]
        std::array<cudaEvent_t, 4> ev{};
        if (s->timing) {
            if (!s->event_pool.empty()) {
                ev = s->event_pool.back();
                s->event_pool.pop_back();
            } else {
                for (int i = 0; i < 4; ++i) GLM_CUDA_TRY(cudaEventCreate(&ev[i]));
            }
            GLM_CUDA_TRY(event_record(ev[0], stream));
        }
        int r = GLM_OK;
        if (!(launched == 0 && have_perm0))
            r = stream_perm(s->st, 0, (uint64_t)launched * (uint64_t)m, m, P, ps, stream);
        if (r) return r;
        auto fork = [&]() -> int {
            if ((r = ensure_side())) return r;
            GLM_CUDA_TRY(cudaEventRecord(s->ev_fork, stream));
            GLM_CUDA_TRY(cudaStreamWaitEvent(s->side, s->ev_fork, 0));
            if ((r = stream_perm(nullptr, next_state, 0, m, P_alt, ps, s->side))) return r;
            GLM_CUDA_TRY(cudaEventRecord(s->ev_join, s->side));
            s->prefetched = true;
            s->prefetch_m = m;
            s->prefetch_alt = true;
            return GLM_OK;
        };
        if (early && launched == 0 && fork_mode == 0 && (r = fork())) return r;
        if (s->timing) GLM_CUDA_TRY(event_record(ev[1], stream));
        if (launched > 0) {   // attempt 0's snapshot was written by begin_kernel
            count_launch();
            snapshot_kernel<<<grid_stride_blocks(d), 256, 0, stream>>>(s->st, s->view[0],
                                                                       s->view[1], d, -1);
        }
        if (narrow) {
            r = launch_narrow(ep, a->mode != GLM_MODE_SEQUENTIAL, nbudget, s->vpad, stream);
        } else if (a->mode == GLM_MODE_SEQUENTIAL) {
            if (dense) r = seq_bs == 32 ? launch_seq_t<32, true>(ep, stream) : launch_seq_t<256, true>(ep, stream);
            else r = seq_bs == 32 ? launch_seq_t<32, false>(ep, stream) : launch_seq_t<256, false>(ep, stream);
        } else {
            r = dense ? launch_async<true>(ep, lanes, a->max_inflight, a->flags, stream)
                      : launch_async<false>(ep, lanes, a->max_inflight, a->flags, stream);
        }
        if (r) return r;
        if (early && launched == 0 && fork_mode == 1 && (r = fork())) return r;
        if (s->timing) GLM_CUDA_TRY(event_record(ev[2], stream));
        if (!turn) {          // GLM_FLAG_TURN: glm_round_turn takes the value
            count_launch();
            value_kernel<<<value_grid_view(d), VALUE_THREADS, 0, stream>>>(vp);
            GLM_CUDA_TRY(cudaGetLastError());
        }
        if (s->timing) {
            GLM_CUDA_TRY(event_record(ev[3], stream));
            s->events.push_back(ev);
        }
        ++launched;
        return GLM_OK;
    };

    const bool peer_fin = (a->flags & GLM_FLAG_PEER_FINALIZE) && a->peer && a->accumulate &&
                          delta_out;
    auto plain_finalize = [&]() -> int {
        count_launch();
        finalize_kernel<<<grid_stride_blocks(m > d ? m : d), 256, 0, stream>>>(
            s->st, s->delta[0], s->delta[1], s->view[0], s->view[1], a->lin, a->quad, m, d,
            delta_out, dv_out, a->accumulate, a->kind == GLM_DUAL_L2_SVM ? 1 : 0, early ? 1 : 0,
            next_state);
        GLM_CUDA_TRY(cudaGetLastError());
        return GLM_OK;
    };
    // outputs enqueued before the adaptive loop's synchronisation (see HostCopies)
    const bool spec = hc && !turn && !peer_fin && !a->accumulate && !s->timing && m > 0;
    auto copies = [&]() -> int {
        if (hc->delta && delta_out)
            GLM_CUDA_TRY(cudaMemcpyAsync(hc->delta, delta_out, sizeof(double) * m,
                                         cudaMemcpyDeviceToHost, stream));
        if (hc->dv && dv_out && d > 0)
            GLM_CUDA_TRY(cudaMemcpyAsync(hc->dv, dv_out, sizeof(double) * d,
                                         cudaMemcpyDeviceToHost, stream));
        return GLM_OK;
    };
    bool finalized = false;
    if (m > 0) {
        if (a->max_attempts > 0) {
            for (int i = 0; i < a->max_attempts; ++i)
                if ((rc = attempt())) return rc;
        } else {
            int batch = a->epochs;
            for (;;) {
                for (int i = 0; i < batch; ++i)
                    if ((rc = attempt())) return rc;
                if (spec && ((rc = plain_finalize()) || (rc = copies()))) return rc;
                glm_solve_result r;
                if ((rc = read_result(s, &r, nullptr, 0, stream))) return rc;
                if (r.done) {
                    finalized = spec;
                    break;
                }
                batch = a->epochs - r.epochs_run;
                if (batch < 1) batch = 1;
            }
        }
    } else {
        // no coordinates: the reference still runs `epochs` empty passes whose
        // value never changes (permute(0) consumes no keys, solver.py:86-88)
        count_launch();
        empty_solve_kernel<<<1, 1, 0, stream>>>(s->st);
    }
    if (turn || finalized) {
        // turn: value, finalize and the exchange run in glm_round_turn;
        // finalized: the speculative finalize + copies were the last ones
    } else if (s->timing && (rc = glue_begin(s, 0, stream))) {
        return rc;
    } else if (peer_fin) {
        // Delta v goes to this rank's peer-exchange buffer (peer.cu)
        rc = peer_finalize(s, a->peer, a->lin, a->quad, m, d, delta_out,
                           a->kind == GLM_DUAL_L2_SVM ? 1 : 0, early ? 1 : 0, next_state, stream);
        if (rc) return rc;
    } else {
        if ((rc = plain_finalize())) return rc;
        if (hc && (rc = copies())) return rc;
    }
    if (!turn && !finalized && s->timing && (rc = glue_end(s, stream))) return rc;
    s->last_epochs = a->epochs;
    s->last_m = m;
    if (early) {
        s->host_gen = next_state;
    } else {
        s->host_known = false;
        if ((a->flags & GLM_FLAG_PREFETCH_PERM) && m > 0 && fork_mode != 2) {
            // generate the next solve's attempt-0 permutation from gen_next while
            // the caller runs its fold / all-reduce / round-start kernels
            if ((rc = ensure_side())) return rc;
            GLM_CUDA_TRY(cudaEventRecord(s->ev_fork, stream));
            GLM_CUDA_TRY(cudaStreamWaitEvent(s->side, s->ev_fork, 0));
            rc = stream_perm_from(&s->st->gen_next, m, P, ps, s->side);
            if (rc) return rc;
            GLM_CUDA_TRY(cudaEventRecord(s->ev_join, s->side));
            s->prefetched = true;
            s->prefetch_m = m;
            s->prefetch_alt = false;
        }
    }
    if (res) {
        if (finalized) {                      // the loop's copy of the state is final
            fill_result(s, res, nullptr, 0);
            return GLM_OK;
        }
        return read_result(s, res, nullptr, 0, stream);
    }
    return GLM_OK;
}

// ------------------------------------------------- chunked (out-of-core)
// The per-chunk damped pass of the streaming pipeline (_train_chunk,
// pipeline.py:158-193) on the same kernels: chunk `seq` is opened only once
// chunk seq-1 has finished (so the host may enqueue chunk seq+1 before it
// has checked chunk seq), every attempt kernel is guarded by the open
// sequence number, and the close kernel commits the accepted pass into the
// partition-wide delta and reports to host-mapped memory.

__global__ void stream_begin_kernel(SolveState *st, double *view0, double *view1,
                                    const double *lin, int64_t d, double *dfull, int64_t m,
                                    int zero_delta, int keep_view, double damping) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = tid; r < d; r += nth) {
        const double v = keep_view ? view0[r] : lin[r];
        view0[r] = v;
        view1[r] = v;
    }
    if (zero_delta)
        for (int64_t j = tid; j < m; j += nth) dfull[j] = 0.0;
    if (tid == 0) {
        st->damping = damping;
        st->status = GLM_OK;
        st->done = 0;
        st->seq = -1;
        st->dc = 0;
        st->vw = 0;
        st->block_counter = 0;
        st->epoch_blocks = 0;
        st->retries = 0;
        st->attempts = 0;
        st->plateaued = 0;
        st->epochs_run = 0;
        st->epochs_target = 1;
    }
}

__global__ void chunk_open_kernel(SolveState *st, int64_t seq) {
    if (st->status != GLM_OK || st->seq == seq) return;
    if (st->seq != seq - 1 || (seq > 0 && !st->done)) return;   // previous chunk unfinished
    st->seq = seq;
    st->done = 0;
    st->dc = 0;
    st->plateaued = 0;
    st->epochs_run = 0;
    st->epochs_target = 1;
    st->block_counter = 0;
}

__global__ void chunk_close_kernel(SolveState *st, int64_t seq, const double *dwork,
                                   double *dfull, int64_t nc, ChunkRecord *rec) {
    const bool mine = st->seq == seq;
    if (mine && st->done && st->dc == 1) {     // an accepted pass: commit it
        const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        const int64_t nth = (int64_t)gridDim.x * blockDim.x;
        for (int64_t j = tid; j < nc; j += nth) dfull[j] = dwork[j];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        volatile ChunkRecord *r = rec;
        r->cur = st->seq;
        r->done = mine ? st->done : 0;
        r->status = st->status;
        r->retries = st->retries;
        r->attempts = st->attempts;
        r->plateaued = mine ? st->plateaued : 0;
        r->accepted = mine ? st->dc : 0;
        r->damping = st->damping;
        r->value = st->value;
        __threadfence_system();
        r->seq = seq;
        __threadfence_system();
    }
}

int stream_begin(glm_solver *s, const StreamSolve &a, bool zero_delta, bool keep_view,
                 double damping, cudaStream_t stream) {
    int rc = join_prefetch(s, stream);
    if (rc) return rc;
    count_launch();
    stream_begin_kernel<<<grid_stride_blocks(a.d > a.m ? a.d : a.m), 256, 0, stream>>>(
        s->st, s->view[0], s->view[1], a.lin, a.d, a.dfull, a.m, zero_delta ? 1 : 0,
        keep_view ? 1 : 0, damping);
    GLM_CUDA_TRY(cudaGetLastError());
    ValueParams vp{};
    vp.st = s->st;
    vp.mode = 0;
    vp.kind = a.kind;
    vp.lam = a.lam;
    vp.rho = a.rho;
    vp.quad = a.quad;
    vp.cnst = a.cnst;
    vp.m = a.m;
    vp.d = a.d;
    vp.lin = a.lin;
    vp.base = a.base;
    vp.y = a.y;
    vp.dfull = zero_delta ? nullptr : a.dfull;
    vp.view_terms = keep_view ? 1 : 0;
    vp.seq = -1;
    vp.view0 = s->view[0];
    vp.view1 = s->view[1];
    vp.partials = s->partials;
    vp.gpart = s->gpart;
    int64_t n = a.m > a.d ? a.m : a.d;
    int64_t b = (n + VALUE_THREADS - 1) / VALUE_THREADS;
    b = b < 1 ? 1 : (b > VALUE_MAX_BLOCKS ? VALUE_MAX_BLOCKS : b);
    count_launch();
    value_kernel<<<(int)b, VALUE_THREADS, 0, stream>>>(vp);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

int chunk_enqueue(glm_solver *s, const StreamSolve &a, const ChunkJob &c, cudaStream_t stream) {
    const glm_matrix *A = c.A;
    const int64_t nc = A->n_cols, d = A->n_rows;
    if (nc > s->max_coords || d > s->max_rows)
        return glm_set_error(GLM_USAGE, "chunk larger than the stream solver");
    int rc = ensure_device_tables();
    if (rc) return rc;
    if (c.gen_perm && nc > 0) {
        const PermScratch ps = carve_perm_scratch(s->perm_mem, s->max_coords, nc);
        rc = chunk_perm(c.key_seed, nc, c.perm, ps, stream);
        if (rc) return rc;
    }
    if (c.open) {
        count_launch();
        chunk_open_kernel<<<1, 1, 0, stream>>>(s->st, c.seq);
        GLM_CUDA_TRY(cudaGetLastError());
    }
    ValueParams vp{};
    vp.st = s->st;
    vp.kind = a.kind;
    vp.lam = a.lam;
    vp.rho = a.rho;
    vp.quad = a.quad;
    vp.cnst = a.cnst;
    vp.lin = a.lin;
    vp.seq = c.seq;
    vp.view0 = s->view[0];
    vp.view1 = s->view[1];
    vp.partials = s->partials;
    vp.gpart = s->gpart;
    auto grid_of = [](int64_t n) {
        int64_t b = (n + VALUE_THREADS - 1) / VALUE_THREADS;
        return (int)(b < 1 ? 1 : (b > VALUE_MAX_BLOCKS ? VALUE_MAX_BLOCKS : b));
    };
    if (c.open) {   // the chunk's g-sum in the accepted state (mode 2)
        vp.mode = 2;
        vp.m = nc;
        vp.d = 0;
        vp.base = a.base + c.lo;
        vp.y = a.y ? a.y + c.lo : nullptr;
        vp.dfull = a.dfull + c.lo;
        count_launch();
        value_kernel<<<grid_of(nc), VALUE_THREADS, 0, stream>>>(vp);
        GLM_CUDA_TRY(cudaGetLastError());
    }
    EpochParams ep{};
    ep.st = s->st;
    ep.kind = a.kind;
    ep.lam = a.lam;
    ep.rho = a.rho;
    ep.quad = a.quad;
    ep.m = nc;
    ep.d = d;
    ep.indptr = A->indptr;
    ep.rows = A->rows;
    ep.vals = A->vals;
    ep.sq = A->sqnorms;
    ep.meta = nullptr;
    ep.base = a.base + c.lo;
    ep.y = a.y ? a.y + c.lo : nullptr;
    ep.delta0 = a.dfull + c.lo;     // read: the accepted state (st->dc == 0)
    ep.delta1 = s->delta[1];        // written: the attempt
    ep.view0 = s->view[0];
    ep.view1 = s->view[1];
    ep.perm = c.perm;
    ep.gpart = s->gpart;
    ep.nnz = A->nnz;
    ep.seq = c.seq;
    vp.mode = 1;
    vp.chunked = 1;
    vp.m = nc;
    vp.d = d;
    vp.base = nullptr;
    vp.y = nullptr;
    vp.dfull = nullptr;
    const bool dense = A->layout == GLM_DENSE;
    const double avg = dense ? (double)d : (nc > 0 ? (double)A->nnz / (double)nc : 0.0);
    const int lanes = a.group_lanes > 0 ? a.group_lanes : auto_lanes(avg, dense, d);
    for (int i = 0; i < c.attempts && nc > 0; ++i) {
        count_launch();
        snapshot_kernel<<<grid_stride_blocks(d), 256, 0, stream>>>(s->st, s->view[0], s->view[1],
                                                                   d, c.seq);
        if (a.mode == GLM_MODE_SEQUENTIAL) {
            const bool small = avg <= 96.0;
            if (dense) rc = small ? launch_seq_t<32, true>(ep, stream) : launch_seq_t<256, true>(ep, stream);
            else rc = small ? launch_seq_t<32, false>(ep, stream) : launch_seq_t<256, false>(ep, stream);
        } else {
            rc = dense ? launch_async<true>(ep, lanes, a.max_inflight, a.flags, stream)
                       : launch_async<false>(ep, lanes, a.max_inflight, a.flags, stream);
        }
        if (rc) return rc;
        count_launch();
        value_kernel<<<grid_of(d), VALUE_THREADS, 0, stream>>>(vp);
        GLM_CUDA_TRY(cudaGetLastError());
    }
    if (nc == 0 && c.open) {   // an empty chunk is one accepted no-op pass
        count_launch();
        empty_chunk_kernel<<<1, 1, 0, stream>>>(s->st, c.seq);
    }
    count_launch();
    chunk_close_kernel<<<grid_stride_blocks(nc), 256, 0, stream>>>(s->st, c.seq, s->delta[1],
                                                                   a.dfull + c.lo, nc, c.rec);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

int stream_finalize(glm_solver *s, const StreamSolve &a, double *dv_out, cudaStream_t stream) {
    if (!dv_out) return GLM_OK;
    count_launch();
    finalize_kernel<<<grid_stride_blocks(a.d), 256, 0, stream>>>(
        s->st, nullptr, nullptr, s->view[0], s->view[1], a.lin, a.quad, 0, a.d, nullptr, dv_out,
        0, 0);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

}  // namespace glm
