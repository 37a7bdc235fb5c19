// peer.cu — the Delta v exchange of one CoCoA round fused with the next
// round's start, over NVLink peer memory (one process per GPU).
//
// Reference: the round's only collective, allreduce_sum(v_bar) with the
// ascending-rank fold of canonical_sum (engine.py:282, comm.py:41-46, 83-98),
// followed by v += total (engine.py:306) and the next round's outer/inner
// model (engine.py:271-272, 242-250, 148-166) and solve start (solver.py:
// 268-270).  Here:
//
//   finalize (rank r):  alpha += delta; dv_r[b] = B delta; publish: one
//                       system-scope fence, then the flag word (R+1, accept
//                       bits) stored into slot r of every rank's flags
//   round start:        wait until every LOCAL flag slot j >= R (acquire,
//                       system scope; no remote round trip per poll);
//                       v += sum_j dv_j[b] in ascending rank order (the bits of
//                       canonical_sum on every rank); grad = f'(v); lin = grad;
//                       view = lin; f(v); solver state reset (begin)
//
// The turn kernel writes Delta v speculatively while it evaluates the attempt
// and publishes right at the damping decision; the flag word carries whether
// the attempt was accepted (else the true Delta v is exactly zero).
// dv_r lives in rank r's HBM, double-buffered by round parity; every rank
// reads every peer's buffer through cudaIpc-mapped pointers (NVLink/NVSwitch).
// A rank cannot overwrite dv_r[b] (round R+2) before every rank has consumed
// it (round start R+1 precedes its own finalize R+2), so two buffers suffice.
// Round counters live on the device, so CUDA-graph replays stay consistent.
#include "solver.cuh"

#include <cstring>
#include <vector>

struct glm_peer {
    int device = 0, rank = 0, world = 1;
    int64_t d = 0;
    // [ctl: 16 x i64 | flag slots: 24 x i64 | reduced-flag slots: 24 x i64 | pad to
    //  PEER_HEADER B | dv: 2 x pstride doubles | reduced slice sums: 2 x pstride doubles]
    char *mem = nullptr;
    int64_t *ctl = nullptr;       // [0] published rounds, [1] consumed, [2] block counter,
                                  // [3] "every rank published" (turn), [4] their accept
                                  // bits, [5] our last flag word, [6] round-start ticket,
                                  // [7] error word (a wait that timed out), [8] reduce-
                                  // scatter arrivals, [9] "every rank reduced" (turn)
    int64_t *flags = nullptr;     // local slots: flags[j] = rank j's last flag word
    double *dv = nullptr;         // 2 halves of pstride doubles (Delta v[d], padded)
    int64_t pstride = 0;
    double **bufs_dev = nullptr;  // world pointers to each rank's dv (device array)
    double **red_dev = nullptr;   // world pointers to each rank's reduced slice sums
    int64_t *flags2 = nullptr;    // local reduced-flag slots
    int64_t **flags2_dev = nullptr;  // world pointers to each rank's reduced-flag slots
    int rs = 0;                   // turn P3 as reduce-scatter + all-gather
    int64_t **flags_dev = nullptr;  // world pointers to each rank's flag slots
    std::vector<void *> opened;   // cudaIpc-opened peer allocations
    uint64_t *stamps = nullptr;   // glm_peer_stamps: turn phase timestamps (debug)
    uint64_t timeout_ns = 60000000000ull;   // every device-side wait (comm.py:30 DEFAULT_TIMEOUT)
    int turn_blocks = 0;          // co-resident grid of round_turn (occupancy-checked)
    cudaIpcMemHandle_t handle{};
};

namespace glm {

constexpr int PEER_BLOCKS = 2 * NUM_SMS;
constexpr int PEER_THREADS = 256;
constexpr int PEER_MAX_WORLD = 24;      // flag slots per array in the header
constexpr int PEER_HEADER = 512;        // ctl[16] + flags[24] + flags2[24] doubles-aligned
constexpr int PEER_FLAGS = 16, PEER_FLAGS2 = 40;   // i64 offsets of the flag arrays

// doubles per parity half: Delta v[d] padded to 256 B
inline int64_t peer_pstride(int64_t d) { return ((d > 0 ? d : 1) + 1 + 31) / 32 * 32; }

__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t *p) {
    int64_t v;
    asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(int64_t *p, int64_t v) {
    asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Strong store without its own fence: after one fence.sc.sys, a run of these
// forms the release pattern for each (one MEMBAR.SYS instead of one per store).
__device__ __forceinline__ void st_relaxed_sys(int64_t *p, int64_t v) {
    asm volatile("st.relaxed.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Flag word: R << 2 | accept bits; bit (R & 1) says whether round R's Delta v
// is the attempt's (1) or exactly zero (0, a rejected attempt: the view went
// back to the snapshot, which is lin).  Publishing R+1 keeps the bit of R, so
// a peer still reading round R after we moved on sees the right one (we
// cannot reach R+2 before that peer publishes R+1).  ctl[5] keeps our word.
// One thread, after every block's writes were fenced: our slot in every
// rank's flags; the peers then poll their own memory.
__device__ __forceinline__ void publish(int64_t *ctl, int64_t *const *flags, int world,
                                        int rank, int64_t R, int accept,
                                        uint64_t *stamps = nullptr) {
    const int64_t keep = ctl[5] & (int64_t)(1 << ((R & 1) ^ 1));
    const int64_t word = (R << 2) | keep | (int64_t)((accept ? 1 : 0) << (R & 1));
    ctl[0] = R;
    ctl[5] = word;
    if (world > 1) {
        __threadfence_system();
        if (stamps) stamps[5] = gtimer();
        for (int j = 0; j < world; ++j) st_relaxed_sys(flags[j] + rank, word);
        if (stamps) stamps[6] = gtimer();
    } else {
        __threadfence();
        atomicExch(reinterpret_cast<unsigned long long *>(flags[0]), (unsigned long long)word);
    }
}

// Error word ctl[7] (read by glm_peer_error): the first wait that ran past
// the deadline records what it waited for; the kernel then runs to its end
// (a missing rank contributes +0.0) so the host can raise instead of hanging.
enum : int64_t { PEER_ERR_FLAGS = 1, PEER_ERR_GRID = 2 };

__device__ __forceinline__ void peer_fail(int64_t *ctl, int64_t code, int64_t what) {
    atomicCAS(reinterpret_cast<unsigned long long *>(ctl + 7), 0ull,
              (unsigned long long)((code << 32) | (what & 0xffffffff)));
}

// A spin with a %globaltimer deadline: true once `timeout` ns have passed
// since t0 (t0 = 0 starts the clock).
__device__ __forceinline__ bool expired(uint64_t &t0, uint64_t timeout) {
    const uint64_t t = gtimer();
    if (t0 == 0) t0 = t;
    return t - t0 > timeout;
}

// Every local flag slot at round >= R (one thread); returns the ranks'
// accept bits of round R.  A rank that has not published within the deadline
// is recorded in ctl[7] and counted as not accepted (its Delta v is skipped).
__device__ __forceinline__ uint32_t wait_flags(const int64_t *flags, int world, int64_t R,
                                               int64_t *ctl, uint64_t timeout) {
    uint32_t mask = 0;
    uint64_t t0 = 0;
    for (int j = 0; j < world; ++j) {
        int64_t f;
        bool late = false;
        while (((f = ld_acquire_sys(flags + j)) >> 2) < R) {
            __nanosleep(32);
            if (expired(t0, timeout)) {
                peer_fail(ctl, PEER_ERR_FLAGS, j);
                late = true;
                break;
            }
        }
        if (!late) mask |= (uint32_t)((f >> (R & 1)) & 1) << j;
    }
    return mask;
}

// Every local reduced-flag slot at round >= R (one thread), with the deadline.
__device__ __forceinline__ void wait_rounds(const int64_t *flags, int world, int64_t R,
                                            int64_t *ctl, uint64_t timeout) {
    uint64_t t0 = 0;
    for (int j = 0; j < world; ++j)
        while (ld_acquire_sys(flags + j) < R) {
            __nanosleep(32);
            if (expired(t0, timeout)) {
                peer_fail(ctl, PEER_ERR_FLAGS, j);
                break;
            }
        }
}

// Finalize of a solve whose Delta v goes to the peer exchange: alpha += delta
// (kept in the SVM box), dv_r[(R+1)&1] = (view - lin)/quad, the generator
// jump, and — once every block is done — flag_r = R+1.
__global__ void __launch_bounds__(PEER_THREADS) peer_finalize_kernel(
    SolveState *st, const double *delta0, const double *delta1, const double *view0,
    const double *view1, const double *lin, double quad, int64_t m, int64_t d, double *alpha,
    int box, double *dv, int64_t pstride, int64_t *ctl, int64_t *const *flags, int world,
    int rank, int next_known, uint64_t next_state) {
    __shared__ int s_last;
    const int dc = st->dc;
    const double *dl = dc < 0 ? nullptr : (dc ? delta1 : delta0);
    const double *V = st->vw ? view1 : view0;
    const int64_t R = ctl[0];
    double *out = dv + ((R + 1) & 1) * pstride;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    if (dl) {
        if (box)
            for (int64_t j = tid; j < m; j += nth) alpha[j] = fmin(1.0, fmax(0.0, alpha[j] + dl[j]));
        else
            for (int64_t j = tid; j < m; j += nth) alpha[j] += dl[j];
    }
    for (int64_t r = tid; r < d; r += nth) out[r] = (V[r] - lin[r]) / quad;
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        // the host knows the next state when every solve runs exactly one
        // attempt; else jump by the attempts this solve consumed
        const uint64_t g = next_known ? next_state
                                      : warp_jump(st->gen_state, (uint64_t)st->attempts * (uint64_t)m);
        if (threadIdx.x == 0) st->gen_next = g;
    }
    __syncthreads();
    if (threadIdx.x == 0) {     // the block's writes (observed through the barrier)
        __threadfence();        // before its arrival (GPU scope: peers read this
                                // memory through this GPU's L2); the last block
                                // then releases at system scope, cumulatively
        s_last = atomicAdd(reinterpret_cast<unsigned long long *>(ctl + 2), 1ull) ==
                 (unsigned long long)(gridDim.x - 1);
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        ctl[2] = 0;
        publish(ctl, flags, world, rank, R + 1, 1);   // the solve's final Delta v
    }
}

// sum_j bufs[j][i] in ascending rank order (canonical_sum's bits): the (remote,
// NVLink) loads of up to 8 ranks are issued together, then added in order.  A
// rank whose accept bit is 0 contributes +0.0 (its Delta v is exactly zero).
__device__ __forceinline__ double rank_sum(double *const *bufs, int world, int64_t i,
                                          uint32_t acc) {
    double s = 0.0;
    if (world <= 8) {
        double x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = j < world && ((acc >> j) & 1) ? __ldcg(bufs[j] + i) : 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (j < world) s += x[j];
        return s;
    }
    for (int j = 0; j < world; ++j) s += ((acc >> j) & 1) ? __ldcg(bufs[j] + i) : 0.0;
    return s;
}

struct RoundStart {
    int mode;                  // 0 apply pending Delta v only; 1 + model; 2 + solve start
    int kind;
    double lam;
    const double *tgt;
    double *v;
    int64_t d;
    double *grad, *lin, *out_fv, *cnst;
    double K, L;
    int world;
    double *const *bufs;
    int64_t pstride;
    const int64_t *flags;      // local flag slots
    int64_t *ctl;
    SolveState *st;            // mode 2
    double *view0, *view1;
    int epochs;
    double *scratch;
    uint64_t timeout;
};

__global__ void __launch_bounds__(PEER_THREADS) round_start_kernel(RoundStart p) {
    __shared__ int s_apply;
    __shared__ int64_t s_R;
    __shared__ uint32_t s_acc;
    if (threadIdx.x == 0) {
        const int64_t R = p.ctl[0], C = p.ctl[1];
        s_R = R;
        s_apply = R > C;
        s_acc = R > C ? wait_flags(p.flags, p.world, R, p.ctl, p.timeout) : 0u;
    }
    __syncthreads();
    const int apply = s_apply;
    const int64_t off = (s_R & 1) * p.pstride;
    const uint32_t accm = s_acc;
    double acc[1] = {0.0};
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const bool dual = kind_is_dual(p.kind);
    for (int64_t r = tid; r < p.d; r += nth) {
        double x = p.v[r];
        if (apply) {
            x += rank_sum(p.bufs, p.world, off + r, accm);
            p.v[r] = x;
        }
        if (p.mode == 0) continue;
        double f, g;                              // outer_model_kernel's arithmetic
        if (dual) {
            f = x * x;
            g = x / p.lam;
        } else {
            f_terms(p.kind, p.lam, p.tgt[r], x, f, g);
            if (f_halved(p.kind)) f *= 2.0;
        }
        acc[0] += f;
        p.grad[r] = g;
        p.lin[r] = g;
        if (p.mode == 2) {
            p.view0[r] = g;
            p.view1[r] = g;
        }
    }
    if (p.mode == 0) {
        // consumed = R only after every block has read (ctl[0], ctl[1]) and made
        // its apply decision: the last block to arrive on the ticket ctl[6]
        // writes it (a block scheduled late must still see C < R)
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const unsigned long long t =
                atomicAdd(reinterpret_cast<unsigned long long *>(p.ctl + 6), 1ull);
            if (t == (unsigned long long)(gridDim.x - 1)) {
                p.ctl[6] = 0;
                if (apply) p.ctl[1] = s_R;
            }
        }
        return;
    }
    if (!reduce_last<1>(acc, p.scratch)) return;
    double f = acc[0];
    if (dual) f = f / (2.0 * p.lam);
    else if (f_halved(p.kind)) f = 0.5 * f;
    *p.out_fv = f;
    const double cn = (f / p.K + 0.0) / p.L;
    *p.cnst = cn;
    if (apply) p.ctl[1] = s_R;
    if (p.mode == 2) {         // begin_kernel with reuse_gsum and reset damping
        SolveState *st = p.st;
        const double G0 = cn + st->gsum_acc;
        st->value = G0;
        st->initial = G0;
        st->gen_state = st->gen_next;
        st->damping = 1.0;
        st->epochs_target = p.epochs;
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


// ---------------------------------------------------------------- turn
// One kernel between two epochs (GLM_FLAG_TURN solves: one attempt each):
//   P1  the attempt's value G and the damping decision (value_kernel mode 1);
//       the same pass writes Delta v to this rank's exchange buffer, and the
//       deciding block sets the accept word and publishes
//   P2  alpha += delta of the accepted attempt (while the peers finish)
//   P3  wait for every rank's Delta v, then the next round's start
//       (round_start_kernel mode 2)
// P1 -> P2 is a grid barrier on st->turn (the deciding block bumps it), P1 ->
// P3 is the ranks' publication flags (ours is released only after all our
// blocks arrived in P1).  Blocks spin only on work that finishes
// independently of them and the grid is sized from the occupancy (1 block per
// SM for a short Delta v, 2 for a long one; glm_peer_create), so every block
// becomes resident; every spin has a %globaltimer deadline.  Block 0 resets
// the solver state for the next round as soon as every block has read the
// decision.  Replaces value + finalize + round start: three kernel launches,
// ramps and tails per round become one.
// decide_attempt (scd.cu) from state loaded up front: the fold's loads and
// the state's loads share one round trip.  Returns 0 when the attempt was
// rejected (the view goes back to the snapshot), else 1.
constexpr int EPOCH_GPART_MAX = 16 * NUM_SMS;     // scd.cu EPOCH_PARTIALS
struct DecideCache {
    double value, damping, cnst, gsum;
    int attempts, status, retries, dc, vw, epochs_run, epochs_target;
};

__device__ __forceinline__ void load_decide(volatile SolveState *st, const double *cnst,
                                            DecideCache &c) {
    c.value = st->value;
    c.damping = st->damping;
    c.cnst = *cnst;
    c.gsum = st->gsum_acc;
    c.attempts = st->attempts;
    c.status = st->status;
    c.retries = st->retries;
    c.dc = st->dc;
    c.vw = st->vw;
    c.epochs_run = st->epochs_run;
    c.epochs_target = st->epochs_target;
}

__device__ __forceinline__ int decide_cached(SolveState *st, const DecideCache &c, double G,
                                             double gnew, double nonfinite) {
    st->attempts = c.attempts + 1;
    if (nonfinite > 0.0) {         // solver.py:279-280
        st->status = GLM_SOLVER_ERROR;
        st->done = 1;
        return 1;
    }
    if (c.status != GLM_OK) {
        st->done = 1;
        return 1;
    }
    if (G > c.value) {
        st->vw = c.vw ^ 1;
        if (G - c.value <= PLATEAU_REL * (1.0 + fabs(c.value))) {
            st->plateaued = 1;
            st->done = 1;
            return 0;
        }
        st->retries = c.retries + 1;
        const double dmp = c.damping * 0.5;
        st->damping = dmp;
        if (dmp < DAMPING_FLOOR) {
            st->status = GLM_DIVERGENCE;
            st->done = 1;
        }
        return 0;
    }
    st->value = G;
    st->gsum_acc = gnew;
    st->dc = c.dc == 0 ? 1 : 0;
    if (c.epochs_run < MAX_EPOCH_VALUES) st->epoch_values[c.epochs_run] = G;
    st->epochs_run = c.epochs_run + 1;
    if (c.epochs_run + 1 >= c.epochs_target) st->done = 1;
    return 1;
}

struct TurnParams {
    SolveState *st;
    double *view0, *view1;
    const double *delta0, *delta1;
    double *partials;          // [blocks][3]
    const double *gpart;
    double quad;
    double *cnst;              // this round's const in, the next round's out
    int64_t m, d;
    double *alpha;
    int box, next_known;
    uint64_t next_state;
    int world, rank;
    double *const *bufs;
    int64_t *const *flags;     // every rank's flag slots
    const int64_t *flags_in;   // local flag slots
    int64_t *ctl;
    double *dv_own;
    int64_t pstride;
    int kind;
    double lam;
    const double *tgt;
    double *v, *grad, *lin, *out_fv;
    double K, L;
    int epochs;
    double *scratch;
    uint64_t *stamps;          // optional phase timestamps (globaltimer ns)
    uint64_t timeout;          // deadline of every wait (ns)
    int rs;                    // P3 as reduce-scatter + all-gather
    double *red_own;           // this rank's reduced slice sums (2 parity halves)
    double *const *red;        // every rank's reduced slice sums
    int64_t *const *flags2;    // every rank's reduced-flag slots
    const int64_t *flags2_in;  // local reduced-flag slots
};


__device__ __forceinline__ uint64_t ld_acquire_gpu_u64(const int64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t ld_acquire_gpu_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

constexpr int TURN_THREADS = 512;
constexpr int TURN_UNROLL = 2;      // rows per thread and pass in P1 / P3

__global__ void __launch_bounds__(TURN_THREADS) round_turn_kernel(TurnParams p) {
    __shared__ double sm[32 * 4];      // block_sum<4>
    __shared__ int s_last;
    __shared__ uint32_t s_turn0;
    __shared__ int64_t s_R;
    __shared__ int s_dc;
    __shared__ uint32_t s_acc;
    SolveState *st = p.st;
    volatile SolveState *vst = st;
    pdl_wait();                 // the epoch kernel's view, partials and state
    tl_start(TL_TURN);
    if (threadIdx.x == 0) {
        s_turn0 = vst->turn;
        s_R = p.ctl[0];
        if (p.stamps && blockIdx.x == 0) p.stamps[0] = gtimer();
    }
    __syncthreads();
    const bool active = !vst->done;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    double *out = p.dv_own + ((s_R + 1) & 1) * p.pstride;
    // ---- P1: value of the attempt; Delta v = (view - lin)/quad goes to the
    // exchange buffer on the same pass (the loads are shared).  If the attempt
    // is rejected the view reverts to the snapshot, which is lin, so the true
    // Delta v is exactly zero: the accept word tells the peers to add +0.0.
    // The same pass sums f(v) for the round's constant: v has not changed
    // since the previous turn's P3 (which therefore skips that reduction), so
    // const = f(v)/K/L and G(0) = const + g-sum are formed here, where the
    // decision needs them.
    {
        const int vw0 = vst->vw;
        const double *V = vw0 ? p.view1 : p.view0;
        const bool dual = kind_is_dual(p.kind);
        double acc[3] = {0.0, 0.0, 0.0};           // f(v), view terms, non-finite
        // TURN_UNROLL rows per thread and pass, every load issued before any
        // is used (the same rows per thread and the same summation order as a
        // plain grid-stride loop)
        for (int64_t r0 = tid; r0 < p.d; r0 += TURN_UNROLL * nth) {
            double x[TURN_UNROLL], l[TURN_UNROLL], vr[TURN_UNROLL], t[TURN_UNROLL];
#pragma unroll
            for (int k = 0; k < TURN_UNROLL; ++k) {
                const int64_t r = r0 + k * nth;
                const bool in = r < p.d;
                x[k] = in ? __ldcg(V + r) : 0.0;
                l[k] = in ? p.lin[r] : 0.0;
                vr[k] = in ? p.v[r] : 0.0;
                t[k] = in && !dual ? p.tgt[r] : 0.0;
            }
#pragma unroll
            for (int k = 0; k < TURN_UNROLL; ++k) {
                const int64_t r = r0 + k * nth;
                if (r >= p.d) break;
                const double u = x[k] - l[k];
                out[r] = u / p.quad;
                double f, g;                        // outer_model_kernel's arithmetic
                if (dual) {
                    f = vr[k] * vr[k];
                } else {
                    f_terms(p.kind, p.lam, t[k], vr[k], f, g);
                    if (f_halved(p.kind)) f *= 2.0;
                }
                acc[0] += f;
                if (active) {
                    if (!isfinite(x[k])) acc[2] += 1.0;
                    acc[1] += l[k] * u + 0.5 * u * u;
                }
            }
        }
        block_sum<3>(acc, sm);
        if (threadIdx.x == 0) {
            p.partials[blockIdx.x * 3 + 0] = acc[0];
            p.partials[blockIdx.x * 3 + 1] = acc[1];
            p.partials[blockIdx.x * 3 + 2] = acc[2];
            __threadfence();        // partials and Delta v before the arrival
            s_last = atomicAdd(&st->block_counter, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            if (p.stamps && threadIdx.x == 0) p.stamps[7] = gtimer();
            // one round of independent loads: the decision's state (thread 0),
            // the block partials and every possible epoch partial (masked by
            // the epoch's grid size once it arrives) — the same sums, in the
            // same order, as value_kernel mode 1 + decide_attempt
            DecideCache dcache;
            if (threadIdx.x == 0) load_decide(vst, p.cnst, dcache);
            const int eb = active ? vst->epoch_blocks : 0;
            double t4[4] = {0.0, 0.0, 0.0, 0.0};       // f(v), view terms, non-finite, g-sum
            for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
                t4[0] += __ldcg(p.partials + b * 3 + 0);
                t4[1] += __ldcg(p.partials + b * 3 + 1);
                t4[2] += __ldcg(p.partials + b * 3 + 2);
            }
            {
                double gp[EPOCH_GPART_MAX / TURN_THREADS];
#pragma unroll
                for (int k = 0; k < EPOCH_GPART_MAX / TURN_THREADS; ++k)
                    gp[k] = __ldcg(p.gpart + threadIdx.x + k * TURN_THREADS);
#pragma unroll
                for (int k = 0; k < EPOCH_GPART_MAX / TURN_THREADS; ++k)
                    if ((int)threadIdx.x + k * TURN_THREADS < eb) t4[3] += gp[k];
            }
            block_sum<4>(t4, sm);
            if (threadIdx.x == 0) {
                st->block_counter = 0;
                double f = t4[0];                       // round_start_kernel's scaling
                if (kind_is_dual(p.kind)) f = f / (2.0 * p.lam);
                else if (f_halved(p.kind)) f = 0.5 * f;
                const double cn = (f / p.K + 0.0) / p.L;
                *p.out_fv = f;
                *p.cnst = cn;
                int accept = 1;
                if (active) {
                    dcache.cnst = cn;
                    dcache.value = cn + dcache.gsum;    // G(0): begin_kernel with reuse_gsum
                    st->value = dcache.value;
                    st->initial = dcache.value;
                    accept = decide_cached(st, dcache, cn + t4[1] / p.quad + t4[3], t4[3], t4[2]);
                }
                __threadfence();
                if (p.stamps) p.stamps[1] = gtimer();
                atomicAdd(&st->turn, 1u);          // the other blocks go on to alpha
                if (p.stamps) p.stamps[2] = gtimer();
                publish(p.ctl, p.flags, p.world, p.rank, s_R + 1, accept, p.stamps);
            }
        }
        if (threadIdx.x == 0) {
            uint64_t t0 = 0;
            while (ld_acquire_gpu_u32(&st->turn) == s_turn0) {
                __nanosleep(32);
                if (expired(t0, p.timeout)) {        // blocks not co-resident
                    peer_fail(p.ctl, PEER_ERR_GRID, 1);
                    break;
                }
            }
            s_dc = vst->dc;
            // read: block 0 may now reset the solver state (end of P3)
            atomicAdd(&st->block_counter, 1u);
        }
        __syncthreads();
    }
    // ---- P2: alpha += delta of the accepted attempt (overlaps the peers)
    {
        const int dc = s_dc;
        const double *dl = dc < 0 ? nullptr : (dc ? p.delta1 : p.delta0);
        if (dl) {   // 4 independent rows per thread and pass: keep loads in flight
            for (int64_t j0 = tid; j0 < p.m; j0 += 4 * nth) {
                double a[4], x[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int64_t j = j0 + u * nth;
                    a[u] = j < p.m ? p.alpha[j] : 0.0;
                    x[u] = j < p.m ? __ldcg(dl + j) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int64_t j = j0 + u * nth;
                    if (j < p.m) p.alpha[j] = p.box ? fmin(1.0, fmax(0.0, a[u] + x[u])) : a[u] + x[u];
                }
            }
        }
        if (blockIdx.x == 0 && threadIdx.x < 32) {
            const uint64_t g = p.next_known
                                   ? p.next_state
                                   : warp_jump(vst->gen_state, (uint64_t)vst->attempts * (uint64_t)p.m);
            if (threadIdx.x == 0) st->gen_next = g;
        }
    }
    // ---- P3: every rank's Delta v, then the next round's start
    pdl_trigger();              // the next epoch may be scheduled as blocks drain
    const int64_t R = s_R + 1;
    if (threadIdx.x == 0) {
        if (blockIdx.x == 0) {
            // block 0 waits with the deadline and relays what it saw (ctl[3],
            // the accept bits in ctl[4]) for a rank that missed it
            const uint32_t mask = wait_flags(p.flags_in, p.world, R, p.ctl, p.timeout);
            s_acc = mask;
            p.ctl[4] = (int64_t)mask;
            __threadfence();
            atomicMax(reinterpret_cast<unsigned long long *>(p.ctl + 3), (unsigned long long)R);
        } else {
            // the other blocks read the local flag slots themselves (the peers
            // store into them over NVLink) — one hop less than block 0's relay
            uint64_t t0 = 0;
            for (;;) {
                uint32_t mask = 0;
                bool all = true;
                for (int j = 0; j < p.world && all; ++j) {
                    const int64_t f = ld_acquire_sys(p.flags_in + j);
                    if ((f >> 2) < R) all = false;
                    else mask |= (uint32_t)((f >> (R & 1)) & 1) << j;
                }
                if (all) {
                    s_acc = mask;
                    break;
                }
                if ((int64_t)ld_acquire_gpu_u64(p.ctl + 3) >= R) {
                    s_acc = (uint32_t)*(volatile int64_t *)(p.ctl + 4);
                    break;
                }
                __nanosleep(32);
                if (expired(t0, 2 * p.timeout)) {    // block 0's own wait has the deadline
                    peer_fail(p.ctl, PEER_ERR_GRID, 3);
                    s_acc = 0;
                    break;
                }
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (p.stamps) p.stamps[3] = gtimer();
        // every block read the decision right after the P1 -> P2 barrier (long
        // done): block 0 resets the solver state for the next round here, off
        // the kernel's tail.  f(v), the constant and G(0) of the next round are
        // formed by its P1.
        uint64_t t0 = 0;
        while (ld_acquire_gpu_u32(&st->block_counter) < gridDim.x) {
            __nanosleep(32);
            if (expired(t0, p.timeout)) {
                peer_fail(p.ctl, PEER_ERR_GRID, 4);
                break;
            }
        }
        st->block_counter = 0;
        p.ctl[1] = R;
        if (st->status == GLM_OK) {                 // else keep the error visible to the host
            st->gen_state = st->gen_next;           // begin_kernel with reuse_gsum
            // damping: an accepted (or plateaued) attempt resets it like the
            // reference's per-round reset (engine.py:251-252); a rejected one
            // keeps the halved value, so the next round is the retry
            // damped_solve would have made (solver.py:282-293) and consecutive
            // rejections reach the floor and GLM_DIVERGENCE (decide_cached)
            // instead of looping at damping 1
            if (st->epochs_run > 0 || st->plateaued) st->damping = 1.0;
            st->epochs_target = p.epochs;
            st->epochs_run = 0;
            st->retries = 0;
            st->plateaued = 0;
            st->attempts = 0;
            st->status = GLM_OK;
            st->done = 0;
            st->dc = -1;
            st->vw = 0;
            st->epoch_blocks = 0;
        }
    }
    __syncthreads();
    const int64_t off = (R & 1) * p.pstride;
    const uint32_t accm = s_acc;
    const bool dual = kind_is_dual(p.kind);
    // Reduce-scatter + all-gather (3+ ranks): rank j sums, in rank order, only
    // its slice [j cs, (j+1) cs) of every rank's Delta v and publishes it; every
    // rank then reads each row's sum from the slice owner — (N-1)/N * 8d bytes
    // read twice instead of (N-1) * 8d, the same rank-order sum per row.
    const int64_t cs = (p.d + (int64_t)p.world * 32 - 1) / ((int64_t)p.world * 32) * 32;
    if (p.rs) {
        const int64_t lo = (int64_t)p.rank * cs, hi = lo + cs < p.d ? lo + cs : p.d;
        for (int64_t r = lo + tid; r < hi; r += nth)
            p.red_own[off + r] = rank_sum(p.bufs, p.world, off + r, accm);
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const bool last = atomicAdd(reinterpret_cast<unsigned long long *>(p.ctl + 8), 1ull) ==
                              (unsigned long long)(gridDim.x - 1);
            if (last) {                // every block's slice rows are written: publish
                p.ctl[8] = 0;
                __threadfence_system();
                for (int j = 0; j < p.world; ++j) st_relaxed_sys(p.flags2[j] + p.rank, R);
            }
            if (blockIdx.x == 0) {
                wait_rounds(p.flags2_in, p.world, R, p.ctl, p.timeout);
                __threadfence();
                atomicMax(reinterpret_cast<unsigned long long *>(p.ctl + 9), (unsigned long long)R);
            } else {
                uint64_t t0 = 0;
                while ((int64_t)ld_acquire_gpu_u64(p.ctl + 9) < R) {
                    __nanosleep(32);
                    if (expired(t0, 2 * p.timeout)) {
                        peer_fail(p.ctl, PEER_ERR_GRID, 5);
                        break;
                    }
                }
            }
        }
        __syncthreads();
    }
    for (int64_t r0 = tid; r0 < p.d; r0 += TURN_UNROLL * nth) {
        double sm2[TURN_UNROLL], v0[TURN_UNROLL];
#pragma unroll
        for (int k = 0; k < TURN_UNROLL; ++k) {   // every rank's rows in flight together
            const int64_t r = r0 + k * nth;
            const bool in = r < p.d;
            sm2[k] = !in ? 0.0
                         : p.rs ? __ldcg(p.red[r / cs] + off + r)
                                : rank_sum(p.bufs, p.world, off + r, accm);
            v0[k] = in ? p.v[r] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < TURN_UNROLL; ++k) {
            const int64_t r = r0 + k * nth;
            if (r >= p.d) break;
            const double x = v0[k] + sm2[k];
            p.v[r] = x;
            double f, g;
            if (dual) {
                g = x / p.lam;
            } else {
                f_terms(p.kind, p.lam, p.tgt[r], x, f, g);
            }
            p.grad[r] = g;
            p.lin[r] = g;
            p.view0[r] = g;
            p.view1[r] = g;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        tl_end(TL_TURN);
        if (p.stamps) p.stamps[4] = gtimer();    // block 0's own P3 rows done
    }
}

__global__ void peer_consume_kernel(int64_t *ctl) { ctl[1] = ctl[0]; }

int peer_finalize(glm_solver *s, glm_peer *pr, const double *lin, double quad, int64_t m,
                  int64_t d, double *alpha, int box, int next_known, uint64_t next_state,
                  cudaStream_t stream) {
    if (pr->d != d) return glm_set_error(GLM_USAGE, "peer exchange sized for another d");
    count_launch();
    int64_t blocks = ((m > d ? m : d) + 4 * PEER_THREADS - 1) / (4 * PEER_THREADS);
    blocks = blocks < 1 ? 1 : (blocks > 8 * NUM_SMS ? 8 * NUM_SMS : blocks);
    peer_finalize_kernel<<<(int)blocks, PEER_THREADS, 0, stream>>>(
        s->st, s->delta[0], s->delta[1], s->view[0], s->view[1], lin, quad, m, d, alpha, box,
        pr->dv, pr->pstride, pr->ctl, pr->flags_dev, pr->world, pr->rank, next_known, next_state);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

}  // namespace glm

using namespace glm;

extern "C" {

int glm_peer_destroy(glm_peer *p) {
    if (!p) return GLM_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(p->device);
    cudaDeviceSynchronize();
    for (void *q : p->opened) cudaIpcCloseMemHandle(q);
    cudaFree(p->mem);
    cudaFree(p->bufs_dev);
    cudaFree(p->flags_dev);
    cudaFree(p->red_dev);
    cudaFree(p->flags2_dev);
    cudaSetDevice(prev);
    delete p;
    return GLM_OK;
}

int glm_peer_create(int device, int64_t d, int rank, int world, glm_peer **out) {
    if (!out || d < 0 || world < 1 || rank < 0 || rank >= world)
        return glm_set_error(GLM_USAGE, "bad peer arguments");
    if (world > PEER_MAX_WORLD) return glm_set_error(GLM_USAGE, "peer exchange: world > 24");
    GLM_CUDA_TRY(cudaSetDevice(device));
    glm_peer *p = new (std::nothrow) glm_peer();
    if (!p) return glm_set_error(GLM_USAGE, "out of host memory");
    p->device = device;
    p->rank = rank;
    p->world = world;
    p->d = d;
    p->pstride = peer_pstride(d);
    const size_t bytes = PEER_HEADER + sizeof(double) * 4 * (size_t)p->pstride;
    cudaError_t e = cudaMalloc(&p->mem, bytes);
    if (e == cudaSuccess) e = cudaMemset(p->mem, 0, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&p->bufs_dev, sizeof(double *) * world);
    if (e == cudaSuccess) e = cudaMalloc(&p->flags_dev, sizeof(int64_t *) * world);
    if (e == cudaSuccess) e = cudaMalloc(&p->red_dev, sizeof(double *) * world);
    if (e == cudaSuccess) e = cudaMalloc(&p->flags2_dev, sizeof(int64_t *) * world);
    if (e == cudaSuccess && world > 1) e = cudaIpcGetMemHandle(&p->handle, p->mem);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        glm_peer_destroy(p);
        return glm_set_cuda_error(e, "glm_peer_create", __FILE__, __LINE__);
    }
    // round_turn spins on work of its other blocks, so its grid must be
    // co-resident: size it from this device's SM count and the kernel's
    // occupancy (fail rather than risk a deadlock)
    int sms = 0, occ = 0;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, round_turn_kernel, TURN_THREADS, 0);
    if (e != cudaSuccess || occ < 1 || sms < 1) {
        glm_peer_destroy(p);
        if (e != cudaSuccess) return glm_set_cuda_error(e, "glm_peer_create", __FILE__, __LINE__);
        return glm_set_error(GLM_USAGE, "round_turn_kernel cannot be resident on this device");
    }
    // A short Delta v (C2: 100k rows) leaves the turn latency-bound: one block
    // per SM, and the rest of the SM takes the permutation prefetch and the
    // next epoch's first CTAs while the turn waits on its peers (bench.py C2,
    // one box, 3 runs each: 2 per SM -> 1 per SM 3713 -> 3829 epochs/s at 2
    // ranks, 6347 -> 6769 at 4; at 1 rank with the early release 1934).  A long
    // one (C4: 10M rows) makes P1 and P3 bandwidth passes that want every
    // thread: 2 per SM (1 per SM: 330 -> 297 epochs/s at 2 ranks, 495 -> 457 at 4).
    int per_sm = d >= (int64_t)1 << 20 ? (occ < 2 ? occ : 2) : 1;
    if (const char *env = getenv("GLM_TURN_BLOCKS_PER_SM"))   // experiments: 1 or 2
        per_sm = atoi(env) >= 1 && atoi(env) <= (occ < 2 ? occ : 2) ? atoi(env) : per_sm;
    p->turn_blocks = per_sm * sms;
    if (p->turn_blocks > PEER_BLOCKS) p->turn_blocks = PEER_BLOCKS;
    p->ctl = reinterpret_cast<int64_t *>(p->mem);
    p->dv = reinterpret_cast<double *>(p->mem + PEER_HEADER);
    p->flags = p->ctl + PEER_FLAGS;
    p->flags2 = p->ctl + PEER_FLAGS2;
    // reduce-scatter + all-gather for 3+ ranks and a large Delta v (at 2 ranks
    // it moves the same bytes as reading the peer's whole Delta v; for a small
    // one its extra flag round trip costs more than the bytes it saves: C2's
    // 800 KB at 4 GPUs, turn 32.7 -> 38.5 us); GLM_PEER_RS=0/1 overrides
    p->rs = world >= 3 && d >= (int64_t)1 << 22;
    if (const char *env = getenv("GLM_PEER_RS")) p->rs = env[0] == '1';
    if (world == 1) {
        p->rs = 0;
        double *b = p->dv, *rd = p->dv + 2 * p->pstride;
        int64_t *f = p->flags, *f2 = p->flags2;
        GLM_CUDA_TRY(cudaMemcpy(p->bufs_dev, &b, sizeof(b), cudaMemcpyHostToDevice));
        GLM_CUDA_TRY(cudaMemcpy(p->flags_dev, &f, sizeof(f), cudaMemcpyHostToDevice));
        GLM_CUDA_TRY(cudaMemcpy(p->red_dev, &rd, sizeof(rd), cudaMemcpyHostToDevice));
        GLM_CUDA_TRY(cudaMemcpy(p->flags2_dev, &f2, sizeof(f2), cudaMemcpyHostToDevice));
    }
    *out = p;
    return GLM_OK;
}

size_t glm_peer_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

int glm_peer_handle(const glm_peer *p, void *handle_out) {
    if (!p || !handle_out) return glm_set_error(GLM_USAGE, "null argument");
    memcpy(handle_out, &p->handle, sizeof(cudaIpcMemHandle_t));
    return GLM_OK;
}

int glm_peer_open(glm_peer *p, const void *handles) {
    if (!p) return glm_set_error(GLM_USAGE, "null peer");
    if (p->world == 1) return GLM_OK;
    if (!handles) return glm_set_error(GLM_USAGE, "world > 1 needs every rank's handle");
    GLM_CUDA_TRY(cudaSetDevice(p->device));
    std::vector<double *> bufs(p->world), red(p->world);
    std::vector<int64_t *> flags(p->world), flags2(p->world);
    for (int j = 0; j < p->world; ++j) {
        char *base;
        if (j == p->rank) {
            base = p->mem;
        } else {
            cudaIpcMemHandle_t h;
            memcpy(&h, (const char *)handles + j * sizeof(cudaIpcMemHandle_t), sizeof(h));
            void *q = nullptr;
            GLM_CUDA_TRY(cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess));
            p->opened.push_back(q);
            base = (char *)q;
        }
        flags[j] = reinterpret_cast<int64_t *>(base) + PEER_FLAGS;
        flags2[j] = reinterpret_cast<int64_t *>(base) + PEER_FLAGS2;
        bufs[j] = reinterpret_cast<double *>(base + PEER_HEADER);
        red[j] = bufs[j] + 2 * p->pstride;
    }
    GLM_CUDA_TRY(cudaMemcpy(p->bufs_dev, bufs.data(), sizeof(double *) * p->world,
                            cudaMemcpyHostToDevice));
    GLM_CUDA_TRY(cudaMemcpy(p->flags_dev, flags.data(), sizeof(int64_t *) * p->world,
                            cudaMemcpyHostToDevice));
    GLM_CUDA_TRY(cudaMemcpy(p->red_dev, red.data(), sizeof(double *) * p->world,
                            cudaMemcpyHostToDevice));
    GLM_CUDA_TRY(cudaMemcpy(p->flags2_dev, flags2.data(), sizeof(int64_t *) * p->world,
                            cudaMemcpyHostToDevice));
    return GLM_OK;
}

// Debug: record glm_round_turn phase timestamps (globaltimer ns) into a
// device array of 8 u64 (start, decided, published, peers seen, done).
int glm_peer_stamps(glm_peer *p, uint64_t *device_array) {
    if (!p) return glm_set_error(GLM_USAGE, "null peer");
    p->stamps = device_array;
    return GLM_OK;
}

int glm_peer_set_timeout(glm_peer *p, double seconds) {
    if (!p || !(seconds > 0.0)) return glm_set_error(GLM_USAGE, "bad peer timeout");
    p->timeout_ns = (uint64_t)(seconds * 1e9);
    return GLM_OK;
}

// Synchronises the device, then reads (and with clear != 0 resets) the error
// word: 0 = no wait timed out; else (kind << 32 | what), kind 1 = rank `what`
// did not publish in time, kind 2 = the turn's blocks were not co-resident.
int glm_peer_error(glm_peer *p, int64_t *code_out, int clear) {
    if (!p || !code_out) return glm_set_error(GLM_USAGE, "null argument");
    GLM_CUDA_TRY(cudaSetDevice(p->device));
    GLM_CUDA_TRY(cudaDeviceSynchronize());
    GLM_CUDA_TRY(cudaMemcpy(code_out, p->ctl + 7, sizeof(int64_t), cudaMemcpyDeviceToHost));
    if (clear && *code_out) GLM_CUDA_TRY(cudaMemset(p->ctl + 7, 0, sizeof(int64_t)));
    return GLM_OK;
}

int glm_peer_consume(glm_peer *p, void *stream) {
    if (!p) return glm_set_error(GLM_USAGE, "null peer");
    count_launch();
    peer_consume_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(p->ctl);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

int glm_round_start(glm_peer *p, glm_solver *s, int mode, int kind, double lam,
                    const double *target, double *v, int64_t d, double *grad, double *lin,
                    double *out_fv, double *cnst, double n_nodes, double n_devices, int epochs,
                    double *scratch, void *stream) {
    if (!p || !v || (mode > 0 && (!grad || !lin || !out_fv || !cnst || !scratch)) ||
        (mode == 2 && !s))
        return glm_set_error(GLM_USAGE, "null argument to glm_round_start");
    if (p->d != d) return glm_set_error(GLM_USAGE, "peer exchange sized for another d");
    if (mode == 2 && d > s->max_rows) return glm_set_error(GLM_USAGE, "solver too small");
    RoundStart a{};
    a.mode = mode;
    a.kind = kind;
    a.lam = lam;
    a.tgt = target;
    a.v = v;
    a.d = d;
    a.grad = grad;
    a.lin = lin;
    a.out_fv = out_fv;
    a.cnst = cnst;
    a.K = n_nodes;
    a.L = n_devices;
    a.world = p->world;
    a.bufs = p->bufs_dev;
    a.pstride = p->pstride;
    a.flags = p->flags;
    a.ctl = p->ctl;
    a.st = s ? s->st : nullptr;
    a.view0 = s ? s->view[0] : nullptr;
    a.view1 = s ? s->view[1] : nullptr;
    a.epochs = epochs;
    a.scratch = scratch;
    a.timeout = p->timeout_ns;
    const bool timed = s && s->timing;
    if (timed) {
        int rc = glue_begin(s, 1, (cudaStream_t)stream);
        if (rc) return rc;
    }
    count_launch();
    round_start_kernel<<<PEER_BLOCKS, PEER_THREADS, 0, (cudaStream_t)stream>>>(a);
    GLM_CUDA_TRY(cudaGetLastError());
    if (timed) return glue_end(s, (cudaStream_t)stream);
    return GLM_OK;
}

int glm_round_turn(glm_peer *p, glm_solver *s, int kind, double lam, double quad,
                   double *cnst, double *alpha, int64_t m, const double *target, double *v,
                   int64_t d, double *grad, double *lin, double *out_fv, double n_nodes,
                   double n_devices, int epochs, double *scratch, void *stream) {
    if (!p || !s || !cnst || !alpha || !v || !grad || !lin || !out_fv || !scratch)
        return glm_set_error(GLM_USAGE, "null argument to glm_round_turn");
    if (p->d != d || d > s->max_rows || m > s->max_coords)
        return glm_set_error(GLM_USAGE, "glm_round_turn sizes do not match");
    // measured (bench.py C2, one box, 3 runs each): at 1 rank the epoch's
    // early release of this kernel pays (1906 -> 1934 epochs/s); with peers
    // it costs (3829 -> 3749 at 2 ranks, 6769 -> 6697 at 4)
    s->early_trigger = p->world == 1 ? 1 : 0;
    TurnParams a{};
    a.st = s->st;
    a.view0 = s->view[0];
    a.view1 = s->view[1];
    a.delta0 = s->delta[0];
    a.delta1 = s->delta[1];
    a.partials = s->partials;
    a.gpart = s->gpart;
    a.quad = quad;
    a.cnst = cnst;
    a.m = m;
    a.d = d;
    a.alpha = alpha;
    a.box = kind == GLM_DUAL_L2_SVM ? 1 : 0;
    a.next_known = s->host_known ? 1 : 0;
    a.next_state = s->host_gen;
    a.world = p->world;
    a.rank = p->rank;
    a.bufs = p->bufs_dev;
    a.flags = p->flags_dev;
    a.flags_in = p->flags;
    a.ctl = p->ctl;
    a.dv_own = p->dv;
    a.pstride = p->pstride;
    a.kind = kind;
    a.lam = lam;
    a.tgt = target;
    a.v = v;
    a.grad = grad;
    a.lin = lin;
    a.out_fv = out_fv;
    a.K = n_nodes;
    a.L = n_devices;
    a.epochs = epochs;
    a.scratch = scratch;
    a.stamps = p->stamps;
    a.timeout = p->timeout_ns;
    a.rs = p->rs;
    a.red_own = p->dv + 2 * p->pstride;
    a.red = p->red_dev;
    a.flags2 = p->flags2_dev;
    a.flags2_in = p->flags2;
    cudaStream_t st = (cudaStream_t)stream;
    if (s->timing) {
        int rc = glue_begin(s, 2, st);
        if (rc) return rc;
    }
    count_launch();
    GLM_CUDA_TRY(launch_pdl(true, round_turn_kernel, dim3(p->turn_blocks), dim3(TURN_THREADS), 0,
                            st, a));
    if (s->timing) return glue_end(s, st);
    return GLM_OK;
}

}  // extern "C"
