// common.cuh — shared device code for the B200 GLM/TPA-SCD kernels (sm_100a).
#pragma once
#include <utility>
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "glm_b200.h"

namespace glm {

constexpr double BOUNDARY_EPS = 1e-12;          // objectives.py:26
constexpr double DAMPING_FLOOR = 9.5367431640625e-07;  // 2^-20, solver.py:28
constexpr double PLATEAU_REL = 1e-12;           // solver.py:247
constexpr int MAX_EPOCH_VALUES = 256;           // epoch_values kept per solve
constexpr int NUM_SMS = 148;                    // B200

// Device-resident solver state: the reference's DampingState + the control
// flow of damped_solve (solver.py:250-305) turned into a state machine that
// the kernels of one attempt read, so attempts can be enqueued without host
// round-trips.
struct SolveState {
    uint64_t gen_state;       // PermutationGenerator.state at solve start
    uint64_t gen_next;        // state after the solve (finalize)
    double damping;           // DampingState.delta
    double value;             // current accepted G
    double initial;           // G(0)
    int32_t epochs_target;
    int32_t epochs_run;
    int32_t retries;
    int32_t plateaued;
    int32_t attempts;         // scd_epoch calls executed (== permutations consumed)
    int32_t status;           // GLM_OK / GLM_SOLVER_ERROR / GLM_DIVERGENCE
    int32_t done;
    int32_t dc;               // current delta buffer
    int32_t vw;               // working view buffer
    int32_t epoch_blocks;     // blocks of the last epoch kernel (g-sum partials)
    double gsum_acc;          // sum_j g(base_j + delta_j) of the accepted state
    uint32_t block_counter;   // last-block-done counter for reductions
    uint32_t turn;            // barrier generation of glm_round_turn (peer.cu)
    // chunked (out-of-core) mode, pipeline.py:158-197: the chunk being solved
    // (a sequence number over epochs x chunks; -1 before the first) and the
    // g-sum of its coordinates in the accepted state.
    int64_t seq;
    double gsum_old;
    double epoch_values[MAX_EPOCH_VALUES];
};

__device__ __forceinline__ double ld_cg(const double *p) {
    double v;
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ void red_add(double *p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// Cache-policy variants used by the async epoch kernel (flags of glm_solve_args).
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double ld_stream_f64(const double *p, uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                 : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int ld_stream_i32(const int *p, uint64_t pol) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
                 : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld_cg_hint(const double *p, uint64_t pol) {
    double v;
    asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld_ca_hint(const double *p, uint64_t pol) {
    double v;
    asm volatile("ld.global.ca.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void red_add_hint(double *p, double v, uint64_t pol) {
    asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol)
                 : "memory");
}

template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_sum(double v) { return group_sum<32>(v); }

// Block reduction of NV doubles (blockDim multiple of 32, <= 1024).
template <int NV, int NS>
__device__ __forceinline__ void block_sum(double (&v)[NV], double (&smem)[NS]) {
    static_assert(NS >= 32 * NV, "block_sum needs 32 shared doubles per value");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
    __syncthreads();
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) smem[i * 32 + warp] = v[i];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double x = lane < nw ? smem[i * 32 + lane] : 0.0;
            v[i] = warp_sum(x);
        }
    }
    __syncthreads();
}

// ---------------------------------------------------------------- objectives
__device__ __forceinline__ bool kind_is_dual(int kind) {
    return kind == GLM_DUAL_L2_LOGISTIC || kind == GLM_DUAL_L2_SVM || kind == GLM_DUAL_RIDGE;
}

__device__ __forceinline__ double entropy(double a) {   // objectives.py:142-147
    double t1 = a > 0.0 ? a * log(fmax(a, 1e-320)) : 0.0;
    double b = 1.0 - a;
    double t2 = a < 1.0 ? b * log(fmax(b, 1e-320)) : 0.0;
    return t1 + t2;
}

__device__ __forceinline__ double softplus(double s) {   // np.logaddexp(0, s)
    return s > 0.0 ? s + log1p(exp(-s)) : log1p(exp(s));
}

__device__ __forceinline__ double sigmoid_tanh(double z) {   // modelio.py:78-79
    return 0.5 * (1.0 + tanh(0.5 * z));
}

// g_i(a) (objectives.py:150-173; restated kinds 4..7)
__device__ __forceinline__ double g_one(int kind, double lam, double rho, double y, double a) {
    switch (kind) {
    case GLM_DUAL_L2_LOGISTIC: return entropy(a);
    case GLM_DUAL_L2_SVM: return -a;
    case GLM_RIDGE_PRIMAL:
    case GLM_LOGISTIC_PRIMAL:
    case GLM_SQUARED_HINGE_PRIMAL:
    case GLM_HINGE_PRIMAL: return 0.5 * lam * a * a;
    case GLM_LASSO_PRIMAL: return lam * fabs(a);
    case GLM_DUAL_RIDGE: return 0.5 * a * a - y * a;
    case GLM_ELASTIC_NET_PRIMAL: return lam * (rho * fabs(a) + 0.5 * (1.0 - rho) * a * a);
    }
    return NAN;
}

// g_i*(s) (objectives.py:211-220); NAN when no closed form
__device__ __forceinline__ double g_conj_one(int kind, double lam, double rho, double y, double s) {
    switch (kind) {
    case GLM_DUAL_L2_LOGISTIC: return softplus(s);
    case GLM_DUAL_L2_SVM: return fmax(0.0, s + 1.0);
    case GLM_RIDGE_PRIMAL:
    case GLM_LOGISTIC_PRIMAL:
    case GLM_SQUARED_HINGE_PRIMAL:
    case GLM_HINGE_PRIMAL: return s * s / (2.0 * lam);
    case GLM_DUAL_RIDGE: { double u = s + y; return 0.5 * u * u; }
    case GLM_ELASTIC_NET_PRIMAL: {
        if (rho >= 1.0) return NAN;
        double u = fabs(s) - lam * rho;
        return u > 0.0 ? u * u / (2.0 * lam * (1.0 - rho)) : 0.0;
    }
    }
    return NAN;
}

// Undamped 1-D step (coordinate_update, solver.py:152-187) from ga and
// c = quad*||a||^2.  Returns false on a solver error (non-finite).
__device__ __forceinline__ bool coord_step(int kind, double lam, double rho, double y, double ga,
                                           double c, double t, double &step) {
    if (!isfinite(ga)) return false;
    switch (kind) {
    case GLM_RIDGE_PRIMAL:
    case GLM_LOGISTIC_PRIMAL:
    case GLM_SQUARED_HINGE_PRIMAL:
    case GLM_HINGE_PRIMAL:
        step = -(ga + lam * t) / (c + lam);
        return true;
    case GLM_ELASTIC_NET_PRIMAL:
        if (rho < 1.0) {
            double den = c + lam * (1.0 - rho);
            double z = c * t - ga;
            double m = fabs(z) - lam * rho;
            step = copysign(m > 0.0 ? m : 0.0, z) / den - t;
            return true;
        }
        // rho == 1: exactly the lasso path below
    case GLM_LASSO_PRIMAL: {
        if (c == 0.0) { step = -t; return true; }
        double u = t - ga / c, thr = lam / c;
        double m = fabs(u) - thr;
        step = copysign(m > 0.0 ? m : 0.0, u) - t;
        return true;
    }
    case GLM_DUAL_L2_SVM: {
        double tn;
        if (c == 0.0) tn = ga < 1.0 ? 1.0 : 0.0;
        else tn = fmin(1.0, fmax(0.0, t + (1.0 - ga) / c));
        step = tn - t;
        return true;
    }
    case GLM_DUAL_RIDGE:
        step = -(ga + t - y) / (c + 1.0);
        return true;
    case GLM_DUAL_L2_LOGISTIC: {
        // math.log / the division raise for t outside (0, 1) (solver.py:181);
        // reachable only with a caller-held damping above 1
        if (!(t > 0.0 && t < 1.0)) return false;
        double grad = ga + log(t / (1.0 - t));
        double curv = c + 1.0 / (t * (1.0 - t));
        double tn = t - grad / curv;
        tn = fmin(1.0 - BOUNDARY_EPS, fmax(BOUNDARY_EPS, tn));
        if (!isfinite(tn)) return false;
        step = tn - t;
        return true;
    }
    }
    return false;
}

// f contributions per row r (objectives.py:129-139, 205-208)
// f(v) accumulated as squares and halved once at the end (quadratic kinds),
// or as the per-row values themselves (logistic, smoothed hinge)
__device__ __forceinline__ bool f_halved(int kind) {
    return kind != GLM_LOGISTIC_PRIMAL && kind != GLM_HINGE_PRIMAL;
}

__device__ __forceinline__ void f_terms(int kind, double lam, double tgt, double v, double &f,
                                        double &g) {
    if (kind_is_dual(kind)) { f = v * v / (2.0 * lam); g = v / lam; return; }
    if (kind == GLM_LOGISTIC_PRIMAL) {
        f = softplus(-tgt * v);
        g = -tgt * sigmoid_tanh(-tgt * v);
        return;
    }
    if (kind == GLM_SQUARED_HINGE_PRIMAL) {
        double m = 1.0 - tgt * v;
        f = m > 0.0 ? 0.5 * m * m : 0.0;
        g = m > 0.0 ? -tgt * m : 0.0;
        return;
    }
    if (kind == GLM_HINGE_PRIMAL) {      // smoothed hinge; the row target is y / mu
        const double y = tgt > 0.0 ? 1.0 : -1.0, mu = 1.0 / fabs(tgt), z = y * v;
        if (z >= 1.0) {
            f = 0.0;
            g = 0.0;
        } else if (z > 1.0 - mu) {
            const double m = 1.0 - z;
            f = m * m / (2.0 * mu);
            g = -y * m / mu;
        } else {
            f = 1.0 - z - 0.5 * mu;
            g = -y;
        }
        return;
    }
    double e = v - tgt;
    f = 0.5 * e * e;
    g = e;
}

__device__ __forceinline__ double f_conj_term(int kind, double lam, double tgt, double w) {
    if (kind_is_dual(kind)) return 0.5 * lam * w * w;
    if (kind == GLM_LOGISTIC_PRIMAL) return entropy(-w * tgt);
    if (kind == GLM_SQUARED_HINGE_PRIMAL) { double q = -w * tgt; return 0.5 * q * q - q; }
    if (kind == GLM_HINGE_PRIMAL) {      // h*(u) = u + mu u^2 / 2 on [-1, 0], u = y w
        const double u = (tgt > 0.0 ? 1.0 : -1.0) * w, mu = 1.0 / fabs(tgt);
        return u + 0.5 * mu * u * u;
    }
    return 0.5 * w * w + w * tgt;
}

// Host-side count of kernels this library launched (bench.py "gpu_launches").
void count_launch();

// Debug timeline (glm_debug_timeline): when set, kernels record the earliest
// start (atomicMin) and latest end (atomicMax) of %globaltimer in slot pairs.
enum { TL_EPOCH = 0, TL_PERM_FIRST = 1, TL_PERM_LAST = 2, TL_TURN = 3, TL_SCAN = 4, TL_SCATTER = 5,
       TL_SLOTS = 8 };
// Programmatic dependent launch (kernels launched with launch_pdl): the
// dependent grid is scheduled while this one drains; it waits for this grid's
// completion and memory before touching its outputs.  No-ops otherwise.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ unsigned long long *d_timeline = nullptr;   // (one translation unit)
__device__ __forceinline__ unsigned long long tl_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void tl_start(int slot) {
    unsigned long long *t = d_timeline;
    if (t && threadIdx.x == 0) atomicMin(t + 2 * slot, tl_now());
}
__device__ __forceinline__ void tl_end(int slot) {
    unsigned long long *t = d_timeline;
    if (t && threadIdx.x == 0) atomicMax(t + 2 * slot + 1, tl_now());
}
__device__ __forceinline__ void tl_end_warp(int slot) {
    unsigned long long *t = d_timeline;
    if (t && (threadIdx.x & 31) == 0) atomicMax(t + 2 * slot + 1, tl_now());
}

}  // namespace glm

namespace glm {
// <<<grid, block, smem, s>>> with the programmatic-stream-serialization
// attribute when `pdl`: the kernel may be scheduled before its stream
// predecessor has drained (it must call pdl_wait() before reading that
// kernel's outputs).  Captured graphs keep it as a programmatic edge.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block,
                              size_t smem, cudaStream_t s, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = pdl ? attr : nullptr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
}  // namespace glm

#define GLM_CUDA_TRY(expr)                                                   \
    do {                                                                     \
        cudaError_t _e = (expr);                                             \
        if (_e != cudaSuccess) return glm_set_cuda_error(_e, #expr, __FILE__, __LINE__); \
    } while (0)

int glm_set_cuda_error(cudaError_t e, const char *what, const char *file, int line);
int glm_set_error(int code, const char *msg);
