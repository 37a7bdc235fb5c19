// objective.cu — fused objective, duality-gap, engine-glue and prediction
// kernels (sm_100a).  All reductions are deterministic: a fixed grid writes
// per-block partials and the last block to finish folds them in block order.
//
// Reference: objectives.py:129-234 (f, f', f*, g, g*, gap), engine.py:131-166
// (sub-problem models), engine.py:325-351 (objective_and_gap), modelio.py:57-99
// (scores, sigmoid, log-loss, accuracy, mse), solver.py:152-187 (steps).
#include "solver.cuh"

namespace glm {

constexpr int RED_BLOCKS = 2 * NUM_SMS;
constexpr int RED_THREADS = 256;
// column passes (gap part B, predict) are gather-latency bound: one wave of
// as many resident CTAs as the kernel's registers allow keeps the most
// columns in flight (the reduction scratch holds up to 4096 CTA partials)
template <class K>
static int full_grid(K kernel) {
    static const int grid = [kernel] {        // thread-safe once-only initialisation
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, RED_THREADS, 0) !=
                cudaSuccess || per_sm < 1)
            per_sm = 2;
        return (per_sm > 8 ? 8 : per_sm) * NUM_SMS;
    }();
    return grid;
}

// scratch layout: [u32 counter | pad 16B][partials RED_BLOCKS x NV]
template <int NV>
__device__ __forceinline__ bool reduce_last(double (&v)[NV], double *scratch) {
    __shared__ double sm[32 * NV];
    __shared__ int s_last;
    block_sum<NV>(v, sm);
    unsigned *counter = reinterpret_cast<unsigned *>(scratch);
    double *parts = scratch + 2;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) parts[blockIdx.x * NV + i] = v[i];
        __threadfence();
        s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return false;
    __threadfence();
    double tot[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) tot[i] = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
#pragma unroll
        for (int i = 0; i < NV; ++i) tot[i] += __ldcg(parts + b * NV + i);
    }
    block_sum<NV>(tot, sm);
    if (threadIdx.x == 0) {
        *counter = 0;
#pragma unroll
        for (int i = 0; i < NV; ++i) v[i] = tot[i];
        return true;
    }
    return false;
}

// f_eval + f_grad fused (objectives.py:129-139)
__global__ void __launch_bounds__(RED_THREADS) fgrad_kernel(int kind, double lam,
                                                            const double *tgt, const double *v,
                                                            int64_t d, double *grad,
                                                            double *out_fv, double *scratch) {
    double acc[1] = {0.0};
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const bool dual = kind_is_dual(kind);
    for (int64_t r = tid; r < d; r += nth) {
        const double x = v[r];
        if (dual) {
            acc[0] += x * x;
            if (grad) grad[r] = x / lam;
        } else if (kind == GLM_LOGISTIC_PRIMAL) {
            const double y = tgt[r];
            acc[0] += softplus(-y * x);
            if (grad) grad[r] = -y * sigmoid_tanh(-y * x);
        } else if (kind == GLM_HINGE_PRIMAL) {
            double f, g;
            f_terms(kind, lam, tgt[r], x, f, g);
            acc[0] += f;
            if (grad) grad[r] = g;
        } else if (kind == GLM_SQUARED_HINGE_PRIMAL) {
            const double y = tgt[r], mg = 1.0 - y * x;
            acc[0] += mg > 0.0 ? mg * mg : 0.0;
            if (grad) grad[r] = mg > 0.0 ? -y * mg : 0.0;
        } else {
            const double e = x - tgt[r];
            acc[0] += e * e;
            if (grad) grad[r] = e;
        }
    }
    if (reduce_last<1>(acc, scratch)) {
        double f = acc[0];
        if (dual) f = f / (2.0 * lam);
        else if (f_halved(kind)) f = 0.5 * f;
        *out_fv = f;
    }
}

// Outer model at the start of a round fused with the first inner model
// (engine.py:271-272, 242-250, 148-166 with v_bar = 0): grad = f'(v),
// lin = grad, fv = f(v), cnst = f(v) / (K L).
__global__ void __launch_bounds__(RED_THREADS) outer_model_kernel(int kind, double lam,
                                                                  const double *tgt,
                                                                  const double *v, int64_t d,
                                                                  double *grad, double *lin,
                                                                  double *out_fv, double *cnst,
                                                                  double K, double L,
                                                                  double *scratch) {
    double acc[1] = {0.0};
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const bool dual = kind_is_dual(kind);
    for (int64_t r = tid; r < d; r += nth) {
        const double x = v[r];
        double f, g;
        if (dual) {
            f = x * x;
            g = x / lam;
        } else {
            f_terms(kind, lam, tgt[r], x, f, g);
            if (f_halved(kind)) f *= 2.0;   // raw square, halved below
        }
        acc[0] += f;
        grad[r] = g;
        lin[r] = g;
    }
    if (reduce_last<1>(acc, scratch)) {
        double f = acc[0];
        if (dual) f = f / (2.0 * lam);
        else if (f_halved(kind)) f = 0.5 * f;
        *out_fv = f;
        *cnst = (f / K + 0.0) / L;   // ((fv/K) + grad.0 + 0)/L as engine.py:156-162
    }
}

// build_inner_subproblem (engine.py:148-166) with the outer model folded in
// (engine.py:242-250): lin = grad + qo*vbar; cnst = (fv/K + grad.vbar + qo/2 |vbar|^2)/L
__global__ void __launch_bounds__(RED_THREADS) inner_model_kernel(
    const double *grad, const double *vbar, int64_t d, double qo, const double *fv, double K,
    double L, double *lin, double *cnst, double *scratch) {
    double acc[2] = {0.0, 0.0};
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = tid; r < d; r += nth) {
        const double g = grad[r], b = vbar ? vbar[r] : 0.0;
        lin[r] = g + qo * b;
        acc[0] += g * b;
        acc[1] += b * b;
    }
    if (reduce_last<2>(acc, scratch)) *cnst = (*fv / K + acc[0] + 0.5 * qo * acc[1]) / L;
}

__global__ void axpby_kernel(int64_t n, double a, const double *x, double b, double *y) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < n; i += nth) y[i] = (b == 0.0 ? 0.0 : b * y[i]) + a * x[i];
}

// gap part A over the rows: w = f'(v); f(v) and f*(w) (objectives.py:223-234)
__global__ void __launch_bounds__(RED_THREADS) gap_rows_kernel(int kind, double lam,
                                                               const double *tgt,
                                                               const double *v, int64_t d,
                                                               double *w, double *out,
                                                               double *scratch) {
    double acc[2] = {0.0, 0.0};
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = tid; r < d; r += nth) {
        double f, g;
        const double y = tgt ? tgt[r] : 0.0;
        f_terms(kind, lam, y, v[r], f, g);
        w[r] = g;
        acc[0] += f;
        acc[1] += f_conj_term(kind, lam, y, g);
    }
    if (reduce_last<2>(acc, scratch)) {
        out[0] = acc[0] + acc[1];
        out[3] = acc[0];
    }
}

// a_j.w by the G lanes of a column group: each lane takes every G-th entry;
// U entries per lane are loaded (indices, values, then the gathers) before
// any is added, in the same order as a plain strided loop.
template <int G, bool DENSE, int U = 4>
__device__ __forceinline__ double column_dot(int64_t lo, int64_t hi, int gl, const int32_t *rows,
                                             const double *vals, const double *w) {
    double dot = 0.0;
    for (int64_t q0 = lo + gl; q0 < hi; q0 += U * G) {
        int r[U];
        double a[U], x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t q = q0 + (int64_t)u * G;
            r[u] = q < hi ? (DENSE ? (int)(q - lo) : __ldg(rows + q)) : -1;
            a[u] = q < hi ? __ldg(vals + q) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = r[u] >= 0 ? w[r[u]] : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (r[u] >= 0) dot += a[u] * x[u];
    }
    return group_sum<G>(dot);
}

// One warp, 32 consecutive columns cb..cb+31: lane L loads the bounds of
// column cb+L (coalesced), the G-lane groups take the columns GPW at a time
// (bounds handed over by shuffles, no dependent indptr load per column), and
// every dot lands in the lane of its column, so the per-column epilogue
// (transcendentals, loads of alpha / labels) runs on all 32 lanes.
template <int G, bool DENSE, int U = 4>
__device__ __forceinline__ double warp_column_dots(int64_t cb, int64_t n, int64_t d,
                                                   const int64_t *indptr, const int32_t *rows,
                                                   const double *vals, const double *w) {
    constexpr int GPW = 32 / G;
    const int lane = threadIdx.x & 31, sub = lane / G, gl = lane % G;
    int64_t mlo = 0, mhi = 0;
    const int64_t jm = cb + lane;
    if (jm < n) {
        if (DENSE) { mlo = jm * d; mhi = mlo + d; }
        else { mlo = __ldg(indptr + jm); mhi = __ldg(indptr + jm + 1); }
    }
    double mine = 0.0;
#pragma unroll 4
    for (int it = 0; it < G; ++it) {
        const int src = it * GPW + sub;
        const int64_t lo = __shfl_sync(0xffffffffu, mlo, src);
        const int64_t hi = __shfl_sync(0xffffffffu, mhi, src);
        const double dot = column_dot<G, DENSE, U>(lo, hi, gl, rows, vals, w);
        const double v = __shfl_sync(0xffffffffu, dot, (lane % GPW) * G);
        if (lane / GPW == it) mine = v;
    }
    return mine;
}

// gap part B over the columns: s_j = -a_j.w; g(alpha_j) + g*(s_j)
template <int G, bool DENSE, int U = 4>
__global__ void __launch_bounds__(RED_THREADS) gap_cols_kernel(
    int kind, double lam, double rho, const double *y, int64_t n, int64_t d,
    const int64_t *indptr, const int32_t *rows, const double *vals, const double *alpha,
    const double *w, double *out, double *scratch) {
    double acc[2] = {0.0, 0.0};
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t cb = warp * 32; cb < n; cb += nwarps * 32) {
        const double dot = warp_column_dots<G, DENSE, U>(cb, n, d, indptr, rows, vals, w);
        const int64_t j = cb + lane;
        if (j < n) {
            const double yj = y ? y[j] : 0.0;
            acc[0] += g_one(kind, lam, rho, yj, alpha[j]);
            acc[1] += g_conj_one(kind, lam, rho, yj, -dot);
        }
    }
    if (reduce_last<2>(acc, scratch)) {
        out[1] = acc[0];
        out[2] = acc[1];
    }
}

__global__ void __launch_bounds__(RED_THREADS) gsum_kernel(int kind, double lam, double rho,
                                                           const double *y, const double *a,
                                                           int64_t n, double *out,
                                                           double *scratch) {
    double acc[1] = {0.0};
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < n; i += nth) acc[0] += g_one(kind, lam, rho, y ? y[i] : 0.0, a[i]);
    if (reduce_last<1>(acc, scratch)) *out = acc[0];
}

// decision_scores / sigmoid / log_loss / accuracy / mse (modelio.py:64-99)
template <int G, bool DENSE>
__global__ void __launch_bounds__(RED_THREADS) predict_kernel(
    int64_t n, int64_t d, const int64_t *indptr, const int32_t *rows, const double *vals,
    const double *w, const double *y, int classify, double *scores, double *prob, double *out,
    double *scratch) {
    double acc[3] = {0.0, 0.0, 0.0};
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t cb = warp * 32; cb < n; cb += nwarps * 32) {
        const double dot = warp_column_dots<G, DENSE>(cb, n, d, indptr, rows, vals, w);
        const int64_t j = cb + lane;
        if (j < n) {
            if (scores) scores[j] = dot;
            if (classify) {
                const double p = sigmoid_tanh(dot);
                if (prob) prob[j] = p;
                if (y) {
                    const double y01 = y[j] > 0.0 ? 1.0 : 0.0;
                    const double pc = fmin(fmax(p, 1e-15), 1.0 - 1e-15);
                    acc[0] += y01 * log(pc) + (1.0 - y01) * log(1.0 - pc);
                    acc[1] += ((p >= 0.5) == (y01 > 0.5)) ? 1.0 : 0.0;
                }
            } else if (y) {
                const double e = dot - y[j];
                acc[2] += e * e;
            }
        }
    }
    if (reduce_last<3>(acc, scratch)) {
        out[0] = -acc[0];
        out[1] = acc[1];
        out[2] = acc[2];
    }
}

__global__ void coord_steps_kernel(int kind, double lam, double rho, const double *y,
                                   const double *ga, const double *c, const double *t,
                                   int64_t n, double *step, int *err) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < n; i += nth) {
        double s = 0.0;
        if (!coord_step(kind, lam, rho, y ? y[i] : 0.0, ga[i], c[i], t[i], s)) {
            atomicExch(err, 1);
            s = NAN;
        }
        step[i] = s;
    }
}

static int pick_lanes(double avg) {
    if (avg <= 12) return 4;
    if (avg <= 24) return 8;
    if (avg <= 64) return 16;
    return 32;
}

int launch_gap(const glm_matrix *A, int kind, double lam, double rho, const double *tgt,
               const double *y, const double *alpha, const double *v, double *w, double *out,
               double *scratch, cudaStream_t s) {
    count_launch();
    gap_rows_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(kind, lam, tgt, v, A->n_rows, w, out,
                                                       scratch);
    const bool dense = A->layout == GLM_DENSE;
    const double avg = dense ? (double)A->n_rows
                             : (A->n_cols ? (double)A->nnz / (double)A->n_cols : 0.0);
#define GAPL(G)                                                                               \
    (dense ? gap_cols_kernel<G, true><<<full_grid(gap_cols_kernel<G, true>), RED_THREADS, 0, s>>>( \
                 kind, lam, rho, y, A->n_cols, A->n_rows, A->indptr, A->rows, A->vals, alpha, \
                 w, out, scratch)                                                             \
           : gap_cols_kernel<G, false><<<full_grid(gap_cols_kernel<G, false>), RED_THREADS, 0, s>>>( \
                 kind, lam, rho, y, A->n_cols, A->n_rows, A->indptr, A->rows, A->vals, alpha, \
                 w, out, scratch))
    count_launch();
    if (!dense && avg > 12 && avg <= 48) {
        // ~40-nnz columns (C2, C5): 4 lanes x 12 entries each, so a warp has
        // 8 columns' gathers in flight at once instead of 2
        gap_cols_kernel<4, false, 12><<<full_grid(gap_cols_kernel<4, false, 12>), RED_THREADS, 0,
                                        s>>>(kind, lam, rho, y, A->n_cols, A->n_rows, A->indptr,
                                             A->rows, A->vals, alpha, w, out, scratch);
    } else {
        switch (pick_lanes(avg)) {
        case 4: GAPL(4); break;
        case 8: GAPL(8); break;
        case 16: GAPL(16); break;
        default: GAPL(32); break;
        }
    }
#undef GAPL
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

int launch_predict(const glm_matrix *X, const double *w, const double *y, int classify,
                   double *scores, double *prob, double *out, double *scratch, cudaStream_t s) {
    const bool dense = X->layout == GLM_DENSE;
    const double avg = dense ? (double)X->n_rows
                             : (X->n_cols ? (double)X->nnz / (double)X->n_cols : 0.0);
#define PRL(G)                                                                                 \
    (dense ? predict_kernel<G, true><<<full_grid(predict_kernel<G, true>), RED_THREADS, 0, s>>>( \
                 X->n_cols, X->n_rows, X->indptr, X->rows, X->vals, w, y, classify, scores,    \
                 prob, out, scratch)                                                           \
           : predict_kernel<G, false><<<full_grid(predict_kernel<G, false>), RED_THREADS, 0, s>>>( \
                 X->n_cols, X->n_rows, X->indptr, X->rows, X->vals, w, y, classify, scores,    \
                 prob, out, scratch))
    count_launch();
    switch (pick_lanes(avg)) {
    case 4: PRL(4); break;
    case 8: PRL(8); break;
    case 16: PRL(16); break;
    default: PRL(32); break;
    }
#undef PRL
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

}  // namespace glm
