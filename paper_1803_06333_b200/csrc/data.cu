// data.cu — device data layer (sm_100a): column norms, SpMV both ways,
// bit-exact layout transforms and validation.
//
// Reference: SparseColumnMatrix (data.py:42-187) and the layout contract of
// load_training_data (cli.py:146-185).  Index arrays produced here are
// bit-identical to the reference's (tests/test_gpu_data.py); the only library
// call is CUB's stable radix sort for the one-time transpose (the reference's
// np.argsort(rows, kind="stable"), data.py:157).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "solver.cuh"

namespace glm {

// 128-bit accesses over [lo, hi) of an f64 array by `width` cooperating lanes:
// a scalar head up to 16-byte alignment, a double2 body, a scalar tail;
// f(q, x) for every element (each element exactly once).
template <class F>
__device__ __forceinline__ void span_f64(const double *a, int64_t lo, int64_t hi, int lane,
                                         int width, F f) {
    int64_t q = lo;
    if (q < hi && (reinterpret_cast<uintptr_t>(a + q) & 15)) {
        if (lane == 0) f(q, __ldg(a + q));
        ++q;
    }
    const int64_t np = (hi - q) >> 1;
    const double2 *a2 = reinterpret_cast<const double2 *>(a + q);
    for (int64_t t = lane; t < np; t += width) {
        const double2 v = __ldg(a2 + t);
        f(q + 2 * t, v.x);
        f(q + 2 * t + 1, v.y);
    }
    if (q + 2 * np < hi && lane == width - 1) f(hi - 1, __ldg(a + hi - 1));
}

template <int G, bool DENSE>
__global__ void __launch_bounds__(256) colwise_kernel(int op, int64_t n, int64_t d,
                                                      const int64_t *indptr,
                                                      const int32_t *rows, const double *vals,
                                                      const double *w, double *out) {
    // op 0: out[j] = sum vals^2 (col_sqnorms); op 1: out[j] = a_j . w (rmatvec)
    constexpr int GPW = 32 / G;
    const int lane = threadIdx.x & 31, sub = lane / G, gl = lane % G;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t jb = warp * GPW; jb < n; jb += nwarps * GPW) {
        const int64_t j = jb + sub;
        const bool valid = j < n;
        int64_t lo = 0, hi = 0;
        if (valid) {
            if (DENSE) { lo = j * d; hi = lo + d; }
            else { lo = indptr[j]; hi = indptr[j + 1]; }
        }
        double acc = 0.0;
        span_f64(vals, lo, hi, gl, G, [&](int64_t q, double x) {
            if (op == 0) acc += x * x;
            else acc += x * w[DENSE ? (int)(q - lo) : __ldg(rows + q)];
        });
        acc = group_sum<G>(acc);
        if (valid && gl == 0) out[j] = acc;
    }
}

// out = A x (matvec, data.py:109-114): scatter with atomics (order-free).
template <int G, bool DENSE>
__global__ void __launch_bounds__(256) matvec_kernel(int64_t n, int64_t d, const int64_t *indptr,
                                                     const int32_t *rows, const double *vals,
                                                     const double *x, double *out) {
    constexpr int GPW = 32 / G;
    const int lane = threadIdx.x & 31, sub = lane / G, gl = lane % G;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t jb = warp * GPW; jb < n; jb += nwarps * GPW) {
        const int64_t j = jb + sub;
        if (j >= n) continue;
        const double xj = x[j];
        if (xj == 0.0) continue;
        int64_t lo, hi;
        if (DENSE) { lo = j * d; hi = lo + d; }
        else { lo = indptr[j]; hi = indptr[j + 1]; }
        for (int64_t q = lo + gl; q < hi; q += G)
            red_add(out + (DENSE ? (int)(q - lo) : rows[q]), vals[q] * xj);
    }
}

__global__ void zero_kernel(double *p, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = 0.0;
}

static int lanes_for(double avg) {
    if (avg <= 12) return 4;
    if (avg <= 24) return 8;
    if (avg <= 64) return 16;
    return 32;
}

static double avg_nnz(const glm_matrix *A) {
    if (A->layout == GLM_DENSE) return (double)A->n_rows;
    return A->n_cols ? (double)A->nnz / (double)A->n_cols : 0.0;
}

static int blocks_for_groups(int64_t n, int G) {
    int64_t b = (n * G + 255) / 256;
    if (b < 1) b = 1;
    if (b > 16 * NUM_SMS) b = 16 * NUM_SMS;
    return (int)b;
}

int launch_colwise(const glm_matrix *A, int op, const double *w, double *out, cudaStream_t s) {
    if (A->n_cols <= 0) return GLM_OK;
    const bool dense = A->layout == GLM_DENSE;
    const int G = lanes_for(avg_nnz(A));
    const int grid = blocks_for_groups(A->n_cols, G);
#define CW(GG)                                                                                 \
    (dense ? colwise_kernel<GG, true><<<grid, 256, 0, s>>>(op, A->n_cols, A->n_rows, A->indptr, \
                                                           A->rows, A->vals, w, out)            \
           : colwise_kernel<GG, false><<<grid, 256, 0, s>>>(op, A->n_cols, A->n_rows,           \
                                                            A->indptr, A->rows, A->vals, w, out))
    count_launch();
    switch (G) {
    case 4: CW(4); break;
    case 8: CW(8); break;
    case 16: CW(16); break;
    default: CW(32); break;
    }
#undef CW
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

int launch_matvec(const glm_matrix *A, const double *x, double *out, cudaStream_t s) {
    count_launch();
    zero_kernel<<<4 * NUM_SMS, 256, 0, s>>>(out, A->n_rows);
    if (A->n_cols <= 0) return GLM_OK;
    const bool dense = A->layout == GLM_DENSE;
    const int G = lanes_for(avg_nnz(A));
    const int grid = blocks_for_groups(A->n_cols, G);
#define MV(GG)                                                                                 \
    (dense ? matvec_kernel<GG, true><<<grid, 256, 0, s>>>(A->n_cols, A->n_rows, A->indptr,      \
                                                          A->rows, A->vals, x, out)             \
           : matvec_kernel<GG, false><<<grid, 256, 0, s>>>(A->n_cols, A->n_rows, A->indptr,     \
                                                           A->rows, A->vals, x, out))
    count_launch();
    switch (G) {
    case 4: MV(4); break;
    case 8: MV(8); break;
    case 16: MV(16); break;
    default: MV(32); break;
    }
#undef MV
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

// ------------------------------------------------------------- transpose
__global__ void expand_cols_kernel(const int64_t *indptr, int64_t n, int32_t *col_of,
                                   uint32_t *keys, const int32_t *rows, int32_t *pos,
                                   int64_t nnz) {
    // a warp per column writes its column id over its entries (coalesced)
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = warp; j < n; j += nwarps) {
        const int64_t lo = __ldg(indptr + j), hi = __ldg(indptr + j + 1);
        for (int64_t q = lo + lane; q < hi; q += 32) col_of[q] = (int32_t)j;
    }
    // keys = rows, pos = iota: 128-bit loads and stores (the arrays are
    // allocation-aligned), scalar tail
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int64_t n4 = nnz >> 2;
    const int4 *r4 = reinterpret_cast<const int4 *>(rows);
    for (int64_t t = tid; t < n4; t += nth) {
        const int4 r = __ldg(r4 + t);
        reinterpret_cast<uint4 *>(keys)[t] = make_uint4((uint32_t)r.x, (uint32_t)r.y,
                                                         (uint32_t)r.z, (uint32_t)r.w);
        const int32_t q = (int32_t)(4 * t);
        reinterpret_cast<int4 *>(pos)[t] = make_int4(q, q + 1, q + 2, q + 3);
    }
    for (int64_t q = 4 * n4 + tid; q < nnz; q += nth) {
        keys[q] = (uint32_t)rows[q];
        pos[q] = (int32_t)q;
    }
}

__global__ void row_count_kernel(const int32_t *rows, int64_t nnz, int64_t *counts) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int64_t n4 = nnz >> 2;          // rows is allocation-aligned: int4 loads
    auto add = [&](int32_t r) {
        atomicAdd(reinterpret_cast<unsigned long long *>(counts + r + 1), 1ULL);
    };
    for (int64_t t = tid; t < n4; t += nth) {
        const int4 r = __ldg(reinterpret_cast<const int4 *>(rows) + t);
        add(r.x);
        add(r.y);
        add(r.z);
        add(r.w);
    }
    for (int64_t q = 4 * n4 + tid; q < nnz; q += nth) add(rows[q]);
}

__global__ void zero_i64_kernel(int64_t *p, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = 0;
}

__global__ void permute_out_kernel(const int32_t *order, const int32_t *col_of,
                                   const double *vals, int64_t nnz, int32_t *rows_t,
                                   double *vals_t) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int32_t o = order[q];
        rows_t[q] = col_of[o];
        vals_t[q] = vals[o];
    }
}

static int bits_for(int64_t n) {
    int b = 1;
    while ((1LL << b) < n) ++b;
    return b;
}

struct TransposeScratch {
    int32_t *col_of;
    uint32_t *keys, *keys_out;
    int32_t *pos, *order;
    void *cub;
    size_t cub_bytes;
};

static size_t cub_sort_bytes(int64_t nnz, int64_t n_rows) {
    size_t b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (int32_t *)nullptr, (int32_t *)nullptr,
                                    (int)(nnz > 0 ? nnz : 1), 0, bits_for(n_rows));
    size_t b2 = 0;
    cub::DeviceScan::InclusiveSum(nullptr, b2, (int64_t *)nullptr, (int64_t *)nullptr,
                                  (int)(n_rows + 1));
    return b > b2 ? b : b2;
}

size_t transpose_temp_bytes(int64_t nnz, int64_t n_rows) {
    size_t e = (size_t)(nnz > 0 ? nnz : 1);
    return e * (4 * 5) + cub_sort_bytes(nnz, n_rows) + 6 * 256;
}

static TransposeScratch carve_t(void *base, int64_t nnz, int64_t n_rows, size_t total) {
    TransposeScratch t;
    size_t e = (size_t)(nnz > 0 ? nnz : 1);
    char *c = (char *)base;
    auto take = [&](size_t bytes) {
        char *r = c;
        c += (bytes + 255) & ~(size_t)255;
        return r;
    };
    t.col_of = (int32_t *)take(4 * e);
    t.keys = (uint32_t *)take(4 * e);
    t.keys_out = (uint32_t *)take(4 * e);
    t.pos = (int32_t *)take(4 * e);
    t.order = (int32_t *)take(4 * e);
    t.cub = c;
    size_t used = (size_t)(c - (char *)base);
    t.cub_bytes = total > used ? total - used : 0;
    (void)n_rows;
    return t;
}

int launch_transpose(const glm_matrix *A, int64_t *indptr_t, int32_t *rows_t, double *vals_t,
                     void *temp, size_t temp_bytes, cudaStream_t s) {
    if (A->layout != GLM_CSC) return glm_set_error(GLM_USAGE, "transpose needs CSC");
    const int64_t nnz = A->nnz, n = A->n_cols, R = A->n_rows;
    if (nnz >= (1LL << 31)) return glm_set_error(GLM_USAGE, "transpose: nnz >= 2^31");
    if (temp_bytes < transpose_temp_bytes(nnz, R))
        return glm_set_error(GLM_USAGE, "transpose scratch too small");
    TransposeScratch t = carve_t(temp, nnz, R, temp_bytes);
    const int grid = 8 * NUM_SMS;
    count_launch();
    zero_i64_kernel<<<grid, 256, 0, s>>>(indptr_t, R + 1);
    if (nnz > 0) {
        count_launch();
        expand_cols_kernel<<<grid, 256, 0, s>>>(A->indptr, n, t.col_of, t.keys, A->rows, t.pos,
                                                nnz);
        size_t cb = t.cub_bytes;
        GLM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(t.cub, cb, t.keys, t.keys_out, t.pos, t.order,
                                                     (int)nnz, 0, bits_for(R), s));
        count_launch();
        permute_out_kernel<<<grid, 256, 0, s>>>(t.order, t.col_of, A->vals, nnz, rows_t, vals_t);
        count_launch();
        row_count_kernel<<<grid, 256, 0, s>>>(A->rows, nnz, indptr_t);
        cb = t.cub_bytes;
        GLM_CUDA_TRY(cub::DeviceScan::InclusiveSum(t.cub, cb, indptr_t, indptr_t, (int)(R + 1), s));
    }
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

// ---------------------------------------------------------- select/scale
__global__ void select_counts_kernel(const int64_t *indptr, const int64_t *cols, int64_t k,
                                     int64_t *out_indptr) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= k;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i == 0) out_indptr[0] = 0;
        else {
            const int64_t j = cols[i - 1];
            out_indptr[i] = indptr[j + 1] - indptr[j];
        }
    }
}

int launch_select_indptr(const glm_matrix *A, const int64_t *cols, int64_t k,
                         int64_t *out_indptr, void *temp, size_t temp_bytes, cudaStream_t s) {
    count_launch();
    select_counts_kernel<<<4 * NUM_SMS, 256, 0, s>>>(A->indptr, cols, k, out_indptr);
    size_t cb = temp_bytes;
    GLM_CUDA_TRY(cub::DeviceScan::InclusiveSum(temp, cb, out_indptr, out_indptr, (int)(k + 1), s));
    return GLM_OK;
}

size_t select_temp_bytes(int64_t k) {
    size_t b = 0;
    cub::DeviceScan::InclusiveSum(nullptr, b, (int64_t *)nullptr, (int64_t *)nullptr,
                                  (int)(k + 1));
    return b + 256;
}

__global__ void select_gather_kernel(const int64_t *indptr, const int32_t *rows,
                                     const double *vals, const int64_t *cols, int64_t k,
                                     const int64_t *out_indptr, int32_t *out_rows,
                                     double *out_vals) {
    // warp per selected column
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < k; i += nwarps) {
        const int64_t j = cols[i];
        const int64_t lo = indptr[j], hi = indptr[j + 1], o = out_indptr[i];
        for (int64_t q = lo + lane; q < hi; q += 32) {
            out_rows[o + q - lo] = rows[q];
            out_vals[o + q - lo] = vals[q];
        }
    }
}

int launch_select_gather(const glm_matrix *A, const int64_t *cols, int64_t k,
                         const int64_t *out_indptr, int32_t *out_rows, double *out_vals,
                         cudaStream_t s) {
    if (k <= 0) return GLM_OK;
    count_launch();
    select_gather_kernel<<<8 * NUM_SMS, 256, 0, s>>>(A->indptr, A->rows, A->vals, cols, k,
                                                     out_indptr, out_rows, out_vals);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

__global__ void scale_kernel(const int64_t *indptr, int64_t n, int64_t d, int dense,
                             const double *vals, const double *scales, double *out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // 128-bit loads and stores when vals and out share their 16-byte phase
    const bool paired = ((reinterpret_cast<uintptr_t>(vals) ^ reinterpret_cast<uintptr_t>(out)) &
                         15) == 0;
    for (int64_t j = warp; j < n; j += nwarps) {
        const int64_t lo = dense ? j * d : indptr[j], hi = dense ? lo + d : indptr[j + 1];
        const double sc = scales[j];
        if (!paired) {
            for (int64_t q = lo + lane; q < hi; q += 32) out[q] = vals[q] * sc;
            continue;
        }
        int64_t q = lo;
        if (q < hi && (reinterpret_cast<uintptr_t>(vals + q) & 15)) {
            if (lane == 0) out[q] = vals[q] * sc;
            ++q;
        }
        const int64_t np = (hi - q) >> 1;
        const double2 *v2 = reinterpret_cast<const double2 *>(vals + q);
        double2 *o2 = reinterpret_cast<double2 *>(out + q);
        for (int64_t t = lane; t < np; t += 32) {
            const double2 x = __ldg(v2 + t);
            o2[t] = make_double2(x.x * sc, x.y * sc);
        }
        if (q + 2 * np < hi && lane == 31) out[hi - 1] = vals[hi - 1] * sc;
    }
}

int launch_scale(const glm_matrix *A, const double *scales, double *out, cudaStream_t s) {
    if (A->n_cols <= 0) return GLM_OK;
    count_launch();
    scale_kernel<<<8 * NUM_SMS, 256, 0, s>>>(A->indptr, A->n_cols, A->n_rows,
                                             A->layout == GLM_DENSE, A->vals, scales, out);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

// ------------------------------------------------------------ validate
// flags: 1 indptr[0]!=0 or indptr[n]!=nnz, 2 decreasing indptr, 4 row out of
// range, 8 non-finite value, 16 rows not strictly increasing in a column
__global__ void validate_kernel(const int64_t *indptr, const int32_t *rows, const double *vals,
                                int64_t n, int64_t R, int64_t nnz, unsigned *flags) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    unsigned f = 0;
    if (tid == 0 && (indptr[0] != 0 || indptr[n] != nnz)) f |= 1;
    // a warp per column: coalesced row checks, 128-bit value loads
    const int lane = threadIdx.x & 31;
    const int64_t warp = tid >> 5, nwarps = nth >> 5;
    for (int64_t j = warp; j < n; j += nwarps) {
        const int64_t lo = indptr[j], hi = indptr[j + 1];
        if (hi < lo) { f |= 2; continue; }
        if (lo < 0 || hi > nnz) { f |= 1; continue; }
        for (int64_t q = lo + lane; q < hi; q += 32) {
            const int32_t r = rows[q];
            if (r < 0 || r >= R) f |= 4;
            if (q > lo && rows[q - 1] >= r) f |= 16;
        }
        span_f64(vals, lo, hi, lane, 32, [&](int64_t, double x) {
            if (!isfinite(x)) f |= 8;
        });
    }
    if (f) atomicOr(flags, f);
}

int launch_validate(const glm_matrix *A, unsigned *flags_dev, cudaStream_t s) {
    count_launch();
    validate_kernel<<<8 * NUM_SMS, 256, 0, s>>>(A->indptr, A->rows, A->vals, A->n_cols,
                                                A->n_rows, A->nnz, flags_dev);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

}  // namespace glm
