// api.cu — extern "C" entry points of libglm_b200.so (include/glm_b200.h).
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <new>
#include <vector>

#include "solver.cuh"

namespace glm {
int launch_colwise(const glm_matrix *A, int op, const double *w, double *out, cudaStream_t s);
int launch_matvec(const glm_matrix *A, const double *x, double *out, cudaStream_t s);
size_t transpose_temp_bytes(int64_t nnz, int64_t n_rows);
int launch_transpose(const glm_matrix *A, int64_t *indptr_t, int32_t *rows_t, double *vals_t,
                     void *temp, size_t temp_bytes, cudaStream_t s);
size_t select_temp_bytes(int64_t k);
int launch_select_indptr(const glm_matrix *A, const int64_t *cols, int64_t k,
                         int64_t *out_indptr, void *temp, size_t temp_bytes, cudaStream_t s);
int launch_select_gather(const glm_matrix *A, const int64_t *cols, int64_t k,
                         const int64_t *out_indptr, int32_t *out_rows, double *out_vals,
                         cudaStream_t s);
int launch_scale(const glm_matrix *A, const double *scales, double *out, cudaStream_t s);
int launch_validate(const glm_matrix *A, unsigned *flags_dev, cudaStream_t s);
int launch_gap(const glm_matrix *A, int kind, double lam, double rho, const double *tgt,
               const double *y, const double *alpha, const double *v, double *w, double *out,
               double *scratch, cudaStream_t s);
int launch_predict(const glm_matrix *X, const double *w, const double *y, int classify,
                   double *scores, double *prob, double *out, double *scratch, cudaStream_t s);
}  // namespace glm

using namespace glm;

static thread_local char g_err[1024] = "";
static std::atomic<long long> g_launches{0};

namespace glm {
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace glm

int glm_set_error(int code, const char *msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}

int glm_set_cuda_error(cudaError_t e, const char *what, const char *file, int line) {
    snprintf(g_err, sizeof(g_err), "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
             cudaGetErrorString(e), what, file, line);
    return GLM_CUDA_ERROR;
}

#define S(x) ((cudaStream_t)(x))

extern "C" {

const char *glm_last_error(void) { return g_err; }

int glm_version(void) { return 1; }

long long glm_launch_count(void) { return g_launches.load(); }

int glm_solver_timing(glm_solver *s, int enable) {
    if (!s) return glm_set_error(GLM_USAGE, "null solver");
    s->timing = enable;
    return GLM_OK;
}

static int timing_sum(glm_solver *s, double *ms_out, int32_t *n_out, bool consume) {
    if (!s) return glm_set_error(GLM_USAGE, "null solver");
    double acc[3] = {0.0, 0.0, 0.0};
    int n = 0;
    for (auto &ev : s->events) {
        GLM_CUDA_TRY(cudaEventSynchronize(ev[3]));
        float a = 0.f, b = 0.f, c = 0.f;
        GLM_CUDA_TRY(cudaEventElapsedTime(&a, ev[0], ev[1]));
        GLM_CUDA_TRY(cudaEventElapsedTime(&b, ev[1], ev[2]));
        GLM_CUDA_TRY(cudaEventElapsedTime(&c, ev[2], ev[3]));
        acc[0] += a;
        acc[1] += b;
        acc[2] += c;
        ++n;
    }
    if (consume) {
        for (auto &ev : s->events) s->event_pool.push_back(ev);
        s->events.clear();
    }
    if (ms_out) { ms_out[0] = acc[0]; ms_out[1] = acc[1]; ms_out[2] = acc[2]; }
    if (n_out) *n_out = n;
    return GLM_OK;
}

int glm_solver_timing_read(glm_solver *s, double *ms_out, int32_t *n_out) {
    return timing_sum(s, ms_out, n_out, true);
}

int glm_solver_timing_peek(glm_solver *s, double *ms_out, int32_t *n_out) {
    return timing_sum(s, ms_out, n_out, false);
}

int glm_solver_timing_glue(glm_solver *s, double *ms_out, int32_t *n_out, int consume) {
    if (!s) return glm_set_error(GLM_USAGE, "null solver");
    double acc[3] = {0.0, 0.0, 0.0};
    int32_t n[3] = {0, 0, 0};
    for (auto &g : s->glue_events) {
        GLM_CUDA_TRY(cudaEventSynchronize(g.second[1]));
        float t = 0.f;
        GLM_CUDA_TRY(cudaEventElapsedTime(&t, g.second[0], g.second[1]));
        acc[g.first] += t;
        n[g.first] += 1;
    }
    if (consume) {
        for (auto &g : s->glue_events) s->glue_pool.push_back(g.second);
        s->glue_events.clear();
    }
    if (ms_out) for (int i = 0; i < 3; ++i) ms_out[i] = acc[i];
    if (n_out) for (int i = 0; i < 3; ++i) n_out[i] = n[i];
    return GLM_OK;
}

// Debug timeline: kernels write earliest start / latest end %globaltimer
// stamps into device u64[2 * TL_SLOTS] (epoch, first and last permutation
// kernel, round turn); NULL turns it off.
int glm_debug_timeline(unsigned long long *device_slots) {
    GLM_CUDA_TRY(cudaMemcpyToSymbol(d_timeline, &device_slots, sizeof(device_slots)));
    return GLM_OK;
}

int glm_device_count(int *out) {
    GLM_CUDA_TRY(cudaGetDeviceCount(out));
    return GLM_OK;
}

uint64_t glm_xorshift_jump(uint64_t state, uint64_t steps) { return host_jump(state, steps); }

uint64_t glm_derive_seed(uint64_t base, const uint64_t *idx, int n_idx) {
    auto sm = [](uint64_t x) {
        x += 0x9E3779B97F4A7C15ULL;
        x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
        x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
        return x ^ (x >> 31);
    };
    uint64_t s = sm(base);
    for (int i = 0; i < n_idx; ++i) s = sm(s ^ (idx[i] + 0x632BE59BD9B4E019ULL));
    return s ? s : 0x9E3779B97F4A7C15ULL;
}

// ------------------------------------------------------------------ solver
int glm_solver_destroy(glm_solver *s) {
    if (!s) return GLM_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(s->device);
    cudaDeviceSynchronize();
    cudaFree(s->st);
    cudaFreeHost(s->st_host);
    cudaFree(s->delta[0]);
    cudaFree(s->delta[1]);
    cudaFree(s->view[0]);
    cudaFree(s->view[1]);
    cudaFree(s->perm);
    cudaFree(s->perm_b);
    cudaFree(s->perm_mem);
    cudaFree(s->partials);
    cudaFree(s->gpart);
    cudaFree(s->scratch);
    cudaFree(s->vpad);
    cudaFree(s->meta);
    if (s->side) {
        cudaStreamSynchronize(s->side);
        cudaStreamDestroy(s->side);
        cudaEventDestroy(s->ev_fork);
        cudaEventDestroy(s->ev_join);
    }
    for (auto &ev : s->events) s->event_pool.push_back(ev);
    for (auto &ev : s->event_pool)
        for (int i = 0; i < 4; ++i) cudaEventDestroy(ev[i]);
    for (auto &g : s->glue_events) s->glue_pool.push_back(g.second);
    for (auto &ev : s->glue_pool)
        for (int i = 0; i < 2; ++i) cudaEventDestroy(ev[i]);
    cudaSetDevice(prev);
    delete s;
    return GLM_OK;
}

int glm_solver_create(int device, int64_t max_coords, int64_t max_rows, glm_solver **out) {
    if (!out || max_coords < 0 || max_rows < 0) return glm_set_error(GLM_USAGE, "bad solver sizes");
    GLM_CUDA_TRY(cudaSetDevice(device));
    int rc = ensure_device_tables();
    if (rc) return rc;
    glm_solver *s = new (std::nothrow) glm_solver();
    if (!s) return glm_set_error(GLM_USAGE, "out of host memory");
    s->device = device;
    s->max_coords = max_coords;
    s->max_rows = max_rows;
    const size_t mc = (size_t)(max_coords > 0 ? max_coords : 1);
    const size_t mr = (size_t)(max_rows > 0 ? max_rows : 1);
    cudaError_t e = cudaSuccess;
    auto chk = [&](cudaError_t x) { if (x != cudaSuccess && e == cudaSuccess) e = x; };
    chk(cudaMalloc(&s->st, sizeof(SolveState)));
    chk(cudaMallocHost(&s->st_host, sizeof(SolveState)));
    chk(cudaMalloc(&s->delta[0], sizeof(double) * mc));
    chk(cudaMalloc(&s->delta[1], sizeof(double) * mc));
    chk(cudaMalloc(&s->view[0], sizeof(double) * mr));
    chk(cudaMalloc(&s->view[1], sizeof(double) * mr));
    chk(cudaMalloc(&s->perm, sizeof(int32_t) * mc));
    chk(cudaMalloc(&s->perm_b, sizeof(int32_t) * mc));
    size_t pb = perm_scratch_bytes((int64_t)mc);
    chk(cudaMalloc(&s->perm_mem, pb));
    chk(cudaMalloc(&s->partials, sizeof(double) * 3 * 8 * NUM_SMS));
    chk(cudaMalloc(&s->gpart, sizeof(double) * 16 * NUM_SMS));
    chk(cudaMalloc(&s->scratch, REDUCE_SCRATCH_BYTES));
    chk(cudaMalloc(&s->vpad, sizeof(double) * NARROW_MAX_ROWS * PAD_STRIDE));
    if (e == cudaSuccess) {
        chk(cudaMemset(s->perm_mem, 0, pb));
        chk(cudaMemset(s->scratch, 0, REDUCE_SCRATCH_BYTES));
        chk(cudaMemset(s->st, 0, sizeof(SolveState)));
        chk(cudaMemset(s->delta[0], 0, sizeof(double) * mc));
        chk(cudaMemset(s->delta[1], 0, sizeof(double) * mc));
    }
    if (e != cudaSuccess) {
        glm_solver_destroy(s);
        return glm_set_cuda_error(e, "glm_solver_create", __FILE__, __LINE__);
    }
    rc = set_state(s, 0x9E3779B97F4A7C15ULL, 1.0, 0);
    if (rc) { glm_solver_destroy(s); return rc; }
    GLM_CUDA_TRY(cudaDeviceSynchronize());
    *out = s;
    return GLM_OK;
}

// Packed per-coordinate records of a CSC partition for the async epoch kernel
// (one 16-byte load instead of the indptr pair and |a_j|^2; the records are
// static for the matrix, so this runs once, outside any captured graph).
int glm_solver_prepare(glm_solver *s, const glm_matrix *A, void *stream) {
    if (!s || !A) return glm_set_error(GLM_USAGE, "null argument");
    if (A->layout != GLM_CSC || !A->indptr || !A->sqnorms) return GLM_OK;   // dense: nothing
    if (A->n_cols > s->max_coords) return glm_set_error(GLM_USAGE, "partition too large");
    GLM_CUDA_TRY(cudaSetDevice(s->device));
    if (!s->meta)
        GLM_CUDA_TRY(cudaMalloc(&s->meta, sizeof(longlong2) * (size_t)(s->max_coords > 0 ? s->max_coords : 1)));
    const int64_t m = A->n_cols;
    if (m > 0) {
        count_launch();
        meta_build_kernel<<<grid_stride_blocks(m), 256, 0, (cudaStream_t)stream>>>(
            A->indptr, A->sqnorms, m, s->meta);
        GLM_CUDA_TRY(cudaGetLastError());
    }
    s->meta_indptr = A->indptr;
    s->meta_sq = A->sqnorms;
    s->meta_m = m;
    return GLM_OK;
}

int glm_solver_set_state(glm_solver *s, uint64_t gen_state, double damping, void *stream) {
    if (!s) return glm_set_error(GLM_USAGE, "null solver");
    return set_state(s, gen_state, damping, S(stream));
}

int glm_solve(glm_solver *s, const glm_matrix *A, const glm_solve_args *args, double *delta_out,
              double *dv_out, glm_solve_result *res, void *stream) {
    if (!s) return glm_set_error(GLM_USAGE, "null solver");
    int rc = solve(s, A, args, delta_out, dv_out, res, S(stream));
    if (rc) return rc;
    if (res && res->status != GLM_OK) {
        if (res->status == GLM_DIVERGENCE)
            glm_set_error(GLM_DIVERGENCE, "damping floor reached without subproblem decrease");
        else
            glm_set_error(res->status, "non-finite entries in shared view or coordinate update");
        return res->status;
    }
    return GLM_OK;
}

int glm_solver_join(glm_solver *s, void *stream) {
    if (!s) return glm_set_error(GLM_USAGE, "null solver");
    return join_prefetch(s, S(stream));
}

int glm_solver_result(glm_solver *s, glm_solve_result *res, double *epoch_values, int capacity,
                      void *stream) {
    if (!s) return glm_set_error(GLM_USAGE, "null solver");
    return read_result(s, res, epoch_values, capacity, S(stream));
}

// ------------------------------------------------------------ permutations
int glm_perm_keys(uint64_t state, int64_t n, uint32_t *keys, void *stream) {
    int rc = ensure_device_tables();
    if (rc) return rc;
    return stream_keys(state ? state : 0x9E3779B97F4A7C15ULL, 0, n, keys, S(stream));
}

int glm_chunk_keys(uint64_t seed, int64_t n, uint32_t *keys, void *stream) {
    int rc = ensure_device_tables();
    if (rc) return rc;
    return chunk_keys(seed, n, keys, S(stream));
}

size_t glm_argsort_temp_bytes(int64_t n) { return perm_scratch_bytes(n); }

int glm_argsort_u32(const uint32_t *keys, int64_t n, int32_t *perm, void *temp,
                    size_t temp_bytes, void *stream) {
    if (temp_bytes < perm_scratch_bytes(n))
        return glm_set_error(GLM_USAGE, "argsort scratch too small");
    GLM_CUDA_TRY(cudaMemsetAsync(temp, 0, perm_scratch_head_bytes(n), S(stream)));
    PermScratch ps = carve_perm_scratch(temp, n, n);
    return array_perm(keys, n, perm, ps, S(stream));
}

int glm_perm(uint64_t state, int64_t n, int32_t *perm, void *temp, size_t temp_bytes,
             void *stream) {
    int rc = ensure_device_tables();
    if (rc) return rc;
    if (temp_bytes < perm_scratch_bytes(n))
        return glm_set_error(GLM_USAGE, "permutation scratch too small");
    GLM_CUDA_TRY(cudaMemsetAsync(temp, 0, perm_scratch_head_bytes(n), S(stream)));
    PermScratch ps = carve_perm_scratch(temp, n, n);
    return stream_perm(nullptr, state ? state : 0x9E3779B97F4A7C15ULL, 0, n, perm, ps,
                       S(stream));
}

int glm_chunk_perm(uint64_t seed, int64_t n, int32_t *perm, void *temp, size_t temp_bytes,
                   void *stream) {
    int rc = ensure_device_tables();
    if (rc) return rc;
    if (temp_bytes < perm_scratch_bytes(n))
        return glm_set_error(GLM_USAGE, "permutation scratch too small");
    GLM_CUDA_TRY(cudaMemsetAsync(temp, 0, perm_scratch_head_bytes(n), S(stream)));
    PermScratch ps = carve_perm_scratch(temp, n, n);
    return chunk_perm(seed, n, perm, ps, S(stream));
}

// ---------------------------------------------------------------- data
int glm_col_sqnorms(const glm_matrix *A, double *out, void *stream) {
    return launch_colwise(A, 0, nullptr, out, S(stream));
}
int glm_matvec(const glm_matrix *A, const double *x, double *out, void *stream) {
    return launch_matvec(A, x, out, S(stream));
}
int glm_rmatvec(const glm_matrix *A, const double *w, double *out, void *stream) {
    return launch_colwise(A, 1, w, out, S(stream));
}
size_t glm_transpose_temp_bytes(int64_t nnz, int64_t n_rows) {
    return transpose_temp_bytes(nnz, n_rows);
}
int glm_transpose(const glm_matrix *A, int64_t *indptr_t, int32_t *rows_t, double *vals_t,
                  void *temp, size_t temp_bytes, void *stream) {
    return launch_transpose(A, indptr_t, rows_t, vals_t, temp, temp_bytes, S(stream));
}
size_t glm_select_temp_bytes(int64_t k) { return select_temp_bytes(k); }
int glm_select_indptr(const glm_matrix *A, const int64_t *cols, int64_t k, int64_t *out_indptr,
                      void *temp, size_t temp_bytes, void *stream) {
    return launch_select_indptr(A, cols, k, out_indptr, temp, temp_bytes, S(stream));
}
int glm_select_gather(const glm_matrix *A, const int64_t *cols, int64_t k,
                      const int64_t *out_indptr, int32_t *out_rows, double *out_vals,
                      void *stream) {
    return launch_select_gather(A, cols, k, out_indptr, out_rows, out_vals, S(stream));
}
int glm_scale_columns(const glm_matrix *A, const double *scales, double *vals_out, void *stream) {
    return launch_scale(A, scales, vals_out, S(stream));
}
int glm_validate(const glm_matrix *A, void *stream) {
    if (A->layout != GLM_CSC) return GLM_OK;
    unsigned *flags = nullptr;
    GLM_CUDA_TRY(cudaMallocAsync((void **)&flags, sizeof(unsigned), S(stream)));
    GLM_CUDA_TRY(cudaMemsetAsync(flags, 0, sizeof(unsigned), S(stream)));
    int rc = launch_validate(A, flags, S(stream));
    unsigned h = 0;
    if (!rc) {
        GLM_CUDA_TRY(cudaMemcpyAsync(&h, flags, sizeof(h), cudaMemcpyDeviceToHost, S(stream)));
        GLM_CUDA_TRY(cudaStreamSynchronize(S(stream)));
    }
    cudaFreeAsync(flags, S(stream));
    if (rc) return rc;
    if (h & 1) return glm_set_error(GLM_USAGE, "indptr does not span the value arrays");
    if (h & 2) return glm_set_error(GLM_USAGE, "indptr must be non-decreasing");
    if (h & 4) return glm_set_error(GLM_USAGE, "row index out of range");
    if (h & 8) return glm_set_error(GLM_USAGE, "non-finite value in matrix");
    if (h & 16) return glm_set_error(GLM_USAGE, "row indices must be strictly increasing per column");
    return GLM_OK;
}

// ---------------------------------------------------------- objectives
size_t glm_reduce_scratch_bytes(void) { return REDUCE_SCRATCH_BYTES; }

int glm_fgrad(int kind, double lam, const double *target, const double *v, int64_t d,
              double *grad, double *out_fv, double *scratch, void *stream) {
    count_launch();
    fgrad_kernel<<<2 * NUM_SMS, 256, 0, S(stream)>>>(kind, lam, target, v, d, grad, out_fv,
                                                     scratch);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

int glm_outer_model(int kind, double lam, const double *target, const double *v, int64_t d,
                    double *grad, double *lin, double *out_fv, double *cnst_out,
                    double n_nodes, double n_devices, double *scratch, void *stream) {
    count_launch();
    outer_model_kernel<<<2 * NUM_SMS, 256, 0, S(stream)>>>(kind, lam, target, v, d, grad, lin,
                                                           out_fv, cnst_out, n_nodes,
                                                           n_devices, scratch);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

int glm_inner_model(const double *grad, const double *vbar, int64_t d, double qo,
                    const double *fv, double n_nodes, double n_devices, double *lin,
                    double *cnst_out, double *scratch, void *stream) {
    count_launch();
    inner_model_kernel<<<2 * NUM_SMS, 256, 0, S(stream)>>>(grad, vbar, d, qo, fv, n_nodes,
                                                           n_devices, lin, cnst_out, scratch);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

int glm_axpby(int64_t n, double a, const double *x, double b, double *y, void *stream) {
    if (n <= 0) return GLM_OK;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 8 * NUM_SMS) blocks = 8 * NUM_SMS;
    count_launch();
    axpby_kernel<<<(int)blocks, 256, 0, S(stream)>>>(n, a, x, b, y);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

int glm_gap_terms(const glm_matrix *A, int kind, double lam, double l1_ratio,
                  const double *target, const double *coord_target, const double *alpha,
                  const double *v, double *w_scratch, double *out, double *scratch,
                  void *stream) {
    return launch_gap(A, kind, lam, l1_ratio, target, coord_target, alpha, v, w_scratch, out,
                      scratch, S(stream));
}

int glm_gsum(int kind, double lam, double l1_ratio, const double *coord_target,
             const double *alpha, int64_t n, double *out, double *scratch, void *stream) {
    count_launch();
    gsum_kernel<<<2 * NUM_SMS, 256, 0, S(stream)>>>(kind, lam, l1_ratio, coord_target, alpha, n,
                                                    out, scratch);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

int glm_predict(const glm_matrix *X, const double *w, const double *y, int classify,
                double *scores, double *prob, double *out, double *scratch, void *stream) {
    return launch_predict(X, w, y, classify, scores, prob, out, scratch, S(stream));
}

int glm_coordinate_steps(int kind, double lam, double l1_ratio, const double *y,
                         const double *ga, const double *c, const double *t, int64_t n,
                         double *step, void *stream) {
    int *err = nullptr;
    GLM_CUDA_TRY(cudaMallocAsync((void **)&err, sizeof(int), S(stream)));
    GLM_CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(int), S(stream)));
    if (n > 0)
        count_launch();
        coord_steps_kernel<<<4 * NUM_SMS, 256, 0, S(stream)>>>(kind, lam, l1_ratio, y, ga, c, t, n,
                                                               step, err);
    int h = 0;
    GLM_CUDA_TRY(cudaMemcpyAsync(&h, err, sizeof(int), cudaMemcpyDeviceToHost, S(stream)));
    GLM_CUDA_TRY(cudaStreamSynchronize(S(stream)));
    cudaFreeAsync(err, S(stream));
    if (h) return glm_set_error(GLM_SOLVER_ERROR, "non-finite coordinate update");
    return GLM_OK;
}

// ------------------------------------------------------ host-facing ctx
struct glm_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    glm_matrix A{};
    int64_t *indptr = nullptr;
    int32_t *rows = nullptr;
    double *vals = nullptr, *sq = nullptr;
    glm_solver *solver = nullptr;
    double *lin = nullptr, *base = nullptr, *y = nullptr, *cnst = nullptr;
    double *dalpha = nullptr, *dv = nullptr, *alpha = nullptr, *v = nullptr, *w = nullptr;
    double *tgt = nullptr, *out4 = nullptr, *scratch = nullptr;
    double *pin_cnst = nullptr;   // pinned host staging for the scalar input
};

int glm_ctx_destroy(glm_ctx *c) {
    if (!c) return GLM_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    glm_solver_destroy(c->solver);
    void *ptrs[] = {c->indptr, c->rows, c->vals, c->sq, c->lin, c->base, c->y, c->cnst,
                    c->dalpha, c->dv, c->alpha, c->v, c->w, c->tgt, c->out4, c->scratch};
    for (void *p : ptrs) cudaFree(p);
    if (c->pin_cnst) cudaFreeHost(c->pin_cnst);
    if (c->stream) cudaStreamDestroy(c->stream);
    cudaSetDevice(prev);
    delete c;
    return GLM_OK;
}

int glm_ctx_create(int device, int layout, int64_t n_rows, int64_t n_cols, const int64_t *indptr,
                   const int32_t *rows, const double *vals, glm_ctx **out) {
    if (!out || n_rows < 0 || n_cols < 0 || !vals)
        return glm_set_error(GLM_USAGE, "bad ctx arguments");
    if (layout == GLM_CSC && (!indptr || !rows)) return glm_set_error(GLM_USAGE, "CSC needs indptr/rows");
    GLM_CUDA_TRY(cudaSetDevice(device));
    glm_ctx *c = new (std::nothrow) glm_ctx();
    if (!c) return glm_set_error(GLM_USAGE, "out of host memory");
    c->device = device;
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    const int64_t nnz = layout == GLM_CSC ? indptr[n_cols] : n_rows * n_cols;
    const size_t m1 = (size_t)(n_cols > 0 ? n_cols : 1), d1 = (size_t)(n_rows > 0 ? n_rows : 1);
    auto chk = [&](cudaError_t x) { if (x != cudaSuccess && e == cudaSuccess) e = x; };
    if (layout == GLM_CSC) {
        chk(cudaMalloc(&c->indptr, sizeof(int64_t) * (n_cols + 1)));
        chk(cudaMalloc(&c->rows, sizeof(int32_t) * (nnz > 0 ? nnz : 1)));
    }
    chk(cudaMalloc(&c->vals, sizeof(double) * (nnz > 0 ? nnz : 1)));
    chk(cudaMalloc(&c->sq, sizeof(double) * m1));
    for (double **p : {&c->base, &c->y, &c->dalpha, &c->alpha}) chk(cudaMalloc(p, sizeof(double) * m1));
    for (double **p : {&c->lin, &c->dv, &c->v, &c->w, &c->tgt}) chk(cudaMalloc(p, sizeof(double) * d1));
    chk(cudaMalloc(&c->cnst, sizeof(double) * 8));
    chk(cudaMalloc(&c->out4, sizeof(double) * 8));
    chk(cudaMalloc(&c->scratch, REDUCE_SCRATCH_BYTES));
    chk(cudaMallocHost(&c->pin_cnst, sizeof(double)));
    if (e == cudaSuccess) {
        chk(cudaMemsetAsync(c->scratch, 0, REDUCE_SCRATCH_BYTES, c->stream));
        if (layout == GLM_CSC) {
            chk(cudaMemcpyAsync(c->indptr, indptr, sizeof(int64_t) * (n_cols + 1),
                                cudaMemcpyHostToDevice, c->stream));
            if (nnz > 0)
                chk(cudaMemcpyAsync(c->rows, rows, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice,
                                    c->stream));
        }
        if (nnz > 0)
            chk(cudaMemcpyAsync(c->vals, vals, sizeof(double) * nnz, cudaMemcpyHostToDevice,
                                c->stream));
    }
    if (e != cudaSuccess) {
        glm_ctx_destroy(c);
        return glm_set_cuda_error(e, "glm_ctx_create", __FILE__, __LINE__);
    }
    c->A.n_rows = n_rows;
    c->A.n_cols = n_cols;
    c->A.nnz = nnz;
    c->A.layout = layout;
    c->A.indptr = c->indptr;
    c->A.rows = c->rows;
    c->A.vals = c->vals;
    c->A.sqnorms = c->sq;
    int rc = launch_colwise(&c->A, 0, nullptr, c->sq, c->stream);
    if (!rc) rc = glm_solver_create(device, n_cols, n_rows, &c->solver);
    if (!rc) rc = glm_solver_prepare(c->solver, &c->A, c->stream);   // packed records (CSC)
    if (!rc) {
        cudaError_t e2 = cudaStreamSynchronize(c->stream);
        if (e2 != cudaSuccess) rc = glm_set_cuda_error(e2, "ctx sync", __FILE__, __LINE__);
    }
    if (rc) {
        glm_ctx_destroy(c);
        return rc;
    }
    *out = c;
    return GLM_OK;
}

int glm_device_solve(glm_ctx *c, int kind, double lam, double l1_ratio,
                     const double *coord_target, const double *lin, double quad, double cnst,
                     const double *base, uint64_t *gen_state_io, double *damping_io, int epochs,
                     int mode, double *dalpha_out, double *dv_out, double *values_out,
                     int32_t *info_out, double *scal_out) {
    if (!c || !lin || !base || !gen_state_io || !damping_io)
        return glm_set_error(GLM_USAGE, "null argument to glm_device_solve");
    if (epochs < 1) return glm_set_error(GLM_USAGE, "t_epochs must be >= 1");
    GLM_CUDA_TRY(cudaSetDevice(c->device));
    const int64_t m = c->A.n_cols, d = c->A.n_rows;
    cudaStream_t s = c->stream;
    int rc = set_state(c->solver, *gen_state_io, *damping_io, s);
    // attempt 0's permutation depends only on the generator state: build it
    // on the side stream while the inputs cross PCIe
    if (!rc) rc = prefetch_first_perm(c->solver, m, s);
    if (rc) return rc;
    if (d > 0) GLM_CUDA_TRY(cudaMemcpyAsync(c->lin, lin, sizeof(double) * d, cudaMemcpyHostToDevice, s));
    if (m > 0) GLM_CUDA_TRY(cudaMemcpyAsync(c->base, base, sizeof(double) * m, cudaMemcpyHostToDevice, s));
    if (coord_target && m > 0)
        GLM_CUDA_TRY(cudaMemcpyAsync(c->y, coord_target, sizeof(double) * m, cudaMemcpyHostToDevice, s));
    *c->pin_cnst = cnst;              // pinned: the copy never stages through pageable memory
    GLM_CUDA_TRY(cudaMemcpyAsync(c->cnst, c->pin_cnst, sizeof(double), cudaMemcpyHostToDevice, s));
    glm_solve_args a{};
    a.kind = kind;
    a.mode = mode;
    a.lam = lam;
    a.l1_ratio = l1_ratio;
    a.quad = quad;
    a.cnst = c->cnst;
    a.lin = c->lin;
    a.base = c->base;
    a.coord_target = coord_target ? c->y : nullptr;
    a.epochs = epochs;
    a.max_attempts = 0;
    a.group_lanes = 0;
    a.reset_damping = 0;
    glm_solve_result r{};
    HostCopies hc;
    hc.delta = dalpha_out;
    hc.dv = dv_out;
    // one host round trip when the batch is accepted: finalize and the copies
    // are enqueued before the solve's synchronisation (solve's HostCopies)
    rc = solve(c->solver, &c->A, &a, c->dalpha, c->dv, &r, s, &hc);
    if (rc) return rc;
    if (values_out) fill_result(c->solver, nullptr, values_out, epochs);
    *gen_state_io = r.gen_state;
    *damping_io = r.damping;
    if (info_out) {
        info_out[0] = r.epochs_run;
        info_out[1] = r.retries;
        info_out[2] = r.plateaued;
        info_out[3] = r.attempts;
        info_out[4] = r.status;
    }
    if (scal_out) {
        scal_out[0] = r.initial_value;
        scal_out[1] = r.final_value;
    }
    if (r.status == GLM_DIVERGENCE)
        return glm_set_error(GLM_DIVERGENCE, "damping floor reached without subproblem decrease");
    if (r.status != GLM_OK)
        return glm_set_error(r.status, "non-finite entries in shared view or coordinate update");
    return GLM_OK;
}

int glm_ctx_gap_terms(glm_ctx *c, int kind, double lam, double l1_ratio, const double *target,
                      const double *coord_target, const double *alpha, const double *v,
                      double *out) {
    if (!c || !alpha || !v || !out) return glm_set_error(GLM_USAGE, "null argument");
    GLM_CUDA_TRY(cudaSetDevice(c->device));
    const int64_t m = c->A.n_cols, d = c->A.n_rows;
    cudaStream_t s = c->stream;
    if (m > 0) GLM_CUDA_TRY(cudaMemcpyAsync(c->alpha, alpha, sizeof(double) * m, cudaMemcpyHostToDevice, s));
    if (d > 0) GLM_CUDA_TRY(cudaMemcpyAsync(c->v, v, sizeof(double) * d, cudaMemcpyHostToDevice, s));
    if (target && d > 0)
        GLM_CUDA_TRY(cudaMemcpyAsync(c->tgt, target, sizeof(double) * d, cudaMemcpyHostToDevice, s));
    if (coord_target && m > 0)
        GLM_CUDA_TRY(cudaMemcpyAsync(c->y, coord_target, sizeof(double) * m, cudaMemcpyHostToDevice, s));
    int rc = launch_gap(&c->A, kind, lam, l1_ratio, target ? c->tgt : nullptr,
                        coord_target ? c->y : nullptr, c->alpha, c->v, c->w, c->out4, c->scratch,
                        s);
    if (rc) return rc;
    GLM_CUDA_TRY(cudaMemcpyAsync(out, c->out4, sizeof(double) * 4, cudaMemcpyDeviceToHost, s));
    GLM_CUDA_TRY(cudaStreamSynchronize(s));
    return GLM_OK;
}

}  // extern "C"
