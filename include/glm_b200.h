/*
 * glm_b200.h — C-ABI of the B200-native GLM / TPA-SCD hot path.
 *
 * Plain pointers and sizes only (no torch types).  Two levels:
 *
 *  (1) Reference-facing, HOST buffers (the drop-in boundary).  These replace
 *      the reference's device-solve plugin hook:
 *        Engine(..., chunk_runner=fn) -> fn(sub, dev, cfg)
 *        (/root/reference/pkg/src/hierglm/engine.py:177-179, 228-233)
 *      whose default body is damped_solve(sub, dev.gen, cfg.epochs, ...,
 *      damping=dev.damping) (solver.py:250-305).  glm_ctx_* owns a device
 *      partition (the matrix resident in HBM, created once like the reference's
 *      _Device.data, engine.py:113-118); glm_device_solve is one subtask.
 *
 *  (2) Device-resident (DEVICE pointers + a cudaStream_t passed as void*):
 *      the kernels the Python engine drives without host round-trips.
 *
 * Status codes (mapped 1:1 onto the reference's exceptions by the host layer):
 *   GLM_OK                0
 *   GLM_SOLVER_ERROR      1  -> SolverError      (solver.py:31-32, 160-161, 185-186, 279-280)
 *   GLM_DIVERGENCE        2  -> SolverDivergence (solver.py:35-38, 289-293)
 *   GLM_USAGE             3  -> ValueError / UsageError
 *   GLM_CUDA_ERROR        4  -> RuntimeError (CUDA failure; message via glm_last_error)
 *
 * Objective kinds: indices 0..3 are objectives.py:22 KINDS in order; 4..7 are
 * restated kinds (parity unpinned by the reference).
 */
#ifndef GLM_B200_H
#define GLM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GLM_OK 0
#define GLM_SOLVER_ERROR 1
#define GLM_DIVERGENCE 2
#define GLM_USAGE 3
#define GLM_CUDA_ERROR 4

enum glm_kind {
    GLM_DUAL_L2_LOGISTIC = 0,     /* objectives.py:5  */
    GLM_DUAL_L2_SVM = 1,          /* objectives.py:7  */
    GLM_RIDGE_PRIMAL = 2,         /* objectives.py:8  */
    GLM_LASSO_PRIMAL = 3,         /* objectives.py:9  */
    GLM_DUAL_RIDGE = 4,           /* restated */
    GLM_ELASTIC_NET_PRIMAL = 5,   /* restated */
    GLM_LOGISTIC_PRIMAL = 6,      /* restated */
    GLM_SQUARED_HINGE_PRIMAL = 7, /* restated */
    GLM_HINGE_PRIMAL = 8          /* restated: smoothed hinge, row target y_r / mu */
};

enum glm_layout { GLM_CSC = 0, GLM_DENSE = 1 };

enum glm_mode {
    GLM_MODE_SEQUENTIAL = 0,  /* deterministic fixed-permutation mode: run_pass n_threads=1 (solver.py:202-211) */
    GLM_MODE_ASYNC = 1        /* TPA-SCD: concurrent coordinate groups, atomic scatter (solver.py:213-239) */
};

/* Matrix in HBM.  CSC: indptr i64[n_cols+1], rows i32[nnz] (sorted unique per
 * column), vals f64[nnz]  (data.py:42-62).  DENSE: vals f64[n_rows*n_cols]
 * column-major (column j at vals + j*n_rows), indptr/rows NULL. */
typedef struct {
    int64_t n_rows;
    int64_t n_cols;
    int64_t nnz;
    int32_t layout;
    int32_t _pad;
    const int64_t *indptr;
    const int32_t *rows;
    const double *vals;
    const double *sqnorms;   /* f64[n_cols] (col_sqnorms, data.py:98-107) */
} glm_matrix;

typedef struct glm_peer glm_peer;       /* NVLink peer-memory Delta v exchange (4) */

/* One subtask (the LocalSubproblem of solver.py:107-135) on device memory. */
typedef struct {
    int32_t kind;
    int32_t mode;           /* glm_mode */
    double lam;
    double l1_ratio;        /* elastic-net rho (kind 5); ignored otherwise */
    double quad;            /* LocalSubproblem.quad */
    const double *cnst;     /* device scalar: LocalSubproblem.const */
    const double *lin;      /* device f64[n_rows] */
    const double *base;     /* device f64[n_cols] */
    const double *coord_target; /* device f64[n_cols] per-coordinate y (kind 4) or NULL */
    int32_t epochs;         /* t_epochs (solver.py:250) */
    int32_t max_attempts;   /* 0 = run until done (host-synchronous retry loop) */
    int32_t group_lanes;    /* async: lanes per coordinate (0 = auto) */
    int32_t max_inflight;   /* async: cap on concurrently processed coordinates
                               (0 = auto: min(resident groups, n/32)) */
    int32_t reset_damping;  /* 1: DampingState.reset() before solving (engine.py:251-252) */
    int32_t accumulate;     /* 1: delta_out += delta, dv_out += B delta (fold in place,
                               engine.py:264-266, 302-306); 0: overwrite */
    int32_t flags;          /* bit 0 / bit 1: async cache policy (1 gather the view through
                               L1; 2 stream the column L2 evict_first, view evict_last);
                               GLM_FLAG_REUSE_GSUM: base equals the previous solve's
                               base + delta (folded in place), reuse its g-sum for G(0) */
    glm_peer *peer;         /* GLM_FLAG_PEER_FINALIZE: the round's Delta v exchange */
} glm_solve_args;

#define GLM_FLAG_REUSE_GSUM 4
/* After the solve, generate the next solve's first permutation on a side
 * stream (from the advanced generator state) so it overlaps the caller's
 * fold / all-reduce; the next glm_solve of the same solver consumes it. */
#define GLM_FLAG_PREFETCH_PERM 8
/* Write B delta into this rank's peer-exchange buffer and publish it (with
 * accumulate = 1: delta_out += delta; dv_out unused) — see glm_round_start. */
#define GLM_FLAG_PEER_FINALIZE 32
/* glm_round_start(mode 2) already started this solve (requires REUSE_GSUM). */
#define GLM_FLAG_SKIP_BEGIN 64
/* One attempt (epochs = max_attempts = 1) whose value check, finalize and
 * Delta v exchange are left to glm_round_turn on the same stream. */
#define GLM_FLAG_TURN 128

/* Result of a subtask (SubtaskResult, solver.py:138-149 + DampingState). */
typedef struct {
    int32_t status;
    int32_t epochs_run;
    int32_t retries;
    int32_t plateaued;
    int32_t attempts;       /* scd_epoch calls == permutations consumed */
    int32_t done;
    double damping;         /* DampingState.delta after the solve */
    double initial_value;   /* initial_subproblem_value */
    double final_value;     /* final_subproblem_value (= DampingState.last_subproblem_value) */
    uint64_t gen_state;     /* PermutationGenerator.state after the solve */
} glm_solve_result;

typedef struct glm_solver glm_solver;   /* per-partition scratch + device state */
typedef struct glm_ctx glm_ctx;         /* host-facing partition: matrix + solver */

/* ---------------------------------------------------------------- misc */
const char *glm_last_error(void);
int glm_version(void);
/* Number of kernels this library has launched (process-wide, monotone). */
long long glm_launch_count(void);
int glm_device_count(int *out);
/* Debug: kernels record min start / max end %globaltimer (ns) into device
 * u64[16] slot pairs: [0,1] epoch, [2,3] first permutation kernel, [4,5] last
 * permutation kernel, [6,7] round turn.  NULL: off. */
int glm_debug_timeline(unsigned long long *device_slots);
/* Host-side xorshift64 jump: state after `steps` steps (solver.py:41-46). */
uint64_t glm_xorshift_jump(uint64_t state, uint64_t steps);
uint64_t glm_derive_seed(uint64_t base, const uint64_t *idx, int n_idx); /* solver.py:57-61 */

/* ------------------------------------------------ (1) host-facing drop-in */
/* Copy a host CSC/dense partition into HBM and compute its column norms.
 * Replaces _Device(...) data placement (engine.py:113-118). */
int glm_ctx_create(int device, int layout, int64_t n_rows, int64_t n_cols,
                   const int64_t *indptr, const int32_t *rows, const double *vals,
                   glm_ctx **out);
int glm_ctx_destroy(glm_ctx *ctx);
/* One device subtask with HOST buffers: the semantics of
 * damped_solve(sub, gen, epochs, n_threads, damping) (solver.py:250-305) where
 * mode selects sequential (n_threads=1) or asynchronous execution.
 * gen_state_io  <-> dev.gen.state          (solver.py:70-89)
 * damping_io    <-> dev.damping.delta      (solver.py:92-104)
 * values_out    <-  SubtaskResult.epoch_values (capacity `epochs`)
 * info_out[5]   <-  epochs_run, retries, plateaued, attempts, status
 * scal_out[2]   <-  initial / final subproblem value */
int glm_device_solve(glm_ctx *ctx, int kind, double lam, double l1_ratio,
                     const double *coord_target, const double *lin, double quad,
                     double cnst, const double *base, uint64_t *gen_state_io,
                     double *damping_io, int epochs, int mode, double *dalpha_out,
                     double *dv_out, double *values_out, int32_t *info_out,
                     double *scal_out);
/* Fused duality gap over the ctx partition with host buffers
 * (objectives.duality_gap, objectives.py:223-234): out[0]=f(v)+f*(w),
 * out[1]=sum g(alpha), out[2]=sum g*(-a^T w), out[3]=f(v). */
int glm_ctx_gap_terms(glm_ctx *ctx, int kind, double lam, double l1_ratio,
                      const double *target, const double *coord_target,
                      const double *alpha, const double *v, double *out);

/* --------------------------------------------- (2) device-resident API */
int glm_solver_create(int device, int64_t max_coords, int64_t max_rows, glm_solver **out);
int glm_solver_destroy(glm_solver *s);
/* Set the solver's permutation stream (PermutationGenerator(seed).state) and
 * damping (DampingState.delta) held in device memory. */
int glm_solver_set_state(glm_solver *s, uint64_t gen_state, double damping, void *stream);
/* Optional, once per CSC partition (outside any captured graph): build packed
 * 16-byte per-coordinate records {start | count << 40, |a_j|^2} that the async
 * epoch kernel then loads in one sector instead of the indptr pair and the
 * norm.  Later solves on the same (indptr, sqnorms, n_cols) use them. */
int glm_solver_prepare(glm_solver *s, const glm_matrix *A, void *stream);
/* Asynchronous subtask: all attempts are enqueued on `stream`; outputs are
 * device arrays.  If args->max_attempts == 0 the call synchronises to run the
 * retry loop to completion and fills `res`; otherwise it enqueues exactly
 * max_attempts attempts (skipped on device once done) and `res` may be NULL
 * (read later with glm_solver_result). */
int glm_solve(glm_solver *s, const glm_matrix *A, const glm_solve_args *args,
              double *delta_out, double *dv_out, glm_solve_result *res, void *stream);
/* Bracket every attempt with CUDA events on the solve stream:
 * ms_out[0] = permutation kernels, [1] = snapshot + epoch kernel, [2] = value
 * kernel, summed over the attempts since the last read; *n_out = attempts. */
int glm_solver_timing(glm_solver *s, int enable);
int glm_solver_timing_read(glm_solver *s, double *ms_out, int32_t *n_out);
/* Same sums without releasing the events (graph-captured attempts re-record
 * them on every replay). */
int glm_solver_timing_peek(glm_solver *s, double *ms_out, int32_t *n_out);
/* Finalize ([0]), glm_round_start ([1]) and glm_round_turn ([2]) kernels
 * bracketed while timing is on: ms_out[3] sums, n_out[3] counts; consume = 0
 * keeps graph-captured events. */
int glm_solver_timing_glue(glm_solver *s, double *ms_out, int32_t *n_out, int consume);
/* Make `stream` wait for a pending permutation prefetch (before ending a
 * graph capture or reusing the solver from another stream). */
int glm_solver_join(glm_solver *s, void *stream);
/* Copy the device-side solve state to the host (synchronises `stream`).
 * epoch_values may be NULL; else capacity >= epochs of the last solve. */
int glm_solver_result(glm_solver *s, glm_solve_result *res, double *epoch_values,
                      int capacity, void *stream);

/* Permutations (solver.py:77-89, pipeline.py:29-78).  keys/perm are device. */
int glm_perm_keys(uint64_t state, int64_t n, uint32_t *keys, void *stream);
int glm_chunk_keys(uint64_t seed, int64_t n, uint32_t *keys, void *stream);
size_t glm_argsort_temp_bytes(int64_t n);
/* stable argsort of u32 keys -> int32 perm (np.argsort(kind="stable")) */
int glm_argsort_u32(const uint32_t *keys, int64_t n, int32_t *perm, void *temp,
                    size_t temp_bytes, void *stream);
/* Fused generate + stable argsort, the solver's own permutation path:
 * PermutationGenerator(state).permute(n) (solver.py:86-89) and
 * keys_to_permutation(generate_keys(seed, n)) (pipeline.py:29-78).  The keys
 * are regenerated in both passes, never stored.  temp: glm_argsort_temp_bytes(n)
 * bytes (its counters are zeroed by the call). */
int glm_perm(uint64_t state, int64_t n, int32_t *perm, void *temp, size_t temp_bytes,
             void *stream);
int glm_chunk_perm(uint64_t seed, int64_t n, int32_t *perm, void *temp, size_t temp_bytes,
                   void *stream);

/* Data layer (data.py:98-187, cli.py:146-185).  All device pointers. */
int glm_col_sqnorms(const glm_matrix *A, double *out, void *stream);
int glm_matvec(const glm_matrix *A, const double *x, double *out, void *stream);   /* out = A x (atomic scatter) */
int glm_rmatvec(const glm_matrix *A, const double *w, double *out, void *stream);  /* out = A^T w */
/* Stable transpose (data.py:155-165): outputs sized n_rows+1 / nnz / nnz. */
size_t glm_transpose_temp_bytes(int64_t nnz, int64_t n_rows);
int glm_transpose(const glm_matrix *A, int64_t *indptr_t, int32_t *rows_t, double *vals_t,
                  void *temp, size_t temp_bytes, void *stream);
/* select_columns (data.py:132-145): cols i64[k]; glm_select_indptr fills
 * out_indptr i64[k+1] (device scan), then glm_select_gather copies. */
size_t glm_select_temp_bytes(int64_t k);
int glm_select_indptr(const glm_matrix *A, const int64_t *cols, int64_t k,
                      int64_t *out_indptr, void *temp, size_t temp_bytes, void *stream);
int glm_select_gather(const glm_matrix *A, const int64_t *cols, int64_t k,
                      const int64_t *out_indptr, int32_t *out_rows, double *out_vals,
                      void *stream);
/* scale_columns (data.py:147-153): vals_out[p] = vals[p] * scales[col(p)] */
int glm_scale_columns(const glm_matrix *A, const double *scales, double *vals_out,
                      void *stream);
/* Validation (data.py:64-84); synchronises `stream`.  GLM_USAGE + message on failure. */
int glm_validate(const glm_matrix *A, void *stream);

/* Objective / engine glue (objectives.py:129-234, engine.py:131-166, 269-351).
 * Scalars are device f64 pointers so rounds never leave the device.
 * `scratch`: device buffer of glm_reduce_scratch_bytes(), zero-filled once,
 * not shared by concurrently running calls (deterministic block-order sums). */
size_t glm_reduce_scratch_bytes(void);
/* grad = f'(v) (grad may be NULL); out_fv[0] = f(v) */
int glm_fgrad(int kind, double lam, const double *target, const double *v, int64_t d,
              double *grad, double *out_fv, double *scratch, void *stream);
/* Round start (engine.py:271-272) fused with the first inner model (v_bar = 0):
 * grad = f'(v), lin = grad, out_fv[0] = f(v), cnst_out[0] = f(v) / (K L). */
int glm_outer_model(int kind, double lam, const double *target, const double *v, int64_t d,
                    double *grad, double *lin, double *out_fv, double *cnst_out,
                    double n_nodes, double n_devices, double *scratch, void *stream);
/* Inner subproblem (engine.py:148-166) with the outer model (engine.py:242-250):
 * lin = grad + qo*vbar; cnst_out = (fv/K + grad.vbar + qo/2 |vbar|^2) / L.
 * vbar may be NULL (= 0). */
int glm_inner_model(const double *grad, const double *vbar, int64_t d, double qo,
                    const double *fv, double n_nodes, double n_devices, double *lin,
                    double *cnst_out, double *scratch, void *stream);
/* y = a*x + b*y elementwise (fold / apply steps, engine.py:264-266, 302-306) */
int glm_axpby(int64_t n, double a, const double *x, double b, double *y, void *stream);
/* Fused gap terms (engine.py:325-351, objectives.py:223-234) over partition A:
 * out[0] = f(v)+f*(w), out[1] = sum g(alpha), out[2] = sum g*(-a^T w), out[3] = f(v).
 * w_scratch f64[n_rows]. */
int glm_gap_terms(const glm_matrix *A, int kind, double lam, double l1_ratio,
                  const double *target, const double *coord_target, const double *alpha,
                  const double *v, double *w_scratch, double *out, double *scratch,
                  void *stream);
/* out[0] = sum g(alpha) (g_sum, objectives.py:165-173) */
int glm_gsum(int kind, double lam, double l1_ratio, const double *coord_target,
             const double *alpha, int64_t n, double *out, double *scratch, void *stream);
/* Prediction over an example-major matrix X (columns = examples, n_rows <= len(w)):
 * scores = X^T w (decision_scores, modelio.py:64-75); prob = 0.5(1+tanh(z/2));
 * out[0] = -sum[y log p + (1-y) log(1-p)] (clip 1e-15), out[1] = #(p>=0.5 == y>0),
 * out[2] = sum (score - y)^2.  y (raw labels) may be NULL. */
int glm_predict(const glm_matrix *X, const double *w, const double *y, int classify,
                double *scores, double *prob, double *out, double *scratch, void *stream);
/* Batched undamped coordinate steps (coordinate_update, solver.py:152-187)
 * from (ga, c = quad*|a|^2, t) triples.  GLM_SOLVER_ERROR if any non-finite. */
int glm_coordinate_steps(int kind, double lam, double l1_ratio, const double *y,
                         const double *ga, const double *c, const double *t, int64_t n,
                         double *step, void *stream);

/* ------------------------------------ (3) out-of-core streaming pipeline
 * Replaces chunked_device_runner / pipelined_epoch / _train_chunk
 * (/root/reference/pkg/src/hierglm/pipeline.py:158-340): the engine's
 * chunk_runner hook (engine.py:228-229) for a device partition cut into
 * chunks.  Chunks within `device_budget` bytes stay resident in HBM (<= 0:
 * all resident); the rest stream every epoch through two device slots,
 * double-buffered against the solve (loader thread -> pinned staging ->
 * cudaMemcpyAsync on a copy stream).  Per chunk: keys
 * generate_keys(derive_seed(seed, epoch_index + e, chunk)) (pipeline.py:
 * 226-227), stable argsort, one damped pass with chunk-granular
 * restore / plateau / halve / divergence (pipeline.py:180-193). */
typedef struct glm_stream glm_stream;

#define GLM_STREAM_DELTA_IN 16   /* delta_io holds the starting delta (else zero) */
#define GLM_STREAM_VIEW_IN 32    /* view_io holds the starting view (else lin) */
#define GLM_STREAM_TIMING 64     /* record the per-chunk schedule (glm_stream_schedule) */
#define GLM_STREAM_SCHED_COLS 6  /* epoch, chunk, load_ms, h2d_ms, train_ms, t_ms */

typedef struct {
    int32_t kind;
    int32_t mode;               /* glm_mode: per-chunk run_pass n_threads==1 / > 1 */
    double lam;
    double l1_ratio;
    double quad;
    double cnst;                /* LocalSubproblem.const of the whole device partition */
    const double *lin;          /* f64[n_rows]  (host or device memory) */
    const double *base;         /* f64[n_cols]  (host or device memory) */
    const double *coord_target; /* f64[n_cols] or NULL */
    uint64_t seed;              /* chunked_device_runner(store, seed, ...) */
    uint64_t epoch_index;       /* the runner's global epoch counter at this call */
    int32_t epochs;
    int32_t attempts_per_chunk; /* attempts enqueued ahead per chunk (0 = 2) */
    int32_t group_lanes;
    int32_t max_inflight;
    int32_t flags;              /* bits 0-1 cache policy (glm_solve_args.flags), GLM_STREAM_* */
    int32_t _pad;
} glm_stream_args;

/* Host CSC arrays (pinned arrays are DMA'd directly; pin_host=1 registers
 * pageable arrays, else they are staged through pinned buffers); chunk c =
 * columns [col_offsets[c], col_offsets[c+1]).  The arrays must outlive the
 * stream. */
int glm_stream_create_host(int device, int64_t n_rows, int64_t n_cols, const int64_t *indptr,
                           const int32_t *rows, const double *vals, int n_chunks,
                           const int64_t *col_offsets, int64_t device_budget, int pin_host,
                           glm_stream **out);
/* A GLMCHUNK v1 file (data.py:307-431) read with pread by the loader thread:
 * chunk_offsets = ChunkDescriptor.offset (the <IQ chunk head) as scanned by
 * open_chunks (data.py:362-398). */
int glm_stream_create_file(int device, const char *path, int64_t n_rows, int n_chunks,
                           const int64_t *chunk_offsets, const int64_t *chunk_cols,
                           const int64_t *chunk_nnz, int64_t device_budget, glm_stream **out);
int glm_stream_destroy(glm_stream *s);
/* File streams only: read streamed chunk bodies with O_DIRECT (the page cache
 * bypassed: an aligned superset of each body into the pinned staging buffer;
 * falls back to buffered reads where the file system refuses O_DIRECT — see
 * glm_stream_info out[7]) and with io_threads concurrent preads per body.
 * Buffered reads also advise the kernel to read the next chunk ahead. */
int glm_stream_set_io(glm_stream *s, int direct_io, int io_threads);
/* out[8] = n_chunks, resident chunks, resident bytes, streaming-slot bytes,
 * direct DMA (0/1), n_cols, n_rows, O_DIRECT reads active (0/1) */
int glm_stream_info(const glm_stream *s, int64_t *out);
/* `epochs` passes over every chunk (chunked_device_runner's runner body).
 * delta_io f64[n_cols] (in with GLM_STREAM_DELTA_IN; out: the partition's
 * Delta alpha), view_io f64[n_rows] or NULL (the running view, in with
 * GLM_STREAM_VIEW_IN), dv_out = B delta = (view - lin)/quad or NULL,
 * values_out[epochs] = device value after each epoch, info_out[5] =
 * epochs_run, retries, plateaued chunks, attempts, status; scal_out[4] =
 * initial value, final value, wall ms, ms the solve waited for loads.
 * Pointers may be host or device memory. */
int glm_stream_solve(glm_stream *s, const glm_stream_args *args, double *damping_io,
                     double *delta_io, double *view_io, double *dv_out, double *values_out,
                     int32_t *info_out, double *scal_out);
/* Per-chunk schedule of the last solve with GLM_STREAM_TIMING (PipelineSchedule,
 * pipeline.py:81-138): GLM_STREAM_SCHED_COLS doubles per chunk. */
int glm_stream_schedule(const glm_stream *s, double *out, int capacity_rows, int *n_rows_out);

/* ------------------------------ (4) fused Delta v exchange over peer memory
 * The round's collective (allreduce_sum(v_bar) with canonical_sum's
 * ascending-rank fold, engine.py:282, comm.py:41-46) fused with v += total
 * (engine.py:306) and the next round's model + solve start (engine.py:
 * 242-272, 148-166): one process per GPU, every rank's Delta v in its own HBM
 * mapped into every peer through CUDA IPC (NVLink / NVSwitch).  A solve with
 * GLM_FLAG_PEER_FINALIZE publishes its Delta v; glm_round_start waits for all
 * ranks' publications (system-scope acquire), sums them in rank order (the
 * same bits on every rank, = canonical_sum), applies them to v and runs the
 * outer model; mode 2 also starts the solver (views, G(0), state).
 * mode 0 only applies pending Delta v (before reading v). */
int glm_peer_create(int device, int64_t n_rows, int rank, int world, glm_peer **out);
size_t glm_peer_handle_bytes(void);
int glm_peer_handle(const glm_peer *p, void *handle_out);
/* handles: world x glm_peer_handle_bytes() bytes, rank order (all_gather) */
int glm_peer_open(glm_peer *p, const void *handles);
/* Mark any published, unapplied Delta v as consumed (engine reset). */
int glm_peer_consume(glm_peer *p, void *stream);
int glm_round_start(glm_peer *p, glm_solver *s, int mode, int kind, double lam,
                    const double *target, double *v, int64_t n_rows, double *grad, double *lin,
                    double *out_fv, double *cnst, double n_nodes, double n_devices, int epochs,
                    double *scratch, void *stream);
int glm_peer_destroy(glm_peer *p);
/* Deadline of every device-side wait of the exchange (default 60 s, the
 * reference's DEFAULT_TIMEOUT, comm.py:30).  A wait that expires records
 * itself in the exchange's error word and lets its kernel finish. */
int glm_peer_set_timeout(glm_peer *p, double seconds);
/* Synchronises the device and reads the error word: 0 = none, else
 * (kind << 32 | what): kind 1 = rank `what` did not publish in time (a dead or
 * stalled peer, -> ReduceError), kind 2 = the turn's grid was not co-resident.
 * clear != 0 resets it. */
int glm_peer_error(glm_peer *p, int64_t *code_out, int clear);
/* Debug: glm_round_turn writes %globaltimer stamps (ns) of its phases into
 * device u64[8]: start, decided, published, every rank seen, done (NULL: off). */
int glm_peer_stamps(glm_peer *p, uint64_t *device_array);
/* After a GLM_FLAG_TURN solve: the attempt's value check and damping decision,
 * alpha += delta, publish Delta v, wait for every rank's, v += their rank-order
 * sum, and the next round's model and solver start — one kernel (peer.cu).
 * cnst holds this round's const on entry and the next round's on exit. */
int glm_round_turn(glm_peer *p, glm_solver *s, int kind, double lam, double quad,
                   double *cnst, double *alpha, int64_t m, const double *target, double *v,
                   int64_t n_rows, double *grad, double *lin, double *out_fv, double n_nodes,
                   double n_devices, int epochs, double *scratch, void *stream);

/* --------------------------------------- (5) host ingest: svmlight parser
 * parse_svmlight (data.py:190-239), multi-threaded: `<label> <idx>:<val> ...`
 * lines, 1-based strictly increasing indices, blank / '#' lines skipped.
 * info[7] = n_examples, nnz, max feature index, error kind (0 ok, 1 bad label,
 * 2 bad feature token, 3 index < 1, 4 not increasing, 5 index out of int32
 * range), error line (1-based), token offset, token length.  On success
 * *out holds the result until glm_svmlight_free; glm_svmlight_fetch fills the
 * example-major CSC (indptr i64[n+1], rows i32[nnz], vals f64[nnz]) and the
 * labels f64[n]. */
typedef struct glm_svmlight glm_svmlight;
int glm_svmlight_parse(const char *text, int64_t len, int n_threads, glm_svmlight **out,
                       int64_t *info);
int glm_svmlight_fetch(const glm_svmlight *r, int64_t *indptr, int32_t *rows, double *vals,
                       double *labels);
int glm_svmlight_free(glm_svmlight *r);

/* ------------------------------------- (6) GLMCHUNK v1 chunk store (host)
 * write_chunks / open_chunks / read_chunk (data.py:17-27, 329-426), byte-for-
 * byte the reference's format.  Status kinds (the Python layer raises the
 * reference's ChunkFormatError messages): 0 ok, 1 truncated header, 2 bad
 * magic, 3 endianness mismatch, 4 unsupported version, 5 truncated row
 * vector, 6 truncated chunk header, 7 column counts do not sum to n_cols,
 * 8 chunk header disagrees with descriptor, 9 truncated chunk body,
 * 10 OS error (errno reported). */
/* labels / row_vector NULL: not stored.  offsets_out: ceil(n_cols/chunk_size)
 * chunk offsets.  *os_errno != 0 if the file could not be written. */
int glm_chunk_write(const char *path, int64_t n_rows, int64_t n_cols, const int64_t *indptr,
                    const int32_t *rows, const double *vals, const double *labels,
                    const double *row_vector, int64_t chunk_size, int64_t *offsets_out,
                    int64_t *os_errno);
typedef struct glm_chunkfile glm_chunkfile;
/* info[8]: status kind, n_rows, n_cols, flags, version, n_chunks, errno;
 * magic_out (8 bytes, may be NULL): the magic read.  *out only when ok. */
int glm_chunk_open(const char *path, glm_chunkfile **out, int64_t *info, char *magic_out);
/* descriptor table (n_chunks each) and the row vector (n_rows, if flagged) */
int glm_chunk_table(const glm_chunkfile *f, int64_t *offsets, int64_t *n_cols, int64_t *nnz,
                    double *row_vector);
int glm_chunk_close(glm_chunkfile *f);
/* one chunk body: indptr i64[n_cols+1] (chunk-relative), rows i32[nnz],
 * vals f64[nnz], labels f64[n_cols] (if has_labels); status[2] = kind, errno */
int glm_chunk_read(const char *path, int64_t offset, int64_t n_cols, int64_t nnz, int has_labels,
                   int64_t *indptr, int32_t *rows, double *vals, double *labels,
                   int64_t *status);

#ifdef __cplusplus
}
#endif
#endif
