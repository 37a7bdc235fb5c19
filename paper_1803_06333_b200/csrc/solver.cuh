// solver.cuh — solver object and kernel-launch entry points shared by the
// C-ABI translation units.
#pragma once
#include "common.cuh"
#include "prng.cuh"

#include <array>
#include <vector>

struct glm_solver {
    int device = 0;
    // the async epoch after a round turn releases the next turn at its start
    // (set by glm_round_turn: 1 rank) instead of at its end
    int early_trigger = 0;
    int64_t max_coords = 0, max_rows = 0;
    glm::SolveState *st = nullptr;        // device
    glm::SolveState *st_host = nullptr;   // pinned mirror
    double *delta[2] = {nullptr, nullptr};
    double *view[2] = {nullptr, nullptr};
    int32_t *perm = nullptr;
    void *perm_mem = nullptr;
    double *partials = nullptr;           // value-kernel block partials
    double *gpart = nullptr;              // epoch-kernel block partial g-sums
    double *scratch = nullptr;            // generic reduction scratch
    double *vpad = nullptr;               // slice-spread view of the narrow async kernel
    int timing = 0;                       // record per-attempt CUDA events
    cudaStream_t side = nullptr;          // permutation prefetch stream
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool prefetched = false;              // a buffer holds the next solve's attempt 0
    int64_t prefetch_m = 0;
    bool prefetch_alt = false;            // ... in the other buffer (early prefetch)
    int32_t *perm_b = nullptr;            // second permutation buffer
    int perm_cur = 0;                     // 0: perm, 1: perm_b
    bool host_known = false;              // host_gen == the device's next start state
    uint64_t host_gen = 0;
    std::vector<std::array<cudaEvent_t, 4>> events, event_pool;
    // glue timing: {kind (0 finalize, 1 round start), start, end}
    std::vector<std::pair<int, std::array<cudaEvent_t, 2>>> glue_events;
    std::vector<std::array<cudaEvent_t, 2>> glue_pool;
    int last_epochs = 0;
    int64_t last_m = 0;
    const double *sq_src = nullptr;       // mean |a|^2 cache (narrow dense budget)
    int64_t sq_n = -1;
    double sq_mean = 1.0;
    // packed coordinate records of a prepared CSC partition (glm_solver_prepare):
    // {start | count << 40, |a_j|^2} — 16 bytes, one sector per coordinate
    longlong2 *meta = nullptr;
    const int64_t *meta_indptr = nullptr;
    const double *meta_sq = nullptr;
    int64_t meta_m = -1;
};

namespace glm {

constexpr int VALUE_THREADS = 256;
constexpr size_t REDUCE_SCRATCH_BYTES = 64 * 1024;

// Host destinations of the solve's outputs (glm_device_solve): with these the
// adaptive solve enqueues finalize + the copies after each batch of attempts,
// before its one synchronisation, so an accepted batch costs a single host
// round trip (a rejected one re-runs the idempotent finalize and copies).
struct HostCopies {
    double *delta = nullptr;   // f64[m]
    double *dv = nullptr;      // f64[d]
};

int solve(glm_solver *s, const glm_matrix *A, const glm_solve_args *a, double *delta_out,
          double *dv_out, glm_solve_result *res, cudaStream_t stream,
          const HostCopies *hc = nullptr);
int read_result(glm_solver *s, glm_solve_result *res, double *epoch_values, int cap,
                cudaStream_t stream);
// fill res / epoch_values from the state last copied to the host
void fill_result(const glm_solver *s, glm_solve_result *res, double *epoch_values, int cap);
int set_state(glm_solver *s, uint64_t gen_state, double damping, cudaStream_t stream);
// After set_state: generate the solve's attempt-0 permutation on the side
// stream now (e.g. under the caller's host->device input copies).
int prefetch_first_perm(glm_solver *s, int64_t m, cudaStream_t stream);
int join_prefetch(glm_solver *s, cudaStream_t stream);
// record the start of a timed glue kernel (returns the pair to close with glue_end)
int glue_begin(glm_solver *s, int kind, cudaStream_t stream);
int glue_end(glm_solver *s, cudaStream_t stream);
int peer_finalize(glm_solver *s, glm_peer *pr, const double *lin, double quad, int64_t m,
                  int64_t d, double *alpha, int box, int next_known, uint64_t next_state,
                  cudaStream_t stream);

// ---- chunked (out-of-core) solves: stream.cu drives these per chunk.
struct ChunkRecord {          // written by the close kernel into host-mapped memory
    int64_t seq;              // chunk sequence number this record answers (written last)
    int64_t cur;              // chunk open on the device when written
    int32_t done, status, retries, attempts, plateaued, accepted;
    double damping, value;
};

struct StreamSolve {          // partition-wide arguments (device pointers)
    int kind, mode;
    double lam, rho, quad;
    const double *cnst;       // device scalar
    const double *lin;        // f64[d]
    const double *base;       // f64[m]
    const double *y;          // f64[m] or null
    double *dfull;            // f64[m] partition delta (accepted state)
    int64_t m, d;
    int group_lanes, max_inflight, flags;
};

struct ChunkJob {
    const glm_matrix *A;      // chunk matrix (columns lo .. lo + n_cols of the partition)
    int64_t lo;
    int64_t seq;              // epoch * n_chunks + chunk
    uint64_t key_seed;        // derive_seed(seed, epoch_index, chunk) (pipeline.py:226-227)
    int32_t *perm;
    bool gen_perm, open;
    int attempts;
    ChunkRecord *rec;         // host-mapped
};

int stream_begin(glm_solver *s, const StreamSolve &a, bool zero_delta, bool keep_view,
                 double damping, cudaStream_t stream);
int chunk_enqueue(glm_solver *s, const StreamSolve &a, const ChunkJob &c, cudaStream_t stream);
int stream_finalize(glm_solver *s, const StreamSolve &a, double *dv_out, cudaStream_t stream);

}  // namespace glm
