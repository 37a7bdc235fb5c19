// stream.cu — the out-of-core training pipeline (sm_100a host runtime).
//
// Replaces pipelined_epoch / chunked_device_runner / _train_chunk
// (pipeline.py:158-340).  The partition's columns are cut into chunks (a
// GLMCHUNK file, data.py:307-431, or column ranges of host CSC arrays).
// Chunks that fit the device budget stay resident in HBM; the rest rotate
// through two device slots:
//
//     loader thread : [read chunk k+2 into pinned staging] -> cudaMemcpyAsync (copy stream)
//     compute stream: [chunk keys -> bucket argsort] -> open -> g-sum -> attempts -> close
//
// The reference's three stages (load / keygen / train, pipeline.py:244-289)
// map to the loader thread + copy engine, the on-device key generator, and
// the chunk solve.  Chunk c+1 is enqueued before the host has checked chunk
// c (its kernels stay no-ops unless c finished, scd.cu chunk_open_kernel),
// so the GPU never waits for the host between chunks; a chunk that needs
// more attempts than enqueued is resumed, and the next chunk re-enqueued.
// Keys are stateless in (seed, epoch, chunk) (pipeline.py:5-9), so the
// result does not depend on the pipeline schedule.
#include <fcntl.h>
#include <unistd.h>

#include <chrono>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "solver.cuh"

namespace glm {

namespace {

constexpr int REC_RING = 64;
constexpr int ATTEMPTS_PER_ENQUEUE = 2;

double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

struct DevChunk {              // a device home for one chunk
    int64_t *indptr = nullptr;
    int32_t *rows = nullptr;
    double *vals = nullptr;
    double *sq = nullptr;
    int64_t cap_cols = 0, cap_nnz = 0;
    int chunk = -1;            // chunk currently held (-1: none)
    int64_t nnz_base = 0;      // indptr values of the held chunk start here
    cudaEvent_t loaded = nullptr;      // end of the H2D copy (timing-enabled)
    cudaEvent_t copy0 = nullptr;       // start of the H2D copy
};

struct LoadJob {
    int64_t seq;
    int chunk;
    int slot;                  // streaming slot
    bool done = false;
    double load_ms = 0.0;      // host read / staging copy
};

}  // namespace
}  // namespace glm

struct glm_stream {
    int device = 0;
    int64_t d = 0, m = 0;
    int n_chunks = 0;
    std::vector<int64_t> col_off;      // chunk c = partition columns [col_off[c], col_off[c+1])
    std::vector<int64_t> nnz;          // per-chunk nnz
    // source
    int src = 0;                       // 0 host arrays, 1 GLMCHUNK file
    const int64_t *h_indptr = nullptr;
    const int32_t *h_rows = nullptr;
    const double *h_vals = nullptr;
    bool direct = false;               // host arrays are pinned: DMA straight from them
    std::vector<void *> registered;    // cudaHostRegister'ed ranges (unregistered on destroy)
    int fd = -1;
    int dfd = -1;                      // O_DIRECT descriptor (glm_stream_set_io), -1 = buffered
    int io_threads = 1;                // concurrent pread stripes per chunk body
    std::string path;
    std::vector<int64_t> foff;         // file offset of chunk c's indptr
    // device
    std::vector<glm::DevChunk> res;    // resident chunks [0, n_res)
    int n_res = 0;
    glm::DevChunk slot[2];             // streaming slots
    int64_t budget = 0, bytes_resident = 0, bytes_slots = 0;
    double *dfull = nullptr, *base = nullptr, *y = nullptr, *lin = nullptr, *cnst = nullptr,
           *dv = nullptr;
    int32_t *perm[2] = {nullptr, nullptr};
    glm_solver *solver = nullptr;
    cudaStream_t cs = nullptr, xs = nullptr;
    glm::ChunkRecord *rec_h = nullptr;
    cudaEvent_t ev_chunk[2] = {nullptr, nullptr};
    cudaEvent_t ev_t0[2] = {nullptr, nullptr}, ev_h2d0[2] = {nullptr, nullptr};
    // pinned staging for pageable / file sources
    char *stage[2] = {nullptr, nullptr};
    int64_t stage_cap = 0;
    cudaEvent_t stage_free[2] = {nullptr, nullptr};
    // loader thread
    std::thread th;
    std::mutex mu;
    std::condition_variable cv;
    std::deque<glm::LoadJob> jobs;     // posted, in order
    std::vector<glm::LoadJob> finished;
    bool quit = false;
    int64_t next_key = 0;              // unique load-job keys across solves
    struct Carry { int chunk, slot; int64_t key; };
    std::vector<Carry> carried;        // loads posted for the next solve's first streamed chunks
    int load_error = 0;
    std::string load_msg;
    // schedule of the last solve: rows of GLM_STREAM_SCHED_COLS doubles
    std::vector<double> sched;
    double totals[8] = {0};
};

namespace glm {
namespace {

int64_t chunk_bytes(int64_t nc, int64_t nz) {
    return 8 * (nc + 1) + 4 * nz + 8 * nz + 8 * nc + 4 * 256;
}

int alloc_chunk(DevChunk &c, int64_t cols, int64_t nz) {
    c.cap_cols = cols;
    c.cap_nnz = nz;
    GLM_CUDA_TRY(cudaMalloc(&c.indptr, sizeof(int64_t) * (cols + 1)));
    GLM_CUDA_TRY(cudaMalloc(&c.rows, sizeof(int32_t) * (nz > 0 ? nz : 1)));
    GLM_CUDA_TRY(cudaMalloc(&c.vals, sizeof(double) * (nz > 0 ? nz : 1)));
    GLM_CUDA_TRY(cudaMalloc(&c.sq, sizeof(double) * (cols > 0 ? cols : 1)));
    GLM_CUDA_TRY(cudaEventCreate(&c.loaded));
    GLM_CUDA_TRY(cudaEventCreate(&c.copy0));
    return GLM_OK;
}

void free_chunk(DevChunk &c) {
    cudaFree(c.indptr);
    cudaFree(c.rows);
    cudaFree(c.vals);
    cudaFree(c.sq);
    if (c.loaded) cudaEventDestroy(c.loaded);
    if (c.copy0) cudaEventDestroy(c.copy0);
    c = DevChunk{};
}

bool pread_all(int fd, void *dst, int64_t bytes, int64_t off) {
    char *p = (char *)dst;
    while (bytes > 0) {
        ssize_t r = pread(fd, p, (size_t)bytes, (off_t)off);
        if (r <= 0) return false;
        p += r;
        bytes -= r;
        off += r;
    }
    return true;
}

// [off, off + len) into dst with `threads` concurrent preads (NVMe wants
// queue depth).  With O_DIRECT the stripes are 4 KiB-aligned and the range
// may run past EOF: `need` bytes must arrive, the rest may come up short.
bool pread_striped(int fd, char *dst, int64_t len, int64_t off, int threads, bool direct,
                   int64_t need) {
    if (threads <= 1 || len < (4 << 20)) {
        if (!direct) return pread_all(fd, dst, len, off);
        int64_t got = 0;
        while (got < len) {
            const ssize_t r = pread(fd, dst + got, (size_t)(len - got), (off_t)(off + got));
            if (r <= 0) break;
            got += r;
        }
        return got >= need;
    }
    int64_t stripe = (len + threads - 1) / threads;
    stripe = (stripe + 4095) & ~(int64_t)4095;
    std::vector<std::thread> th;
    std::vector<int64_t> got(threads, 0);
    auto work = [&](int t) {
        const int64_t a = (int64_t)t * stripe, b = std::min(len, a + stripe);
        int64_t k = 0;
        while (a + k < b) {
            const ssize_t r = pread(fd, dst + a + k, (size_t)(b - a - k), (off_t)(off + a + k));
            if (r <= 0) break;
            k += r;
        }
        got[t] = k;
    };
    for (int t = 1; t < threads; ++t)
        if ((int64_t)t * stripe < len) th.emplace_back(work, t);
    work(0);
    for (auto &x : th) x.join();
    int64_t covered = 0;                       // contiguous bytes from the start
    for (int t = 0; t < threads; ++t) {
        const int64_t a = (int64_t)t * stripe;
        if (a >= len) break;
        const int64_t want = std::min(len, a + stripe) - a;
        covered = a + got[t];
        if (got[t] < want) break;
    }
    return covered >= need;
}

// Copy chunk c into device home `h` on stream `xs` (staging through pinned
// buffer `stage_i` unless the host source is pinned).  Records h.loaded.
int load_chunk(glm_stream *S, int c, DevChunk &h, int stage_i, double *load_ms) {
    const int64_t nc = S->col_off[c + 1] - S->col_off[c];
    const int64_t nz = S->nnz[c];
    const double t0 = now_ms();
    h.chunk = c;
    if (S->src == 0) {
        const int64_t j0 = S->col_off[c];
        const int64_t p0 = S->h_indptr[j0];
        h.nnz_base = p0;
        if (S->direct) {
            GLM_CUDA_TRY(cudaEventRecord(h.copy0, S->xs));
            GLM_CUDA_TRY(cudaMemcpyAsync(h.indptr, S->h_indptr + j0, 8 * (nc + 1),
                                         cudaMemcpyHostToDevice, S->xs));
            if (nz > 0) {
                GLM_CUDA_TRY(cudaMemcpyAsync(h.rows, S->h_rows + p0, 4 * nz,
                                             cudaMemcpyHostToDevice, S->xs));
                GLM_CUDA_TRY(cudaMemcpyAsync(h.vals, S->h_vals + p0, 8 * nz,
                                             cudaMemcpyHostToDevice, S->xs));
            }
        } else {
            GLM_CUDA_TRY(cudaEventSynchronize(S->stage_free[stage_i]));
            char *st = S->stage[stage_i];
            memcpy(st, S->h_indptr + j0, 8 * (nc + 1));
            memcpy(st + 8 * (nc + 1), S->h_rows + p0, 4 * nz);
            memcpy(st + 8 * (nc + 1) + 4 * nz, S->h_vals + p0, 8 * nz);
            *load_ms = now_ms() - t0;
            GLM_CUDA_TRY(cudaEventRecord(h.copy0, S->xs));
            GLM_CUDA_TRY(cudaMemcpyAsync(h.indptr, st, 8 * (nc + 1), cudaMemcpyHostToDevice, S->xs));
            if (nz > 0) {
                GLM_CUDA_TRY(cudaMemcpyAsync(h.rows, st + 8 * (nc + 1), 4 * nz,
                                             cudaMemcpyHostToDevice, S->xs));
                GLM_CUDA_TRY(cudaMemcpyAsync(h.vals, st + 8 * (nc + 1) + 4 * nz, 8 * nz,
                                             cudaMemcpyHostToDevice, S->xs));
            }
            GLM_CUDA_TRY(cudaEventRecord(S->stage_free[stage_i], S->xs));
        }
    } else {
        // GLMCHUNK chunk body (data.py:341-357): indptr u64[nc+1] (chunk-relative),
        // rows u32[nnz], vals f64[nnz] — the same bits as i64 / i32 / f64.
        h.nnz_base = 0;
        GLM_CUDA_TRY(cudaEventSynchronize(S->stage_free[stage_i]));
        char *st = S->stage[stage_i];
        const int64_t body = 8 * (nc + 1) + 12 * nz;
        const int64_t off = S->foff[c];
        if (S->dfd >= 0) {             // O_DIRECT: the aligned superset, the body at an offset
            const int64_t a0 = off & ~(int64_t)4095;
            const int64_t a1 = (off + body + 4095) & ~(int64_t)4095;
            if (!pread_striped(S->dfd, st, a1 - a0, a0, S->io_threads, true, off + body - a0))
                return glm_set_error(GLM_USAGE, "chunk store read failed (truncated file?)");
            st += off - a0;
        } else {
            if (!pread_striped(S->fd, st, body, off, S->io_threads, false, body))
                return glm_set_error(GLM_USAGE, "chunk store read failed (truncated file?)");
            if (c + 1 < S->n_chunks) {  // read-ahead of the next chunk's body
                const int64_t nc1 = S->col_off[c + 2] - S->col_off[c + 1];
                posix_fadvise(S->fd, (off_t)S->foff[c + 1], (off_t)(8 * (nc1 + 1) + 12 * S->nnz[c + 1]),
                              POSIX_FADV_WILLNEED);
            }
        }
        *load_ms = now_ms() - t0;
        GLM_CUDA_TRY(cudaEventRecord(h.copy0, S->xs));
            GLM_CUDA_TRY(cudaMemcpyAsync(h.indptr, st, 8 * (nc + 1), cudaMemcpyHostToDevice, S->xs));
        if (nz > 0) {
            GLM_CUDA_TRY(cudaMemcpyAsync(h.rows, st + 8 * (nc + 1), 4 * nz,
                                         cudaMemcpyHostToDevice, S->xs));
            GLM_CUDA_TRY(cudaMemcpyAsync(h.vals, st + 8 * (nc + 1) + 4 * nz, 8 * nz,
                                         cudaMemcpyHostToDevice, S->xs));
        }
        GLM_CUDA_TRY(cudaEventRecord(S->stage_free[stage_i], S->xs));
    }
    if (S->direct && S->src == 0) *load_ms = 0.0;
    GLM_CUDA_TRY(cudaEventRecord(h.loaded, S->xs));
    return GLM_OK;
}

void loader_main(glm_stream *S) {
    cudaSetDevice(S->device);
    int stage_i = 0;
    for (;;) {
        LoadJob job;
        {
            std::unique_lock<std::mutex> lk(S->mu);
            S->cv.wait(lk, [&] { return S->quit || !S->jobs.empty(); });
            if (S->quit) return;
            job = S->jobs.front();
        }
        double ms = 0.0;
        int rc = load_chunk(S, job.chunk, S->slot[job.slot], stage_i, &ms);
        stage_i ^= 1;
        {
            std::lock_guard<std::mutex> lk(S->mu);
            S->jobs.pop_front();
            job.done = true;
            job.load_ms = ms;
            S->finished.push_back(job);
            if (rc && !S->load_error) {
                S->load_error = rc;
                S->load_msg = glm_last_error();
            }
        }
        S->cv.notify_all();
    }
}

glm_matrix chunk_matrix(const glm_stream *S, const DevChunk &h, int c) {
    glm_matrix A{};
    A.n_rows = S->d;
    A.n_cols = S->col_off[c + 1] - S->col_off[c];
    A.nnz = S->nnz[c];
    A.layout = GLM_CSC;
    A.indptr = h.indptr;
    A.rows = h.rows - h.nnz_base;   // indptr values index the source's arrays
    A.vals = h.vals - h.nnz_base;
    A.sqnorms = h.sq;
    return A;
}

int setup_device(glm_stream *S, int64_t budget) {
    const int C = S->n_chunks;
    int64_t max_cols = 1, max_nnz = 1, max_bytes = 0, total = 0;
    for (int c = 0; c < C; ++c) {
        const int64_t nc = S->col_off[c + 1] - S->col_off[c];
        max_cols = std::max(max_cols, nc);
        max_nnz = std::max(max_nnz, S->nnz[c]);
        max_bytes = std::max(max_bytes, chunk_bytes(nc, S->nnz[c]));
        total += chunk_bytes(nc, S->nnz[c]);
    }
    S->budget = budget;
    // resident prefix: everything if it fits, else as many chunks as leave room
    // for the two streaming slots
    int n_res = 0;
    int64_t used = 0;
    if (budget <= 0 || total <= budget) {
        n_res = C;
        used = total;
    } else {
        const int64_t room = budget - 2 * max_bytes;
        while (n_res < C) {
            const int64_t nc = S->col_off[n_res + 1] - S->col_off[n_res];
            const int64_t b = chunk_bytes(nc, S->nnz[n_res]);
            if (used + b > room) break;
            used += b;
            ++n_res;
        }
    }
    S->n_res = n_res;
    S->bytes_resident = used;
    S->res.resize(n_res);
    for (int c = 0; c < n_res; ++c) {
        int rc = alloc_chunk(S->res[c], S->col_off[c + 1] - S->col_off[c], S->nnz[c]);
        if (rc) return rc;
    }
    if (n_res < C) {
        for (int i = 0; i < 2; ++i) {
            int rc = alloc_chunk(S->slot[i], max_cols, max_nnz);
            if (rc) return rc;
        }
        S->bytes_slots = 2 * max_bytes;
    }
    const size_t m1 = (size_t)(S->m > 0 ? S->m : 1), d1 = (size_t)(S->d > 0 ? S->d : 1);
    GLM_CUDA_TRY(cudaMalloc(&S->dfull, 8 * m1));
    GLM_CUDA_TRY(cudaMalloc(&S->base, 8 * m1));
    GLM_CUDA_TRY(cudaMalloc(&S->y, 8 * m1));
    GLM_CUDA_TRY(cudaMalloc(&S->lin, 8 * d1));
    GLM_CUDA_TRY(cudaMalloc(&S->dv, 8 * d1));
    GLM_CUDA_TRY(cudaMalloc(&S->cnst, 8 * 4));
    for (int i = 0; i < 2; ++i) GLM_CUDA_TRY(cudaMalloc(&S->perm[i], 4 * (size_t)max_cols));
    GLM_CUDA_TRY(cudaStreamCreateWithFlags(&S->cs, cudaStreamNonBlocking));
    GLM_CUDA_TRY(cudaStreamCreateWithFlags(&S->xs, cudaStreamNonBlocking));
    GLM_CUDA_TRY(cudaHostAlloc(&S->rec_h, sizeof(ChunkRecord) * REC_RING, cudaHostAllocMapped));
    memset(S->rec_h, 0xff, sizeof(ChunkRecord) * REC_RING);
    for (int i = 0; i < 2; ++i) {
        GLM_CUDA_TRY(cudaEventCreate(&S->ev_chunk[i]));
        GLM_CUDA_TRY(cudaEventCreate(&S->ev_t0[i]));
        GLM_CUDA_TRY(cudaEventCreate(&S->ev_h2d0[i]));
        GLM_CUDA_TRY(cudaEventCreateWithFlags(&S->stage_free[i], cudaEventDisableTiming));
    }
    if (!S->direct || S->src == 1) {
        // + 8 KiB: an O_DIRECT read covers the body's aligned superset
        S->stage_cap = max_bytes + (S->src == 1 ? 8192 : 0);
        for (int i = 0; i < 2; ++i)
            GLM_CUDA_TRY(cudaHostAlloc((void **)&S->stage[i], (size_t)S->stage_cap,
                                       cudaHostAllocDefault));
    }
    int rc = glm_solver_create(S->device, max_cols, S->d, &S->solver);
    if (rc) return rc;
    GLM_CUDA_TRY(cudaSetDevice(S->device));
    // resident chunks: load once, column norms once
    for (int c = 0; c < n_res; ++c) {
        double ms = 0.0;
        rc = load_chunk(S, c, S->res[c], c & 1, &ms);
        if (rc) return rc;
        GLM_CUDA_TRY(cudaStreamWaitEvent(S->cs, S->res[c].loaded, 0));
        glm_matrix A = chunk_matrix(S, S->res[c], c);
        rc = launch_colwise(&A, 0, nullptr, S->res[c].sq, S->cs);
        if (rc) return rc;
    }
    GLM_CUDA_TRY(cudaStreamSynchronize(S->xs));
    GLM_CUDA_TRY(cudaStreamSynchronize(S->cs));
    if (n_res < C) S->th = std::thread(loader_main, S);
    return GLM_OK;
}

}  // namespace
}  // namespace glm

using namespace glm;

extern "C" {

int glm_stream_destroy(glm_stream *S) {
    if (!S) return GLM_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(S->device);
    if (S->th.joinable()) {
        {
            std::lock_guard<std::mutex> lk(S->mu);
            S->quit = true;
        }
        S->cv.notify_all();
        S->th.join();
    }
    if (S->cs) cudaStreamSynchronize(S->cs);
    if (S->xs) cudaStreamSynchronize(S->xs);
    glm_solver_destroy(S->solver);
    for (auto &c : S->res) free_chunk(c);
    for (auto &c : S->slot) free_chunk(c);
    void *ptrs[] = {S->dfull, S->base, S->y, S->lin, S->cnst, S->dv, S->perm[0], S->perm[1]};
    for (void *p : ptrs) cudaFree(p);
    for (int i = 0; i < 2; ++i) {
        if (S->stage[i]) cudaFreeHost(S->stage[i]);
        cudaEvent_t evs[] = {S->ev_chunk[i], S->ev_t0[i], S->ev_h2d0[i], S->stage_free[i]};
        for (cudaEvent_t e : evs)
            if (e) cudaEventDestroy(e);
    }
    if (S->rec_h) cudaFreeHost(S->rec_h);
    for (void *p : S->registered) cudaHostUnregister(p);
    if (S->cs) cudaStreamDestroy(S->cs);
    if (S->xs) cudaStreamDestroy(S->xs);
    if (S->fd >= 0) close(S->fd);
    if (S->dfd >= 0) close(S->dfd);
    cudaSetDevice(prev);
    delete S;
    return GLM_OK;
}

int glm_stream_create_host(int device, int64_t n_rows, int64_t n_cols, const int64_t *indptr,
                           const int32_t *rows, const double *vals, int n_chunks,
                           const int64_t *col_offsets, int64_t device_budget, int pin_host,
                           glm_stream **out) {
    if (!out || !indptr || !rows || !vals || !col_offsets || n_chunks < 0 || n_rows < 0 ||
        n_cols < 0)
        return glm_set_error(GLM_USAGE, "bad stream arguments");
    if (col_offsets[0] != 0 || col_offsets[n_chunks] != n_cols)
        return glm_set_error(GLM_USAGE, "chunk offsets must span [0, n_cols]");
    for (int c = 0; c < n_chunks; ++c)
        if (col_offsets[c + 1] < col_offsets[c])
            return glm_set_error(GLM_USAGE, "chunk offsets must be non-decreasing");
    GLM_CUDA_TRY(cudaSetDevice(device));
    glm_stream *S = new (std::nothrow) glm_stream();
    if (!S) return glm_set_error(GLM_USAGE, "out of host memory");
    S->device = device;
    S->d = n_rows;
    S->m = n_cols;
    S->n_chunks = n_chunks;
    S->col_off.assign(col_offsets, col_offsets + n_chunks + 1);
    S->nnz.resize(n_chunks);
    for (int c = 0; c < n_chunks; ++c)
        S->nnz[c] = indptr[col_offsets[c + 1]] - indptr[col_offsets[c]];
    S->src = 0;
    S->h_indptr = indptr;
    S->h_rows = rows;
    S->h_vals = vals;
    const int64_t nz = indptr[n_cols];
    auto is_pinned = [](const void *p) {
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return at.type == cudaMemoryTypeHost;
    };
    S->direct = is_pinned(indptr) && is_pinned(rows) && is_pinned(vals);
    if (!S->direct && pin_host) {
        struct R { const void *p; size_t b; } rs[] = {{indptr, (size_t)8 * (n_cols + 1)},
                                                     {rows, (size_t)4 * (nz > 0 ? nz : 1)},
                                                     {vals, (size_t)8 * (nz > 0 ? nz : 1)}};
        bool ok = true;
        for (auto &r : rs) {
            if (is_pinned(r.p)) continue;
            if (cudaHostRegister((void *)r.p, r.b, cudaHostRegisterReadOnly) != cudaSuccess) {
                cudaGetLastError();
                ok = false;
                break;
            }
            S->registered.push_back((void *)r.p);
        }
        S->direct = ok;
    }
    int rc = setup_device(S, device_budget);
    if (rc) {
        glm_stream_destroy(S);
        return rc;
    }
    *out = S;
    return GLM_OK;
}

int glm_stream_create_file(int device, const char *path, int64_t n_rows, int n_chunks,
                           const int64_t *chunk_offsets, const int64_t *chunk_cols,
                           const int64_t *chunk_nnz, int64_t device_budget, glm_stream **out) {
    if (!out || !path || n_chunks < 0 || n_rows < 0 || (n_chunks > 0 && (!chunk_offsets ||
                                                                          !chunk_cols ||
                                                                          !chunk_nnz)))
        return glm_set_error(GLM_USAGE, "bad stream arguments");
    GLM_CUDA_TRY(cudaSetDevice(device));
    glm_stream *S = new (std::nothrow) glm_stream();
    if (!S) return glm_set_error(GLM_USAGE, "out of host memory");
    S->device = device;
    S->d = n_rows;
    S->n_chunks = n_chunks;
    S->src = 1;
    S->col_off.assign(1, 0);
    for (int c = 0; c < n_chunks; ++c) {
        S->col_off.push_back(S->col_off.back() + chunk_cols[c]);
        S->nnz.push_back(chunk_nnz[c]);
        S->foff.push_back(chunk_offsets[c] + 12);   // skip the <IQ chunk head (data.py:341)
    }
    S->m = S->col_off.back();
    S->path = path;
    S->fd = open(path, O_RDONLY);
    if (S->fd < 0) {
        glm_stream_destroy(S);
        return glm_set_error(GLM_USAGE, "cannot open chunk store");
    }
    int rc = setup_device(S, device_budget);
    if (rc) {
        glm_stream_destroy(S);
        return rc;
    }
    *out = S;
    return GLM_OK;
}

int glm_stream_set_io(glm_stream *S, int direct_io, int io_threads) {
    if (!S) return glm_set_error(GLM_USAGE, "null stream");
    if (S->src != 1) return glm_set_error(GLM_USAGE, "I/O options apply to GLMCHUNK file streams");
    S->io_threads = io_threads < 1 ? 1 : (io_threads > 32 ? 32 : io_threads);
    if (S->dfd >= 0) {
        close(S->dfd);
        S->dfd = -1;
    }
    // the file system may not support O_DIRECT (tmpfs): buffered reads then,
    // reported by glm_stream_info out[7]
    if (direct_io) S->dfd = open(S->path.c_str(), O_RDONLY | O_DIRECT);
    return GLM_OK;
}

int glm_stream_info(const glm_stream *S, int64_t *out) {
    if (!S || !out) return glm_set_error(GLM_USAGE, "null argument");
    out[0] = S->n_chunks;
    out[1] = S->n_res;
    out[2] = S->bytes_resident;
    out[3] = S->bytes_slots;
    out[4] = S->direct ? 1 : 0;
    out[5] = S->m;
    out[6] = S->d;
    out[7] = S->dfd >= 0 ? 1 : 0;
    return GLM_OK;
}

int glm_stream_solve(glm_stream *S, const glm_stream_args *a, double *damping_io,
                     double *delta_io, double *view_io, double *dv_out, double *values_out,
                     int32_t *info_out, double *scal_out) {
    if (!S || !a || !a->lin || !a->base || !damping_io || !delta_io)
        return glm_set_error(GLM_USAGE, "null argument to glm_stream_solve");
    if (a->epochs < 1) return glm_set_error(GLM_USAGE, "t_epochs must be >= 1");
    if (a->kind < 0 || a->kind > GLM_HINGE_PRIMAL)
        return glm_set_error(GLM_USAGE, "unknown objective kind");
    if (!(a->quad > 0.0)) return glm_set_error(GLM_USAGE, "quad must be positive");
    if (a->kind == GLM_DUAL_RIDGE && !a->coord_target)
        return glm_set_error(GLM_USAGE, "dual_ridge needs per-coordinate targets");
    GLM_CUDA_TRY(cudaSetDevice(S->device));
    {
        std::lock_guard<std::mutex> lk(S->mu);
        if (S->load_error) return glm_set_error(S->load_error, S->load_msg.c_str());
    }
    const int64_t m = S->m, d = S->d;
    const int C = S->n_chunks;
    cudaStream_t cs = S->cs;
    struct Drain {   // failed solve: let the loader finish, forget its results
        glm_stream *S;
        bool ok = false;
        ~Drain() {
            if (ok) return;   // loads carried into the next solve keep running
            std::unique_lock<std::mutex> lk(S->mu);
            S->cv.wait(lk, [&] { return S->jobs.empty() || S->quit; });
            S->finished.clear();
            S->carried.clear();
            lk.unlock();
            cudaStreamSynchronize(S->xs);
            cudaStreamSynchronize(S->cs);
        }
    } drain{S};
    const bool delta_in = (a->flags & GLM_STREAM_DELTA_IN) != 0;
    const bool view_in = view_io && (a->flags & GLM_STREAM_VIEW_IN) != 0;
    if (d > 0) GLM_CUDA_TRY(cudaMemcpyAsync(S->lin, a->lin, 8 * d, cudaMemcpyDefault, cs));
    if (m > 0) GLM_CUDA_TRY(cudaMemcpyAsync(S->base, a->base, 8 * m, cudaMemcpyDefault, cs));
    if (a->coord_target && m > 0)
        GLM_CUDA_TRY(cudaMemcpyAsync(S->y, a->coord_target, 8 * m, cudaMemcpyDefault, cs));
    if (delta_in && m > 0)
        GLM_CUDA_TRY(cudaMemcpyAsync(S->dfull, delta_io, 8 * m, cudaMemcpyDefault, cs));
    if (view_in && d > 0)
        GLM_CUDA_TRY(cudaMemcpyAsync(S->solver->view[0], view_io, 8 * d, cudaMemcpyDefault, cs));
    double cn = a->cnst;
    GLM_CUDA_TRY(cudaMemcpyAsync(S->cnst, &cn, 8, cudaMemcpyHostToDevice, cs));

    StreamSolve sa{};
    sa.kind = a->kind;
    sa.mode = a->mode;
    sa.lam = a->lam;
    sa.rho = a->l1_ratio;
    sa.quad = a->quad;
    sa.cnst = S->cnst;
    sa.lin = S->lin;
    sa.base = S->base;
    sa.y = a->coord_target ? S->y : nullptr;
    sa.dfull = S->dfull;
    sa.m = m;
    sa.d = d;
    sa.group_lanes = a->group_lanes;
    sa.max_inflight = a->max_inflight;
    sa.flags = a->flags & 3;
    int rc = stream_begin(S->solver, sa, !delta_in, view_in, *damping_io, cs);
    if (rc) return rc;

    const int timing = (a->flags & GLM_STREAM_TIMING) != 0;
    S->sched.clear();
    const int64_t total = (int64_t)a->epochs * C;
    const int attempts = a->attempts_per_chunk > 0 ? a->attempts_per_chunk : ATTEMPTS_PER_ENQUEUE;
    std::vector<ChunkJob> jobs(total > 0 ? (size_t)total : 1);
    std::vector<glm_matrix> mats(jobs.size());
    std::vector<int> slot_of(jobs.size(), -1);
    std::vector<double> load_ms(jobs.size(), 0.0);

    // the streamed chunks in sequence order, and the loads posted so far
    std::vector<int64_t> streamed;
    for (int64_t q = 0; q < total; ++q)
        if ((int)(q % C) >= S->n_res) streamed.push_back(q);
    size_t next_post = 0;
    int free_slots[2] = {1, 1};
    std::vector<int64_t> key_of(jobs.size(), -1);
    auto wait_key = [&](int64_t key, double *ms) -> int {
        std::unique_lock<std::mutex> lk(S->mu);
        for (;;) {
            if (S->load_error) return glm_set_error(S->load_error, S->load_msg.c_str());
            for (size_t i = 0; i < S->finished.size(); ++i)
                if (S->finished[i].seq == key) {
                    if (ms) *ms = S->finished[i].load_ms;
                    S->finished.erase(S->finished.begin() + i);
                    return GLM_OK;
                }
            S->cv.wait(lk);
        }
    };
    {   // loads the previous solve posted ahead become this solve's first streamed chunks
        std::vector<glm_stream::Carry> carried;
        {
            std::lock_guard<std::mutex> lk(S->mu);
            carried.swap(S->carried);
        }
        for (const auto &cj : carried) {
            if (next_post < streamed.size() && (int)(streamed[next_post] % C) == cj.chunk) {
                const int64_t q = streamed[next_post++];
                slot_of[q] = cj.slot;
                key_of[q] = cj.key;
                free_slots[cj.slot] = 0;
            } else {
                int r = wait_key(cj.key, nullptr);   // a stale carry: let it land first
                if (r) return r;
            }
        }
    }
    auto post_loads = [&]() {
        std::lock_guard<std::mutex> lk(S->mu);
        while (next_post < streamed.size()) {
            int sl = free_slots[0] ? 0 : (free_slots[1] ? 1 : -1);
            if (sl < 0) break;
            free_slots[sl] = 0;
            const int64_t q = streamed[next_post++];
            slot_of[q] = sl;
            key_of[q] = S->next_key++;
            LoadJob j;
            j.seq = key_of[q];
            j.chunk = (int)(q % C);
            j.slot = sl;
            S->jobs.push_back(j);
        }
        S->cv.notify_all();
    };
    auto wait_loaded = [&](int64_t q) -> int { return wait_key(key_of[q], &load_ms[q]); };
    const double t_solve0 = now_ms();
    double h2d_wait_ms = 0.0;
    auto enqueue = [&](int64_t q, bool fresh) -> int {
        const int c = (int)(q % C);
        const int e = (int)(q / C);
        ChunkJob &j = jobs[q];
        DevChunk *h;
        if (c < S->n_res) {
            h = &S->res[c];
        } else {
            h = &S->slot[slot_of[q]];
            if (fresh) {
                const double tw = now_ms();
                int r = wait_loaded(q);
                h2d_wait_ms += now_ms() - tw;
                if (r) return r;
                GLM_CUDA_TRY(cudaStreamWaitEvent(cs, h->loaded, 0));
            }
        }
        if (timing && fresh) GLM_CUDA_TRY(cudaEventRecord(S->ev_t0[q & 1], cs));
        mats[q] = chunk_matrix(S, *h, c);
        if (fresh && c >= S->n_res) {   // column norms of a freshly streamed chunk
            int r = launch_colwise(&mats[q], 0, nullptr, h->sq, cs);
            if (r) return r;
        }
        j.A = &mats[q];
        j.lo = S->col_off[c];
        j.seq = q;
        const uint64_t ix[2] = {a->epoch_index + (uint64_t)e, (uint64_t)c};
        j.key_seed = glm_derive_seed(a->seed, ix, 2);
        j.perm = S->perm[q & 1];
        j.gen_perm = fresh;
        j.open = true;
        j.attempts = attempts;
        j.rec = S->rec_h + (q % REC_RING);
        int r = chunk_enqueue(S->solver, sa, j, cs);
        if (r) return r;
        GLM_CUDA_TRY(cudaEventRecord(S->ev_chunk[q & 1], cs));
        return GLM_OK;
    };
    auto read_rec = [&](int64_t q) -> ChunkRecord {
        volatile ChunkRecord *r = S->rec_h + (q % REC_RING);
        ChunkRecord out;
        out.seq = r->seq;
        out.cur = r->cur;
        out.done = r->done;
        out.status = r->status;
        out.retries = r->retries;
        out.attempts = r->attempts;
        out.plateaued = r->plateaued;
        out.accepted = r->accepted;
        out.damping = r->damping;
        out.value = r->value;
        return out;
    };

    int epochs_done = 0, plateaued = 0;
    post_loads();
    if (total > 0) {
        rc = enqueue(0, true);
        if (rc) return rc;
    }
    for (int64_t q = 0; q < total; ++q) {
        if (q + 1 < total) {               // speculative: runs only if q finishes in time
            rc = enqueue(q + 1, true);
            if (rc) return rc;
        }
        GLM_CUDA_TRY(cudaEventSynchronize(S->ev_chunk[q & 1]));
        ChunkRecord r = read_rec(q);
        int guard = 0;
        while (r.seq == q && r.status == GLM_OK && !r.done) {
            // chunk q needs more attempts: let the speculative q+1 drain (its
            // kernels were no-ops), resume q, then re-enqueue q+1
            if (q + 1 < total) GLM_CUDA_TRY(cudaEventSynchronize(S->ev_chunk[(q + 1) & 1]));
            ChunkJob more = jobs[q];
            more.gen_perm = false;
            more.open = false;
            more.attempts = 2 * attempts;
            rc = chunk_enqueue(S->solver, sa, more, cs);
            if (rc) return rc;
            GLM_CUDA_TRY(cudaEventRecord(S->ev_chunk[q & 1], cs));
            GLM_CUDA_TRY(cudaEventSynchronize(S->ev_chunk[q & 1]));
            r = read_rec(q);
            if (r.done && q + 1 < total) {
                ChunkJob nx = jobs[q + 1];
                nx.gen_perm = false;
                rc = chunk_enqueue(S->solver, sa, nx, cs);
                if (rc) return rc;
                GLM_CUDA_TRY(cudaEventRecord(S->ev_chunk[(q + 1) & 1], cs));
            }
            if (++guard > 64) break;
        }
        if (r.seq != q || r.status != GLM_OK || !r.done) {
            cudaStreamSynchronize(cs);
            if (r.seq == q && r.status == GLM_DIVERGENCE)
                return glm_set_error(GLM_DIVERGENCE, "damping floor reached during chunked epoch");
            if (r.seq == q && r.status != GLM_OK)
                return glm_set_error(r.status, "non-finite entries in shared view or coordinate update");
            return glm_set_error(GLM_CUDA_ERROR, "chunk pipeline lost track of the device state");
        }
        plateaued += r.plateaued;
        const int c = (int)(q % C);
        if (timing) {
            float tr = 0.f, th = 0.f;
            cudaEventElapsedTime(&tr, S->ev_t0[q & 1], S->ev_chunk[q & 1]);
            if (c >= S->n_res) {
                const DevChunk &h = S->slot[slot_of[q]];
                cudaEventElapsedTime(&th, h.copy0, h.loaded);
            }
            S->sched.insert(S->sched.end(), {(double)(q / C), (double)c, load_ms[q], (double)th,
                                             (double)tr, now_ms() - t_solve0});
        }
        if (c >= S->n_res) {              // chunk q finished: its slot takes the next load
            free_slots[slot_of[q]] = 1;
            post_loads();
        }
        if (c == C - 1) {
            if (epochs_done < a->epochs && values_out) values_out[epochs_done] = r.value;
            ++epochs_done;
        }
    }
    if (C == 0) {
        GLM_CUDA_TRY(cudaStreamSynchronize(cs));
        epochs_done = a->epochs;
    }
    rc = stream_finalize(S->solver, sa, dv_out ? S->dv : nullptr, cs);
    if (rc) return rc;
    if (m > 0) GLM_CUDA_TRY(cudaMemcpyAsync(delta_io, S->dfull, 8 * m, cudaMemcpyDefault, cs));
    if (dv_out && d > 0) GLM_CUDA_TRY(cudaMemcpyAsync(dv_out, S->dv, 8 * d, cudaMemcpyDefault, cs));
    glm_solve_result res{};
    rc = read_result(S->solver, &res, nullptr, 0, cs);   // synchronises cs
    if (rc) return rc;
    if (view_io && d > 0)
        GLM_CUDA_TRY(cudaMemcpy(view_io, S->solver->st_host->vw ? S->solver->view[1]
                                                                : S->solver->view[0],
                                8 * d, cudaMemcpyDefault));
    if (C == 0 && values_out)
        for (int e = 0; e < a->epochs; ++e) values_out[e] = res.initial_value;
    *damping_io = res.damping;
    if (info_out) {
        info_out[0] = epochs_done;
        info_out[1] = res.retries;
        info_out[2] = plateaued;
        info_out[3] = res.attempts;
        info_out[4] = res.status;
    }
    if (scal_out) {
        scal_out[0] = res.initial_value;
        scal_out[1] = res.final_value;
        scal_out[2] = now_ms() - t_solve0;
        scal_out[3] = h2d_wait_ms;
    }
    if (S->n_res < C) {
        // The next solve (the next outer round) starts with the same streamed
        // chunks: load them now, while the caller folds, exchanges and rebuilds
        // its model, so the next solve's first chunks need no wait.
        std::lock_guard<std::mutex> lk(S->mu);
        const int first = S->n_res, second = S->n_res + 1 < C ? S->n_res + 1 : S->n_res;
        const int ch[2] = {first, second};
        for (int i = 0; i < 2; ++i) {
            LoadJob j;
            j.seq = S->next_key++;
            j.chunk = ch[i];
            j.slot = i;
            S->jobs.push_back(j);
            S->carried.push_back({ch[i], i, j.seq});
        }
        S->cv.notify_all();
    }
    drain.ok = true;
    return GLM_OK;
}

int glm_stream_schedule(const glm_stream *S, double *out, int capacity_rows, int *n_rows_out) {
    if (!S || !n_rows_out) return glm_set_error(GLM_USAGE, "null argument");
    const int rows = (int)(S->sched.size() / GLM_STREAM_SCHED_COLS);
    *n_rows_out = rows;
    if (out)
        for (int i = 0; i < rows && i < capacity_rows; ++i)
            for (int k = 0; k < GLM_STREAM_SCHED_COLS; ++k)
                out[i * GLM_STREAM_SCHED_COLS + k] = S->sched[i * GLM_STREAM_SCHED_COLS + k];
    return GLM_OK;
}

}  // extern "C"
