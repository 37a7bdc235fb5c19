// peer.cu — the Delta v exchange of one CoCoA round fused with the next
// round's start, over NVLink peer memory (one process per GPU).
//
// Reference: the round's only collective, allreduce_sum(v_bar) with the
// ascending-rank fold of canonical_sum (engine.py:282, comm.py:41-46, 83-98),
// followed by v += total (engine.py:306) and the next round's outer/inner
// model (engine.py:271-272, 242-250, 148-166) and solve start (solver.py:
// 268-270).  Here:
//
//   finalize (rank r):  alpha += delta; dv_r[b] = B delta; publish  flag_r = R+1
//   round start:        wait flag_j >= R for all j (acquire, system scope);
//                       v += sum_j dv_j[b] in ascending rank order (the bits of
//                       canonical_sum on every rank); grad = f'(v); lin = grad;
//                       view = lin; f(v); solver state reset (begin)
//
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
    char *mem = nullptr;          // [ctl: 8 x i64 | pad to 256 B | dv: 2 x d doubles]
    int64_t *ctl = nullptr;       // [0] published rounds, [1] consumed, [2] block counter
    double *dv = nullptr;
    double **bufs_dev = nullptr;  // world pointers to each rank's dv (device array)
    int64_t **flags_dev = nullptr;
    std::vector<void *> opened;   // cudaIpc-opened peer allocations
    cudaIpcMemHandle_t handle{};
};

namespace glm {

constexpr int PEER_BLOCKS = 2 * NUM_SMS;
constexpr int PEER_THREADS = 256;

__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t *p) {
    int64_t v;
    asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(int64_t *p, int64_t v) {
    asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Finalize of a solve whose Delta v goes to the peer exchange: alpha += delta
// (kept in the SVM box), dv_r[(R+1)&1] = (view - lin)/quad, the generator
// jump, and — once every block is done — flag_r = R+1.
__global__ void __launch_bounds__(PEER_THREADS) peer_finalize_kernel(
    SolveState *st, const double *delta0, const double *delta1, const double *view0,
    const double *view1, const double *lin, double quad, int64_t m, int64_t d, double *alpha,
    int box, double *dv, int64_t *ctl) {
    __shared__ int s_last;
    const int dc = st->dc;
    const double *dl = dc < 0 ? nullptr : (dc ? delta1 : delta0);
    const double *V = st->vw ? view1 : view0;
    const int64_t R = ctl[0];
    double *out = dv + ((R + 1) & 1) * d;
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
        const uint64_t g = warp_jump(st->gen_state, (uint64_t)st->attempts * (uint64_t)m);
        if (threadIdx.x == 0) st->gen_next = g;
    }
    __syncthreads();
    if (threadIdx.x == 0) {     // the block's writes (observed through the barrier)
        __threadfence_system(); // before its arrival; the last block then releases
        s_last = atomicAdd(reinterpret_cast<unsigned long long *>(ctl + 2), 1ull) ==
                 (unsigned long long)(gridDim.x - 1);
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        ctl[2] = 0;
        __threadfence_system();
        st_release_sys(ctl, R + 1);
    }
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
    int64_t *const *flags;
    int64_t *ctl;
    SolveState *st;            // mode 2
    double *view0, *view1;
    int epochs;
    double *scratch;
};

__global__ void __launch_bounds__(PEER_THREADS) round_start_kernel(RoundStart p) {
    __shared__ int s_apply;
    __shared__ int64_t s_R;
    if (threadIdx.x == 0) {
        const int64_t R = p.ctl[0], C = p.ctl[1];
        s_R = R;
        s_apply = R > C;
        if (R > C)
            for (int j = 0; j < p.world; ++j)
                while (ld_acquire_sys(p.flags[j]) < R) __nanosleep(64);
    }
    __syncthreads();
    const int apply = s_apply;
    const int64_t off = (s_R & 1) * p.d;
    double acc[1] = {0.0};
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const bool dual = kind_is_dual(p.kind);
    for (int64_t r = tid; r < p.d; r += nth) {
        double x = p.v[r];
        if (apply) {
            double s = 0.0;                       // canonical_sum: ascending rank order
            for (int j = 0; j < p.world; ++j) s += __ldcg(p.bufs[j] + off + r);
            x += s;
            p.v[r] = x;
        }
        if (p.mode == 0) continue;
        double f, g;                              // outer_model_kernel's arithmetic
        if (dual) {
            f = x * x;
            g = x / p.lam;
        } else {
            f_terms(p.kind, p.lam, p.tgt[r], x, f, g);
            if (p.kind != GLM_LOGISTIC_PRIMAL) f *= 2.0;
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
        if (blockIdx.x == 0 && threadIdx.x == 0 && apply) p.ctl[1] = s_R;
        return;
    }
    if (!reduce_last<1>(acc, p.scratch)) return;
    double f = acc[0];
    if (dual) f = f / (2.0 * p.lam);
    else if (p.kind != GLM_LOGISTIC_PRIMAL) f = 0.5 * f;
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

__global__ void peer_consume_kernel(int64_t *ctl) { ctl[1] = ctl[0]; }

int peer_finalize(glm_solver *s, glm_peer *pr, const double *lin, double quad, int64_t m,
                  int64_t d, double *alpha, int box, cudaStream_t stream) {
    if (pr->d != d) return glm_set_error(GLM_USAGE, "peer exchange sized for another d");
    count_launch();
    int64_t blocks = ((m > d ? m : d) + 4 * PEER_THREADS - 1) / (4 * PEER_THREADS);
    blocks = blocks < 1 ? 1 : (blocks > 8 * NUM_SMS ? 8 * NUM_SMS : blocks);
    peer_finalize_kernel<<<(int)blocks, PEER_THREADS, 0, stream>>>(
        s->st, s->delta[0], s->delta[1], s->view[0], s->view[1], lin, quad, m, d, alpha, box,
        pr->dv, pr->ctl);
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
    cudaSetDevice(prev);
    delete p;
    return GLM_OK;
}

int glm_peer_create(int device, int64_t d, int rank, int world, glm_peer **out) {
    if (!out || d < 0 || world < 1 || rank < 0 || rank >= world)
        return glm_set_error(GLM_USAGE, "bad peer arguments");
    GLM_CUDA_TRY(cudaSetDevice(device));
    glm_peer *p = new (std::nothrow) glm_peer();
    if (!p) return glm_set_error(GLM_USAGE, "out of host memory");
    p->device = device;
    p->rank = rank;
    p->world = world;
    p->d = d;
    const size_t bytes = 256 + sizeof(double) * 2 * (size_t)(d > 0 ? d : 1);
    cudaError_t e = cudaMalloc(&p->mem, bytes);
    if (e == cudaSuccess) e = cudaMemset(p->mem, 0, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&p->bufs_dev, sizeof(double *) * world);
    if (e == cudaSuccess) e = cudaMalloc(&p->flags_dev, sizeof(int64_t *) * world);
    if (e == cudaSuccess && world > 1) e = cudaIpcGetMemHandle(&p->handle, p->mem);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        glm_peer_destroy(p);
        return glm_set_cuda_error(e, "glm_peer_create", __FILE__, __LINE__);
    }
    p->ctl = reinterpret_cast<int64_t *>(p->mem);
    p->dv = reinterpret_cast<double *>(p->mem + 256);
    if (world == 1) {
        double *b = p->dv;
        int64_t *f = p->ctl;
        GLM_CUDA_TRY(cudaMemcpy(p->bufs_dev, &b, sizeof(b), cudaMemcpyHostToDevice));
        GLM_CUDA_TRY(cudaMemcpy(p->flags_dev, &f, sizeof(f), cudaMemcpyHostToDevice));
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
    std::vector<double *> bufs(p->world);
    std::vector<int64_t *> flags(p->world);
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
        flags[j] = reinterpret_cast<int64_t *>(base);
        bufs[j] = reinterpret_cast<double *>(base + 256);
    }
    GLM_CUDA_TRY(cudaMemcpy(p->bufs_dev, bufs.data(), sizeof(double *) * p->world,
                            cudaMemcpyHostToDevice));
    GLM_CUDA_TRY(cudaMemcpy(p->flags_dev, flags.data(), sizeof(int64_t *) * p->world,
                            cudaMemcpyHostToDevice));
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
    a.flags = p->flags_dev;
    a.ctl = p->ctl;
    a.st = s ? s->st : nullptr;
    a.view0 = s ? s->view[0] : nullptr;
    a.view1 = s ? s->view[1] : nullptr;
    a.epochs = epochs;
    a.scratch = scratch;
    count_launch();
    round_start_kernel<<<PEER_BLOCKS, PEER_THREADS, 0, (cudaStream_t)stream>>>(a);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

}  // extern "C"
