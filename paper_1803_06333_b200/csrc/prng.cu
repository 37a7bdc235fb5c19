// prng.cu — permutation stream on the device (sm_100a).
//
// Reference semantics:
//   PermutationGenerator.keys/permute (solver.py:64-89): key i = low 32 bits
//   of the (i+1)-th successive xorshift64(13,7,17) state; permutation =
//   np.argsort(keys, kind="stable").
//   generate_keys (pipeline.py:29-73): 4096-wide blocks, block b seeded with
//   derive_seed(seed, b).
//
// B200 design: xorshift64 is linear over GF(2), so a thread can jump straight
// to position q of the stream with the precomputed matrices M^(2^i) (64 x u64
// columns each, 32 KB table in global memory) instead of walking the stream
// serially.  Keys are never materialised on the hot path: a first pass
// generates them and builds a histogram of the top `nb` bits (nb chosen so a
// bucket holds ~8 keys), one block scans the histogram, a second pass
// regenerates the keys and scatters (key<<32 | index) pairs into their
// buckets, and one thread per bucket insertion-sorts its ~8 pairs by
// (key, index) — exactly the stable order.  Buckets larger than the register
// budget (rare tail for xorshift keys) are insertion-sorted in place in global
// memory by their thread: slower, same result.
#include <algorithm>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "prng.cuh"

namespace glm {

__device__ uint64_t d_jump_cols[64 * 64];   // [i][k]: column k of M^(2^i)

static uint64_t h_jump_cols[64 * 64];
static std::once_flag h_jump_once;
static bool d_jump_ready[64];
static std::mutex d_jump_mutex;

static inline uint64_t xs_step(uint64_t s) {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    return s;
}

static void build_host_jump() {
    for (int k = 0; k < 64; ++k) h_jump_cols[k] = xs_step(1ULL << k);
    for (int i = 1; i < 64; ++i) {
        const uint64_t *a = h_jump_cols + (i - 1) * 64;
        uint64_t *o = h_jump_cols + i * 64;
        for (int k = 0; k < 64; ++k) {          // o = a∘a applied to e_k
            uint64_t x = a[k], y = 0;
            for (int b = 0; b < 64; ++b)
                if ((x >> b) & 1) y ^= a[b];
            o[k] = y;
        }
    }
}

uint64_t host_jump(uint64_t state, uint64_t steps) {
    std::call_once(h_jump_once, build_host_jump);
    for (int i = 0; i < 64 && steps; ++i, steps >>= 1) {
        if (!(steps & 1)) continue;
        const uint64_t *c = h_jump_cols + i * 64;
        uint64_t y = 0;
        for (int b = 0; b < 64; ++b)
            if ((state >> b) & 1) y ^= c[b];
        state = y;
    }
    return state;
}

int ensure_device_tables() {
    int dev = 0;
    GLM_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(d_jump_mutex);
    if (dev < 64 && d_jump_ready[dev]) return GLM_OK;
    std::call_once(h_jump_once, build_host_jump);
    GLM_CUDA_TRY(cudaMemcpyToSymbol(d_jump_cols, h_jump_cols, sizeof(h_jump_cols)));
    if (dev < 64) d_jump_ready[dev] = true;
    return GLM_OK;
}

__device__ __forceinline__ uint64_t dev_xs(uint64_t s) {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    return s;
}

__device__ __forceinline__ uint64_t dev_jump(uint64_t state, uint64_t steps) {
    for (int i = 0; steps; ++i, steps >>= 1) {
        if (!(steps & 1)) continue;
        const uint64_t *c = d_jump_cols + i * 64;
        uint64_t y = 0;
#pragma unroll 8
        for (int b = 0; b < 64; ++b) y ^= ((state >> b) & 1) ? __ldg(c + b) : 0ULL;
        state = y;
    }
    return state;
}

__device__ __forceinline__ uint64_t dev_splitmix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

__device__ __forceinline__ uint64_t dev_derive1(uint64_t base, uint64_t ix) {
    uint64_t s = dev_splitmix(base);
    s = dev_splitmix(s ^ (ix + 0x632BE59BD9B4E019ULL));
    return s ? s : 0x9E3779B97F4A7C15ULL;
}

// ---------------------------------------------------------------------------
// Key sources.  Each thread owns KPT consecutive keys [q0, q0+KPT).
struct StreamKeys {       // PermutationGenerator stream, attempt offset
    const SolveState *st; // if non-null: base state = st->gen_state, skip when done
    uint64_t state;       // used when st == nullptr
    uint64_t offset;      // position of key 0 in the stream
    __device__ __forceinline__ bool skip() const { return st && st->done; }
    __device__ __forceinline__ uint64_t start(int64_t q0) const {
        uint64_t s0 = st ? st->gen_state : state;
        return dev_jump(s0, offset + (uint64_t)q0);
    }
};

struct ChunkKeys {        // generate_keys(seed, n): 4096-wide blocks
    uint64_t seed;
    __device__ __forceinline__ bool skip() const { return false; }
    __device__ __forceinline__ uint64_t start(int64_t q0) const {
        uint64_t b = (uint64_t)q0 >> 12;
        return dev_jump(dev_derive1(seed, b), (uint64_t)q0 & 4095);
    }
};

constexpr int KPT = 64;   // keys per thread (divides 4096)

template <class Src>
__global__ void __launch_bounds__(256) keys_kernel(Src src, int64_t n, uint32_t *keys) {
    int64_t q0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * KPT;
    if (q0 >= n || src.skip()) return;
    uint64_t s = src.start(q0);
    int64_t q1 = q0 + KPT < n ? q0 + KPT : n;
    for (int64_t q = q0; q < q1; ++q) {
        s = dev_xs(s);
        keys[q] = (uint32_t)s;
    }
}

template <class Src>
__global__ void __launch_bounds__(256) hist_kernel(Src src, int64_t n, int shift,
                                                   uint32_t *hist) {
    int64_t q0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * KPT;
    if (q0 >= n || src.skip()) return;
    uint64_t s = src.start(q0);
    int64_t q1 = q0 + KPT < n ? q0 + KPT : n;
    for (int64_t q = q0; q < q1; ++q) {
        s = dev_xs(s);
        atomicAdd(hist + (shift >= 32 ? 0u : ((uint32_t)s >> shift)), 1u);
    }
}

template <class Src>
__global__ void __launch_bounds__(256) scatter_kernel(Src src, int64_t n, int shift,
                                                      uint32_t *cursor, uint64_t *pairs) {
    int64_t q0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * KPT;
    if (q0 >= n || src.skip()) return;
    uint64_t s = src.start(q0);
    int64_t q1 = q0 + KPT < n ? q0 + KPT : n;
    for (int64_t q = q0; q < q1; ++q) {
        s = dev_xs(s);
        uint32_t key = (uint32_t)s;
        uint32_t pos = atomicAdd(cursor + (shift >= 32 ? 0u : (key >> shift)), 1u);
        pairs[pos] = ((uint64_t)key << 32) | (uint32_t)q;
    }
}

// Array key source variants (glm_argsort_u32 on caller-provided keys).
__global__ void hist_array_kernel(const uint32_t *keys, int64_t n, int shift, uint32_t *hist) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(hist + (shift >= 32 ? 0u : (keys[q] >> shift)), 1u);
}

__global__ void scatter_array_kernel(const uint32_t *keys, int64_t n, int shift,
                                     uint32_t *cursor, uint64_t *pairs) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x) {
        uint32_t key = keys[q];
        uint32_t pos = atomicAdd(cursor + (shift >= 32 ? 0u : (key >> shift)), 1u);
        pairs[pos] = ((uint64_t)key << 32) | (uint32_t)q;
    }
}

// Exclusive scan of hist[0..nbk) -> offs[0..nbk], cursor = offs; hist zeroed
// for the next use; flag[0] = max bucket size.  One block of 1024 threads.
__global__ void __launch_bounds__(1024) scan_kernel(const SolveState *st, uint32_t *hist,
                                                    uint32_t *offs, uint32_t *cursor,
                                                    int64_t nbk, uint32_t *maxb) {
    if (st && st->done) return;
    __shared__ uint32_t ssum[1024];
    __shared__ uint32_t smax[32];
    const int t = threadIdx.x;
    int64_t per = (nbk + 1023) / 1024;
    int64_t lo = t * per, hi = lo + per < nbk ? lo + per : nbk;
    uint32_t sum = 0, mx = 0;
    for (int64_t i = lo; i < hi; ++i) {
        uint32_t h = hist[i];
        sum += h;
        mx = h > mx ? h : mx;
    }
    ssum[t] = sum;
    // warp max
    for (int o = 16; o; o >>= 1) {
        uint32_t x = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = x > mx ? x : mx;
    }
    if ((t & 31) == 0) smax[t >> 5] = mx;
    __syncthreads();
    // Hillis-Steele inclusive scan over 1024 partial sums
    for (int o = 1; o < 1024; o <<= 1) {
        uint32_t x = t >= o ? ssum[t - o] : 0;
        __syncthreads();
        ssum[t] += x;
        __syncthreads();
    }
    uint32_t run = t ? ssum[t - 1] : 0;
    for (int64_t i = lo; i < hi; ++i) {
        uint32_t h = hist[i];
        offs[i] = run;
        cursor[i] = run;
        hist[i] = 0;
        run += h;
    }
    if (t == 1023) offs[nbk] = ssum[1023];
    if (t < 32) {
        uint32_t m2 = smax[t];
        for (int o = 16; o; o >>= 1) {
            uint32_t x = __shfl_xor_sync(0xffffffffu, m2, o);
            m2 = x > m2 ? x : m2;
        }
        if (t == 0) *maxb = m2;
    }
}

constexpr int BUCKET_REG = 32;

// One thread per bucket: insertion sort of (key<<32|idx) pairs; writes perm.
__global__ void __launch_bounds__(256) bucket_sort_kernel(const SolveState *st,
                                                          const uint64_t *pairs,
                                                          const uint32_t *offs, int64_t nbk,
                                                          int32_t *perm, uint64_t *pairs_rw) {
    if (st && st->done) return;
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nbk) return;
    uint32_t lo = offs[b], hi = offs[b + 1];
    uint32_t s = hi - lo;
    if (s == 0) return;
    if (s > BUCKET_REG) {           // rare tail: sort in place in global memory
        uint64_t *g = pairs_rw + lo;
        for (uint32_t i = 1; i < s; ++i) {
            uint64_t x = g[i];
            int64_t j = (int64_t)i - 1;
            while (j >= 0 && g[j] > x) {
                g[j + 1] = g[j];
                --j;
            }
            g[j + 1] = x;
        }
        for (uint32_t i = 0; i < s; ++i) perm[lo + i] = (int32_t)(uint32_t)g[i];
        return;
    }
    uint64_t a[BUCKET_REG];
#pragma unroll
    for (int i = 0; i < BUCKET_REG; ++i)
        if (i < (int)s) a[i] = pairs[lo + i];
    for (int i = 1; i < (int)s; ++i) {
        uint64_t x = a[i];
        int j = i - 1;
        while (j >= 0 && a[j] > x) {
            a[j + 1] = a[j];
            --j;
        }
        a[j + 1] = x;
    }
    for (int i = 0; i < (int)s; ++i) perm[lo + i] = (int32_t)(uint32_t)a[i];
}

// ---------------------------------------------------------------------------
int bucket_bits(int64_t n) {
    int lg = 0;
    while ((1LL << lg) < n) ++lg;
    int nb = lg - 3;               // ~8 keys per bucket
    if (nb < 1) nb = 1;
    if (nb > 24) nb = 24;
    return nb;
}

size_t perm_scratch_bytes(int64_t n) {
    int nb = bucket_bits(n);
    int64_t nbk = 1LL << nb;
    size_t a = sizeof(uint64_t) * (size_t)(n > 0 ? n : 1);                  // pairs
    size_t h = sizeof(uint32_t) * (size_t)(3 * nbk + 1 + 2);                // hist, offs, cursor, flags
    return a + h + 1024;
}

PermScratch carve_perm_scratch(void *base, int64_t capacity, int64_t n) {
    // Region offsets depend only on `capacity` so the zeroed histogram stays
    // in place across calls with different n (the scan re-zeroes what it used).
    PermScratch p;
    p.nb = bucket_bits(n);
    p.nbk = 1LL << p.nb;
    const int64_t nbk_cap = 1LL << bucket_bits(capacity);
    char *c = (char *)base;
    c += sizeof(uint64_t) * (size_t)(capacity > 0 ? capacity : 1);
    c = (char *)(((uintptr_t)c + 255) & ~(uintptr_t)255);
    p.pairs = (uint64_t *)base;
    p.hist = (uint32_t *)c;
    p.offs = p.hist + nbk_cap;
    p.cursor = p.offs + nbk_cap + 1;
    p.flags = p.cursor + nbk_cap;
    return p;
}

static int grid_for(int64_t n) {
    int64_t threads = (n + KPT - 1) / KPT;
    return (int)((threads + 255) / 256);
}

// Stable argsort of the given key source into perm (int32).
template <class Src>
static int perm_from_source(const Src &src, const SolveState *st, int64_t n, int32_t *perm,
                            const PermScratch &sc, cudaStream_t stream,
                            const uint32_t *keys_array) {
    if (n <= 0) return GLM_OK;
    int shift = 32 - sc.nb;
    if (keys_array) {
        int g = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
        count_launch();
        hist_array_kernel<<<g, 256, 0, stream>>>(keys_array, n, shift, sc.hist);
    } else {
        count_launch();
        hist_kernel<<<grid_for(n), 256, 0, stream>>>(src, n, shift, sc.hist);
    }
    count_launch();
    scan_kernel<<<1, 1024, 0, stream>>>(st, sc.hist, sc.offs, sc.cursor, sc.nbk, sc.flags);
    if (keys_array) {
        int g = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
        count_launch();
        scatter_array_kernel<<<g, 256, 0, stream>>>(keys_array, n, shift, sc.cursor, sc.pairs);
    } else {
        count_launch();
        scatter_kernel<<<grid_for(n), 256, 0, stream>>>(src, n, shift, sc.cursor, sc.pairs);
    }
    count_launch();
    bucket_sort_kernel<<<(int)((sc.nbk + 255) / 256), 256, 0, stream>>>(
        st, sc.pairs, sc.offs, sc.nbk, perm, sc.pairs);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

int stream_perm(const SolveState *st, uint64_t state, uint64_t offset, int64_t n,
                int32_t *perm, const PermScratch &sc, cudaStream_t stream) {
    StreamKeys src{st, state, offset};
    return perm_from_source(src, st, n, perm, sc, stream, nullptr);
}

int chunk_perm(uint64_t seed, int64_t n, int32_t *perm, const PermScratch &sc,
               cudaStream_t stream) {
    ChunkKeys src{seed};
    return perm_from_source(src, nullptr, n, perm, sc, stream, nullptr);
}

int array_perm(const uint32_t *keys, int64_t n, int32_t *perm, const PermScratch &sc,
               cudaStream_t stream) {
    ChunkKeys dummy{0};
    return perm_from_source(dummy, nullptr, n, perm, sc, stream, keys);
}

int stream_keys(uint64_t state, uint64_t offset, int64_t n, uint32_t *keys,
                cudaStream_t stream) {
    if (n <= 0) return GLM_OK;
    StreamKeys src{nullptr, state, offset};
    count_launch();
    keys_kernel<<<grid_for(n), 256, 0, stream>>>(src, n, keys);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

int chunk_keys(uint64_t seed, int64_t n, uint32_t *keys, cudaStream_t stream) {
    if (n <= 0) return GLM_OK;
    ChunkKeys src{seed};
    count_launch();
    keys_kernel<<<grid_for(n), 256, 0, stream>>>(src, n, keys);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

}  // namespace glm
