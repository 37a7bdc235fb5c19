// prng.cu — permutation stream on the device (sm_100a).
//
// Reference semantics:
//   PermutationGenerator.keys/permute (solver.py:64-89): key i = low 32 bits
//   of the (i+1)-th successive xorshift64(13,7,17) state; permutation =
//   np.argsort(keys, kind="stable").
//   generate_keys (pipeline.py:29-73): 4096-wide blocks, block b seeded with
//   derive_seed(seed, b).
//
// B200 design.  xorshift64 is linear over GF(2): M^k is a 64x64 bit matrix.
// A CUDA block of 256 threads owns 4096 consecutive keys (16 per thread).
// Warp 0 jumps to the block's first state with the M^(2^i) table, lanes
// splitting the 64 columns and XOR-reducing through shuffles; every thread
// then applies one precomputed matrix M^(16 t) and walks its 16 keys.  For the
// chunk stream the 4096-key CUDA block *is* the reference's key block, so the
// base state is derive_seed(seed, block).
//
// The stable argsort never materialises the keys: pass 1 histograms the top
// `nb` key bits (nb chosen for ~8 keys per bucket), a two-kernel parallel
// scan turns the histogram into bucket offsets, pass 2 regenerates the keys
// and scatters (key<<32 | index) into the buckets, and a warp per 32 buckets
// stages its ~256 pairs in shared memory, insertion-sorts each bucket by
// (key, index) — exactly numpy's stable order — and writes the permutation
// coalesced.  Oversized bucket groups fall back to an in-place sort in global
// memory (slower, same result).
#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "prng.cuh"

namespace glm {

constexpr int PERM_THREADS = 256;
constexpr int KPT = 16;                             // keys per thread
constexpr int KEYS_PER_BLOCK = PERM_THREADS * KPT;  // 4096 == pipeline.KEY_BLOCK

__device__ uint64_t d_jump_cols[64 * 64];            // [i][b]: column b of M^(2^i)
__device__ uint64_t d_thread_jump[PERM_THREADS * 64];  // [t][b]: column b of M^(16 t)

static uint64_t h_jump_cols[64 * 64];
static uint64_t h_thread_jump[PERM_THREADS * 64];
static std::once_flag h_jump_once;
static bool d_jump_ready[64];
static std::mutex d_jump_mutex;

static inline uint64_t xs_step(uint64_t s) {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    return s;
}

static inline uint64_t mat_apply(const uint64_t *cols, uint64_t x) {
    uint64_t y = 0;
    for (int b = 0; b < 64; ++b)
        if ((x >> b) & 1) y ^= cols[b];
    return y;
}

static void build_host_jump() {
    for (int b = 0; b < 64; ++b) h_jump_cols[b] = xs_step(1ULL << b);
    for (int i = 1; i < 64; ++i) {
        const uint64_t *a = h_jump_cols + (i - 1) * 64;
        for (int b = 0; b < 64; ++b) h_jump_cols[i * 64 + b] = mat_apply(a, a[b]);
    }
    // thread matrices M^(KPT*t): columns are the images of e_b after KPT*t steps
    for (int b = 0; b < 64; ++b) {
        uint64_t s = 1ULL << b;
        for (int t = 0; t < PERM_THREADS; ++t) {
            h_thread_jump[t * 64 + b] = s;
            for (int k = 0; k < KPT; ++k) s = xs_step(s);
        }
    }
}

uint64_t host_jump(uint64_t state, uint64_t steps) {
    std::call_once(h_jump_once, build_host_jump);
    for (int i = 0; i < 64 && steps; ++i, steps >>= 1)
        if (steps & 1) state = mat_apply(h_jump_cols + i * 64, state);
    return state;
}

int ensure_device_tables() {
    int dev = 0;
    GLM_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(d_jump_mutex);
    if (dev < 64 && d_jump_ready[dev]) return GLM_OK;
    std::call_once(h_jump_once, build_host_jump);
    GLM_CUDA_TRY(cudaMemcpyToSymbol(d_jump_cols, h_jump_cols, sizeof(h_jump_cols)));
    GLM_CUDA_TRY(cudaMemcpyToSymbol(d_thread_jump, h_thread_jump, sizeof(h_thread_jump)));
    GLM_CUDA_TRY(cudaDeviceSynchronize());
    if (dev < 64) d_jump_ready[dev] = true;
    return GLM_OK;
}

__device__ __forceinline__ uint64_t dev_xs(uint64_t s) {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    return s;
}

__device__ __forceinline__ uint64_t xor_reduce_warp(uint64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v ^= __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Warp-cooperative jump: all 32 lanes call with the same (state, steps).
__device__ __forceinline__ uint64_t warp_jump(uint64_t state, uint64_t steps) {
    const int lane = threadIdx.x & 31;
    for (int i = 0; steps; ++i, steps >>= 1) {
        if (!(steps & 1)) continue;
        const uint64_t *c = d_jump_cols + i * 64;
        uint64_t part = (((state >> lane) & 1) ? c[lane] : 0ULL) ^
                        (((state >> (lane + 32)) & 1) ? c[lane + 32] : 0ULL);
        state = xor_reduce_warp(part);
    }
    return state;
}

__device__ __forceinline__ uint64_t thread_apply(uint64_t state) {
    const uint64_t *c = d_thread_jump + threadIdx.x * 64;
    uint64_t y = 0;
#pragma unroll 16
    for (int b = 0; b < 64; ++b) y ^= ((state >> b) & 1) ? __ldg(c + b) : 0ULL;
    return y;
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
// Key sources: block_base() returns the state before the block's first key
// (called by the 32 lanes of warp 0).
struct StreamKeys {       // PermutationGenerator stream at attempt offset
    const SolveState *st; // non-null: skip once st->done
    const uint64_t *state_ptr;   // device-held start state (else `state`)
    uint64_t state;
    uint64_t offset;
    __device__ __forceinline__ bool skip() const { return st && st->done; }
    __device__ __forceinline__ uint64_t block_base() const {
        const uint64_t s0 = state_ptr ? *state_ptr : state;
        return warp_jump(s0, offset + (uint64_t)blockIdx.x * KEYS_PER_BLOCK);
    }
};

struct ChunkKeys {        // generate_keys(seed, n)
    uint64_t seed;
    __device__ __forceinline__ bool skip() const { return false; }
    __device__ __forceinline__ uint64_t block_base() const {
        return dev_derive1(seed, (uint64_t)blockIdx.x);
    }
};

// Runs f(q, key) over this thread's KPT keys.
template <class Src, class F>
__device__ __forceinline__ void for_keys(const Src &src, int64_t n, F f) {
    __shared__ uint64_t s_base;
    if (threadIdx.x < 32) {
        const uint64_t b = src.block_base();
        if (threadIdx.x == 0) s_base = b;
    }
    __syncthreads();
    const int64_t q0 = (int64_t)blockIdx.x * KEYS_PER_BLOCK + (int64_t)threadIdx.x * KPT;
    if (q0 >= n) return;
    uint64_t s = thread_apply(s_base);
    const int cnt = (int)(n - q0 < KPT ? n - q0 : KPT);
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
        s = dev_xs(s);
        if (i < cnt) f(q0 + i, (uint32_t)s);
    }
}

template <class Src>
__global__ void __launch_bounds__(PERM_THREADS) keys_kernel(Src src, int64_t n, uint32_t *keys) {
    if (src.skip()) return;
    for_keys(src, n, [&](int64_t q, uint32_t k) { keys[q] = k; });
}

template <class Src>
__global__ void __launch_bounds__(PERM_THREADS) hist_kernel(Src src, int64_t n, int shift,
                                                            uint32_t *hist) {
    if (src.skip()) return;
    tl_start(TL_PERM_FIRST);
    for_keys(src, n, [&](int64_t, uint32_t k) { atomicAdd(hist + (k >> shift), 1u); });
    __syncthreads();
    tl_end(TL_PERM_FIRST);
}

template <class Src>
__global__ void __launch_bounds__(PERM_THREADS) scatter_kernel(Src src, int64_t n, int shift,
                                                               uint32_t *cursor,
                                                               uint64_t *pairs) {
    if (src.skip()) return;
    for_keys(src, n, [&](int64_t q, uint32_t k) {
        const uint32_t pos = atomicAdd(cursor + (k >> shift), 1u);
        pairs[pos] = ((uint64_t)k << 32) | (uint32_t)q;
    });
}

// Array key source variants (glm_argsort_u32 on caller-provided keys).
__global__ void hist_array_kernel(const uint32_t *keys, int64_t n, int shift, uint32_t *hist) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(hist + (keys[q] >> shift), 1u);
}

__global__ void scatter_array_kernel(const uint32_t *keys, int64_t n, int shift,
                                     uint32_t *cursor, uint64_t *pairs) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t key = keys[q];
        const uint32_t pos = atomicAdd(cursor + (key >> shift), 1u);
        pairs[pos] = ((uint64_t)key << 32) | (uint32_t)q;
    }
}

// ---------------------------------------------------------------- scan
constexpr int SCAN_TILE = 1024;

__device__ __forceinline__ uint32_t block_excl_scan_1024(uint32_t x, uint32_t *s_warp,
                                                         uint32_t &total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = s_warp[lane];
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        s_warp[lane] = wi - w;        // exclusive warp prefix
        if (lane == 31) s_warp[32] = wi;
    }
    __syncthreads();
    total = s_warp[32];
    return s_warp[warp] + inc - x;
}

__global__ void __launch_bounds__(SCAN_TILE) tile_sum_kernel(const SolveState *st,
                                                             const uint32_t *hist, int64_t nbk,
                                                             uint32_t *tile_sums) {
    if (st && st->done) return;
    __shared__ uint32_t s_warp[33];
    const int64_t i = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x;
    uint32_t total = 0;
    block_excl_scan_1024(i < nbk ? hist[i] : 0u, s_warp, total);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(SCAN_TILE) tile_scan_kernel(const SolveState *st,
                                                              uint32_t *hist, int64_t nbk,
                                                              const uint32_t *tile_sums,
                                                              uint32_t *offs, uint32_t *cursor) {
    if (st && st->done) return;
    __shared__ uint32_t s_warp[33];
    __shared__ uint32_t s_prefix;
    if (threadIdx.x < 32) {      // prefix of the previous tiles' totals
        uint32_t acc = 0;
        for (int t = threadIdx.x; t < (int)blockIdx.x; t += 32) acc += tile_sums[t];
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (threadIdx.x == 0) s_prefix = acc;
    }
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x;
    const uint32_t h = i < nbk ? hist[i] : 0u;
    uint32_t total = 0;
    const uint32_t ex = block_excl_scan_1024(h, s_warp, total) + s_prefix;
    if (i < nbk) {
        offs[i] = ex;
        cursor[i] = ex;
        hist[i] = 0;                 // ready for the next permutation
        if (i == nbk - 1) offs[nbk] = ex + h;
    }
}

// ---------------------------------------------------------- bucket sort
constexpr int BS_WARPS = 8;
constexpr int BS_CAP = 512;   // pairs staged per warp (32 buckets x ~8 expected)

__device__ __forceinline__ void insertion_sort(uint64_t *a, int s) {
    for (int i = 1; i < s; ++i) {
        const uint64_t x = a[i];
        int j = i - 1;
        while (j >= 0 && a[j] > x) {
            a[j + 1] = a[j];
            --j;
        }
        a[j + 1] = x;
    }
}

__global__ void __launch_bounds__(BS_WARPS * 32) bucket_sort_kernel(const SolveState *st,
                                                                    uint64_t *pairs,
                                                                    const uint32_t *offs,
                                                                    int64_t nbk, int32_t *perm) {
    if (st && st->done) return;
    tl_start(TL_PERM_LAST);
    __shared__ uint64_t sbuf[BS_WARPS][BS_CAP];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t b0 = ((int64_t)blockIdx.x * BS_WARPS + warp) * 32;
    if (b0 >= nbk) return;
    const int64_t b1 = b0 + 32 < nbk ? b0 + 32 : nbk;
    const uint32_t lo = offs[b0], hi = offs[b1];
    const int64_t b = b0 + lane;
    const uint32_t my_lo = b < b1 ? offs[b] : hi, my_hi = b < b1 ? offs[b + 1] : hi;
    const uint32_t n = hi - lo;
    if (n <= BS_CAP) {
        uint64_t *buf = sbuf[warp];
        for (uint32_t i = lane; i < n; i += 32) buf[i] = pairs[lo + i];
        __syncwarp();
        insertion_sort(buf + (my_lo - lo), (int)(my_hi - my_lo));
        __syncwarp();
        for (uint32_t i = lane; i < n; i += 32) perm[lo + i] = (int32_t)(uint32_t)buf[i];
        tl_end_warp(TL_PERM_LAST);
    } else {                     // rare: sort in place in global memory
        insertion_sort(pairs + my_lo, (int)(my_hi - my_lo));
        __syncwarp();
        for (uint32_t i = lane; i < n; i += 32) perm[lo + i] = (int32_t)(uint32_t)pairs[lo + i];
        tl_end_warp(TL_PERM_LAST);
    }
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
    const int64_t nbk = 1LL << bucket_bits(n);
    const size_t a = sizeof(uint64_t) * (size_t)(n > 0 ? n : 1);             // pairs
    const size_t h = sizeof(uint32_t) * (size_t)(3 * nbk + 1 + nbk / SCAN_TILE + 2);
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
    p.flags = p.cursor + nbk_cap;     // tile sums (nbk_cap / SCAN_TILE + 1)
    return p;
}

static int key_blocks(int64_t n) { return (int)((n + KEYS_PER_BLOCK - 1) / KEYS_PER_BLOCK); }

template <class Src>
static int perm_from_source(const Src &src, const SolveState *st, int64_t n, int32_t *perm,
                            const PermScratch &sc, cudaStream_t stream,
                            const uint32_t *keys_array) {
    if (n <= 0) return GLM_OK;
    const int shift = 32 - sc.nb;
    const int tiles = (int)((sc.nbk + SCAN_TILE - 1) / SCAN_TILE);
    const int agrid = (int)std::min<int64_t>((n + 255) / 256, NUM_SMS * 16);
    count_launch();
    if (keys_array) hist_array_kernel<<<agrid, 256, 0, stream>>>(keys_array, n, shift, sc.hist);
    else hist_kernel<<<key_blocks(n), PERM_THREADS, 0, stream>>>(src, n, shift, sc.hist);
    count_launch();
    tile_sum_kernel<<<tiles, SCAN_TILE, 0, stream>>>(st, sc.hist, sc.nbk, sc.flags);
    count_launch();
    tile_scan_kernel<<<tiles, SCAN_TILE, 0, stream>>>(st, sc.hist, sc.nbk, sc.flags, sc.offs,
                                                      sc.cursor);
    count_launch();
    if (keys_array)
        scatter_array_kernel<<<agrid, 256, 0, stream>>>(keys_array, n, shift, sc.cursor, sc.pairs);
    else
        scatter_kernel<<<key_blocks(n), PERM_THREADS, 0, stream>>>(src, n, shift, sc.cursor,
                                                                   sc.pairs);
    count_launch();
    const int64_t groups = (sc.nbk + 31) / 32;
    bucket_sort_kernel<<<(int)((groups + BS_WARPS - 1) / BS_WARPS), BS_WARPS * 32, 0, stream>>>(
        st, sc.pairs, sc.offs, sc.nbk, perm);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

int stream_perm(const SolveState *st, uint64_t state, uint64_t offset, int64_t n,
                int32_t *perm, const PermScratch &sc, cudaStream_t stream) {
    StreamKeys src{st, st ? &st->gen_state : nullptr, state, offset};
    return perm_from_source(src, st, n, perm, sc, stream, nullptr);
}

int stream_perm_from(const uint64_t *state_dev, int64_t n, int32_t *perm, const PermScratch &sc,
                     cudaStream_t stream) {
    StreamKeys src{nullptr, state_dev, 0, 0};
    return perm_from_source(src, nullptr, n, perm, sc, stream, nullptr);
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
    StreamKeys src{nullptr, nullptr, state, offset};
    count_launch();
    keys_kernel<<<key_blocks(n), PERM_THREADS, 0, stream>>>(src, n, keys);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

int chunk_keys(uint64_t seed, int64_t n, uint32_t *keys, cudaStream_t stream) {
    if (n <= 0) return GLM_OK;
    ChunkKeys src{seed};
    count_launch();
    keys_kernel<<<key_blocks(n), PERM_THREADS, 0, stream>>>(src, n, keys);
    GLM_CUDA_TRY(cudaGetLastError());
    return GLM_OK;
}

}  // namespace glm
