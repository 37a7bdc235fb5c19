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
// The stable argsort never materialises the keys.  Two variants, same order:
//  * bucket regions (generated keys, n <= 2^21 — every partition and chunk of
//    the configs): 2 kernels.  Pass 1 (one CTA per 4096-key block) walks its
//    keys twice from registers: a shared-memory histogram of the top `nb2`
//    bits (<= 512 keys per bucket on average), one global atomicAdd per
//    non-empty bucket to reserve a run in that bucket's fixed 1024-pair
//    region, then the (key<<32 | index) pairs go to their runs; the last CTA
//    (ticket) scans the bucket totals into output offsets.  Pass 2 (one CTA
//    per bucket) spreads its pairs over 256 sub-buckets (the next 8 key bits)
//    in shared memory, each thread insertion-sorts one, and the CTA writes
//    its slice of the permutation.  The order inside a region depends on the
//    atomics, the sorted result does not (pairs are unique).  A bucket beyond
//    its region spills to an overflow list and is sorted by a slow path.
//  * global buckets (larger n, and argsort of caller keys): pass 1 histograms
//    the top `nb` bits (~8 keys per bucket) with global atomics, a two-kernel
//    scan gives bucket offsets, pass 2 regenerates the keys and scatters, and
//    a warp per 32 buckets insertion-sorts them in shared memory.  Oversized
//    bucket groups fall back to an in-place sort in global memory.
// Block start states: M^(4096 b) s0 from a table of the first 512 block
// jumps (one warp matrix-vector product instead of a chain of ~20 dependent
// jump-table loads); the attempt offset, when not 0, is one warp_jump.
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "prng.cuh"

namespace glm {

constexpr int PERM_THREADS = 256;
constexpr int KPT = 16;                             // keys per thread
constexpr int KEYS_PER_BLOCK = PERM_THREADS * KPT;  // 4096 == pipeline.KEY_BLOCK

__device__ uint64_t d_jump_cols[64 * 64];            // [i][b]: column b of M^(2^i)
__device__ uint64_t d_thread_jump[PERM_THREADS * 64];  // [b][t]: column b of M^(16 t)
constexpr int BLK_JUMPS = 512;                        // 2^21 keys / 4096
__device__ uint64_t d_blk_jump[BLK_JUMPS * 64];       // [blk][b]: column b of M^(4096 blk)

static uint64_t h_jump_cols[64 * 64];
static uint64_t h_thread_jump[PERM_THREADS * 64];
static uint64_t h_blk_jump[BLK_JUMPS * 64];
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
            h_thread_jump[b * PERM_THREADS + t] = s;   // [b][t]: a warp's loads coalesce
            for (int k = 0; k < KPT; ++k) s = xs_step(s);
        }
    }
    // block matrices M^(4096 blk) = (M^4096)^blk, M^4096 = M^(2^12)
    const uint64_t *m4096 = h_jump_cols + 12 * 64;
    for (int b = 0; b < 64; ++b) h_blk_jump[b] = 1ULL << b;
    for (int k = 1; k < BLK_JUMPS; ++k)
        for (int b = 0; b < 64; ++b)
            h_blk_jump[k * 64 + b] = mat_apply(m4096, h_blk_jump[(k - 1) * 64 + b]);
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
    GLM_CUDA_TRY(cudaMemcpyToSymbol(d_blk_jump, h_blk_jump, sizeof(h_blk_jump)));
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

// Warp-cooperative jump: all 32 lanes call with the same (state, steps).  The
// matrix columns do not depend on the state, so the next set bit's columns are
// loaded while the current product is XOR-reduced.
__device__ __forceinline__ uint64_t warp_jump(uint64_t state, uint64_t steps) {
    const int lane = threadIdx.x & 31;
    if (!steps) return state;
    int i = __ffsll((long long)steps) - 1;
    uint64_t c0 = d_jump_cols[i * 64 + lane], c1 = d_jump_cols[i * 64 + lane + 32];
    for (;;) {
        steps &= steps - 1;
        const int nx = steps ? __ffsll((long long)steps) - 1 : -1;
        uint64_t n0 = 0, n1 = 0;
        if (nx >= 0) {
            n0 = d_jump_cols[nx * 64 + lane];
            n1 = d_jump_cols[nx * 64 + lane + 32];
        }
        const uint64_t part = (((state >> lane) & 1) ? c0 : 0ULL) ^
                              (((state >> (lane + 32)) & 1) ? c1 : 0ULL);
        state = xor_reduce_warp(part);
        if (nx < 0) return state;
        c0 = n0;
        c1 = n1;
    }
}

// M^(4096 blk) state for the first BLK_JUMPS blocks: every lane applies two
// columns (one load each), one XOR reduction; later blocks take warp_jump.
__device__ __forceinline__ uint64_t block_jump(uint64_t state, int64_t blk) {
    if (blk >= BLK_JUMPS) return warp_jump(state, (uint64_t)blk * KEYS_PER_BLOCK);
    const int lane = threadIdx.x & 31;
    const uint64_t *c = d_blk_jump + blk * 64;
    const uint64_t c0 = c[lane], c1 = c[lane + 32];
    return xor_reduce_warp((((state >> lane) & 1) ? c0 : 0ULL) ^
                           (((state >> (lane + 32)) & 1) ? c1 : 0ULL));
}

__device__ __forceinline__ uint64_t thread_apply(uint64_t state) {
    const uint64_t *c = d_thread_jump + threadIdx.x;
    uint64_t y = 0;
#pragma unroll
    for (int b = 0; b < 64; ++b) y ^= ((state >> b) & 1) ? __ldg(c + b * PERM_THREADS) : 0ULL;
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
        return block_jump(offset ? warp_jump(s0, offset) : s0, blockIdx.x);
    }
};

struct ChunkKeys {        // generate_keys(seed, n)
    uint64_t seed;
    __device__ __forceinline__ bool skip() const { return false; }
    __device__ __forceinline__ uint64_t block_base() const {
        return dev_derive1(seed, (uint64_t)blockIdx.x);
    }
};

// Thread's KPT keys from its start state s.
template <class F>
__device__ __forceinline__ void walk_keys(uint64_t s, int64_t n, F f) {
    const int64_t q0 = (int64_t)blockIdx.x * KEYS_PER_BLOCK + (int64_t)threadIdx.x * KPT;
    if (q0 >= n) return;
    const int cnt = (int)(n - q0 < KPT ? n - q0 : KPT);
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
        s = dev_xs(s);
        if (i < cnt) f(q0 + i, (uint32_t)s);
    }
}

// Runs f(q, key) over this thread's KPT keys; saves the thread's start state
// to tstate[global thread] when given (a second pass reads it back).
template <class Src, class F>
__device__ __forceinline__ void for_keys(const Src &src, int64_t n, F f,
                                         uint64_t *tstate = nullptr) {
    __shared__ uint64_t s_base;
    if (threadIdx.x < 32) {
        const uint64_t b = src.block_base();
        if (threadIdx.x == 0) s_base = b;
    }
    __syncthreads();
    const int64_t q0 = (int64_t)blockIdx.x * KEYS_PER_BLOCK + (int64_t)threadIdx.x * KPT;
    if (q0 >= n) return;
    const uint64_t s = thread_apply(s_base);
    if (tstate) tstate[(size_t)blockIdx.x * PERM_THREADS + threadIdx.x] = s;
    walk_keys(s, n, f);
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

// ------------------------------------------------- bucket-region variant
constexpr int V2_MAX_LOG = 21;
constexpr int BCAP = 1024;             // pairs per bucket region (<= 512 expected)
constexpr int BS2_THREADS = 256;

__device__ __forceinline__ uint32_t bucket_of(uint32_t k, int nb) {
    return nb ? k >> (32 - nb) : 0u;
}

__device__ __forceinline__ uint32_t block_excl_scan_256(uint32_t x, uint32_t *s_warp) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_warp[w] = inc;
    __syncthreads();
    uint32_t pre = inc - x;
    for (int j = 0; j < w; ++j) pre += s_warp[j];
    return pre;
}

// <= 48 registers (5 CTAs per SM worth): a CTA fits beside the two CTAs of
// the epoch kernel (scd.cu, 104 registers), so the next round's permutation
// runs under the epoch (GLM_PERM_LEAN overrides for experiments)
#ifndef GLM_PERM_LEAN
#define GLM_PERM_LEAN 5
#endif
#define PERM_BOUNDS __launch_bounds__(PERM_THREADS, GLM_PERM_LEAN)

// Pass 1.  ctl: [0] ticket, [1] overflow count, [2] overflow total (for pass 2);
// cnt: per-bucket totals.  Both are zero between uses (the last CTA resets).
template <class Src>
__global__ void PERM_BOUNDS region_scatter_kernel(
    Src src, int64_t n, int nb, uint32_t cap, uint32_t *cnt, uint32_t *boff, uint32_t *ctl,
    uint64_t *region, uint64_t *ovf, uint32_t *ovf_b) {
    if (src.skip()) return;
    tl_start(TL_PERM_FIRST);
    extern __shared__ uint32_t h3[];
    __shared__ uint64_t s_base;
    __shared__ uint32_t s_warp[PERM_THREADS / 32];
    __shared__ bool s_last;
    const int NB = 1 << nb;
    for (int i = threadIdx.x; i < NB; i += PERM_THREADS) h3[i] = 0;
    if (threadIdx.x < 32) {
        const uint64_t b = src.block_base();
        if (threadIdx.x == 0) s_base = b;
    }
    __syncthreads();
    const int64_t q0 = (int64_t)blockIdx.x * KEYS_PER_BLOCK + (int64_t)threadIdx.x * KPT;
    const uint64_t s = q0 < n ? thread_apply(s_base) : 0ULL;
    walk_keys(s, n, [&](int64_t, uint32_t k) { atomicAdd(h3 + bucket_of(k, nb), 1u); });
    __syncthreads();
    {   // reserve this block's runs: every atomic in flight before any result is used
        constexpr int PER = (1 << 12) / PERM_THREADS;
        uint32_t r[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int i = threadIdx.x + j * PERM_THREADS;
            const uint32_t c = i < NB ? h3[i] : 0u;
            r[j] = c ? atomicAdd(cnt + i, c) : 0u;
        }
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int i = threadIdx.x + j * PERM_THREADS;
            if (i < NB) h3[i] = r[j];
        }
    }
    __syncthreads();
    walk_keys(s, n, [&](int64_t q, uint32_t k) {
        const uint32_t b = bucket_of(k, nb);
        const uint32_t pos = atomicAdd(h3 + b, 1u);
        const uint64_t pr = ((uint64_t)k << 32) | (uint32_t)q;
        if (pos < cap) {
            region[(size_t)b * BCAP + pos] = pr;
        } else {
            const uint32_t o = atomicAdd(ctl + 1, 1u);
            ovf[o] = pr;
            ovf_b[o] = b;
        }
    });
    // the last CTA needs only the totals: their atomics returned before the
    // barrier, thread 0's fence orders them before the ticket (the region
    // pairs are for the next kernel, ordered by the kernel boundary)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(ctl, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {       // every block's reservations are in: bucket output offsets
        __threadfence();
        const int per = (NB + PERM_THREADS - 1) / PERM_THREADS;      // <= 16
        const int i0 = threadIdx.x * per;
        uint32_t c[16];
        uint32_t mine = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            c[j] = j < per && i0 + j < NB ? __ldcg(cnt + i0 + j) : 0u;
            mine += c[j];
        }
        uint32_t pre = block_excl_scan_256(mine, s_warp);
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (j < per && i0 + j < NB) {
                boff[i0 + j] = pre;
                pre += c[j];
                cnt[i0 + j] = 0;                 // ready for the next permutation
            }
        if (threadIdx.x == PERM_THREADS - 1) boff[NB] = pre;
        if (threadIdx.x == 0) {
            ctl[2] = atomicExch(ctl + 1, 0u);
            ctl[0] = 0;
        }
    }
    tl_end(TL_PERM_FIRST);
}

// Pass 2: one CTA per bucket.  A counting pass on the next 8 key bits spreads
// the pairs over 256 sub-buckets in shared memory (~2 pairs each), thread t
// insertion-sorts sub-bucket t by (key, index) — numpy's stable order — and
// the CTA writes its slice of the permutation coalesced.
__global__ void PERM_BOUNDS region_sort_kernel(
    const SolveState *st, const uint64_t *region, const uint32_t *boff, int nb, int cap,
    const uint32_t *ctl, const uint64_t *ovf, const uint32_t *ovf_b, uint64_t *tmp,
    int32_t *perm) {
    if (st && st->done) return;
    tl_start(TL_PERM_LAST);
    __shared__ uint64_t s_in[BCAP], s_out[BCAP];
    __shared__ uint32_t s_cur[BS2_THREADS];
    __shared__ uint32_t s_warp[BS2_THREADS / 32];
    const uint32_t lo = boff[blockIdx.x], hi = boff[blockIdx.x + 1];
    const int cnt = (int)(hi - lo);
    const uint64_t *src = region + (size_t)blockIdx.x * BCAP;
    const int t = threadIdx.x;
    if (cnt <= cap) {
        const int sh = 24 - nb;                    // the 8 key bits below the bucket bits
        s_cur[t] = 0;
        __syncthreads();
        for (int i = t; i < cnt; i += BS2_THREADS) {
            const uint64_t p = src[i];
            s_in[i] = p;
            atomicAdd(s_cur + ((uint32_t)(p >> 32) >> sh & 255u), 1u);
        }
        __syncthreads();
        const uint32_t c = s_cur[t];
        const uint32_t ex = block_excl_scan_256(c, s_warp);
        s_cur[t] = ex;
        __syncthreads();
        for (int i = t; i < cnt; i += BS2_THREADS) {
            const uint64_t p = s_in[i];
            s_out[atomicAdd(s_cur + ((uint32_t)(p >> 32) >> sh & 255u), 1u)] = p;
        }
        __syncthreads();
        insertion_sort(s_out + ex, (int)c);
        __syncthreads();
        for (int i = t; i < cnt; i += BS2_THREADS) perm[lo + i] = (int32_t)(uint32_t)s_out[i];
    } else {            // the bucket outgrew its region: region + overflow list, slowly
        for (int i = t; i < cap; i += BS2_THREADS) tmp[lo + i] = src[i];
        if (t == 0) {
            int w = cap;
            const uint32_t no = ctl[2];
            for (uint32_t o = 0; o < no; ++o)
                if (ovf_b[o] == blockIdx.x) tmp[lo + w++] = ovf[o];
        }
        __syncthreads();
        if (t == 0) insertion_sort(tmp + lo, cnt);
        __syncthreads();
        for (int i = t; i < cnt; i += BS2_THREADS) perm[lo + i] = (int32_t)(uint32_t)tmp[lo + i];
    }
    tl_end(TL_PERM_LAST);
}

// Usable pairs per bucket region: BCAP; GLM_PERM_REGION_CAP (tests) lowers it
// so that buckets overflow and the slow path runs.
static int region_cap() {
    static const int v = [] {
        const char *e = getenv("GLM_PERM_REGION_CAP");
        const int c = e ? atoi(e) : BCAP;
        return c >= 1 && c <= BCAP ? c : BCAP;
    }();
    return v;
}

static int v2_bits(int64_t n) {       // <= 512 keys per bucket on average, <= 4096 buckets
    int lg = 0;
    while ((1LL << lg) < n) ++lg;
    int nb = lg - 9;
    if (nb < 0) nb = 0;
    if (nb > 12) nb = 12;
    return nb;
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

// Layout (offsets depend only on `capacity`, so the zeroed counters stay in
// place across calls with different n; every kernel re-zeroes what it used):
//   head: hist | offs | cursor | tile sums | ctl[64] | cnt | boff   (zeroed once)
//   bulk: pairs[capacity] | bucket regions | overflow pairs | overflow buckets
namespace {
struct Layout {
    size_t hist, offs, cursor, flags, ctl, cnt, boff, head;
    size_t pairs, region, ovf, ovf_b, total;
    int64_t nbk_cap, nb2_cap, c2;
};
size_t up256(size_t x) { return (x + 255) & ~(size_t)255; }
Layout layout(int64_t capacity) {
    Layout L{};
    const int64_t cap = capacity > 0 ? capacity : 1;
    L.nbk_cap = 1LL << bucket_bits(cap);
    L.c2 = std::min<int64_t>(cap, 1LL << V2_MAX_LOG);
    L.nb2_cap = 1LL << v2_bits(L.c2);
    size_t o = 0;
    L.hist = o;   o += 4 * (size_t)L.nbk_cap;
    L.offs = o;   o += 4 * (size_t)(L.nbk_cap + 1);
    L.cursor = o; o += 4 * (size_t)L.nbk_cap;
    L.flags = o;  o += 4 * (size_t)(L.nbk_cap / SCAN_TILE + 2);
    o = up256(o);
    L.ctl = o;    o += 4 * 64;
    L.cnt = o;    o += 4 * (size_t)L.nb2_cap;
    L.boff = o;   o += 4 * (size_t)(L.nb2_cap + 1);
    o = up256(o);
    L.head = o;
    L.pairs = o;  o = up256(o + 8 * (size_t)cap);
    L.region = o; o = up256(o + 8 * (size_t)(L.nb2_cap * BCAP));
    L.ovf = o;    o = up256(o + 8 * (size_t)L.c2);
    L.ovf_b = o;  o = up256(o + 4 * (size_t)L.c2);
    L.total = o;
    return L;
}
}  // namespace

size_t perm_scratch_bytes(int64_t n) { return layout(n).total; }
size_t perm_scratch_head_bytes(int64_t n) { return layout(n).head; }

PermScratch carve_perm_scratch(void *base, int64_t capacity, int64_t n) {
    const Layout L = layout(capacity);
    char *c = (char *)base;
    PermScratch p;
    p.nb = bucket_bits(n);
    p.nbk = 1LL << p.nb;
    p.hist = (uint32_t *)(c + L.hist);
    p.offs = (uint32_t *)(c + L.offs);
    p.cursor = (uint32_t *)(c + L.cursor);
    p.flags = (uint32_t *)(c + L.flags);
    p.ctl = (uint32_t *)(c + L.ctl);
    p.cnt = (uint32_t *)(c + L.cnt);
    p.boff = (uint32_t *)(c + L.boff);
    p.pairs = (uint64_t *)(c + L.pairs);
    p.region = (uint64_t *)(c + L.region);
    p.ovf = (uint64_t *)(c + L.ovf);
    p.ovf_b = (uint32_t *)(c + L.ovf_b);
    p.v2 = n <= (1LL << V2_MAX_LOG) && capacity > 0;
    p.nb2 = v2_bits(n);
    return p;
}

static int key_blocks(int64_t n) { return (int)((n + KEYS_PER_BLOCK - 1) / KEYS_PER_BLOCK); }

template <class Src>
static int perm_from_source(const Src &src, const SolveState *st, int64_t n, int32_t *perm,
                            const PermScratch &sc, cudaStream_t stream,
                            const uint32_t *keys_array) {
    if (n <= 0) return GLM_OK;
    if (!keys_array && sc.v2) {
        const int NB = 1 << sc.nb2;
        count_launch();
        region_scatter_kernel<<<key_blocks(n), PERM_THREADS, sizeof(uint32_t) * (size_t)NB,
                                stream>>>(src, n, sc.nb2, (uint32_t)region_cap(), sc.cnt, sc.boff,
                                          sc.ctl, sc.region, sc.ovf, sc.ovf_b);
        count_launch();
        region_sort_kernel<<<NB, BS2_THREADS, 0, stream>>>(st, sc.region, sc.boff, sc.nb2,
                                                           region_cap(), sc.ctl, sc.ovf, sc.ovf_b,
                                                           sc.pairs, perm);
        GLM_CUDA_TRY(cudaGetLastError());
        return GLM_OK;
    }
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
