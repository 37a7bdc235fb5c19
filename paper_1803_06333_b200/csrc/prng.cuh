// prng.cuh — device permutation stream (see prng.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace glm {
struct SolveState;

struct PermScratch {
    int nb = 0;            // bucket bits
    int64_t nbk = 0;       // number of buckets
    uint64_t *pairs = nullptr;
    uint32_t *hist = nullptr;    // zero between uses (scan re-zeroes it)
    uint32_t *offs = nullptr;    // nbk + 1
    uint32_t *cursor = nullptr;
    uint32_t *flags = nullptr;   // tile sums
    // bucket-region variant (generated keys, n <= 2^21)
    bool v2 = false;
    int nb2 = 0;
    uint32_t *ctl = nullptr;     // [0] ticket, [1] overflow count (zero between uses), [2] total
    uint32_t *cnt = nullptr;     // per-bucket totals (zero between uses)
    uint32_t *boff = nullptr;    // bucket output offsets (nb2 buckets + 1)
    uint64_t *region = nullptr;  // 1024 pairs per bucket
    uint64_t *ovf = nullptr;     // pairs beyond their region, and their buckets
    uint32_t *ovf_b = nullptr;
};

uint64_t host_jump(uint64_t state, uint64_t steps);
int ensure_device_tables();
int bucket_bits(int64_t n);
size_t perm_scratch_bytes(int64_t n);
// leading bytes holding the counters that must be zero before the first use
size_t perm_scratch_head_bytes(int64_t n);
// hist region must be zeroed once; bucket count follows n <= capacity
PermScratch carve_perm_scratch(void *base, int64_t capacity, int64_t n);
// Permutation of attempt `offset/n` of the stream whose start state is
// st->gen_state (st != nullptr; kernels skip once st->done) or `state`.
int stream_perm(const SolveState *st, uint64_t state, uint64_t offset, int64_t n,
                int32_t *perm, const PermScratch &sc, cudaStream_t stream);
// Permutation of the stream starting at the device-held state *state_dev.
int stream_perm_from(const uint64_t *state_dev, int64_t n, int32_t *perm,
                     const PermScratch &sc, cudaStream_t stream);
int chunk_perm(uint64_t seed, int64_t n, int32_t *perm, const PermScratch &sc,
               cudaStream_t stream);
int array_perm(const uint32_t *keys, int64_t n, int32_t *perm, const PermScratch &sc,
               cudaStream_t stream);
int stream_keys(uint64_t state, uint64_t offset, int64_t n, uint32_t *keys,
                cudaStream_t stream);
int chunk_keys(uint64_t seed, int64_t n, uint32_t *keys, cudaStream_t stream);
}  // namespace glm
