// view_ceiling.cu — where can the shared view of the TPA-SCD epoch live, and
// what does a random 8-byte gather + f64 add cost there?  (VERDICT r1 next
// #3: measure the alternatives to the L2-resident shared vector.)
//
// The C2 epoch does nnz random gathers and nnz random adds into a d-double
// view (d = 100k, 800 KB).  Candidates, each doing N gathers + N adds
// (random indices from a per-thread xorshift, no index traffic):
//   l2      : global view in L2 (ld.global.cg + red.global.add.f64) — today
//   l2_ca   : gathers through L1 (ld.global.ca)
//   dsmem C : the view sharded over the C CTAs of a thread-block cluster
//             (1 CTA per SM, d/C doubles each); gathers and adds go to the
//             owning CTA's shared memory (ld/red .shared::cluster)
//   smem    : a private per-CTA view of the same size per SM (only fits
//             for d <= 27k doubles: the fastest place there is, for scale)
// Best of 10 after warm-up, CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o view_ceiling tools/view_ceiling.cu
//   ./view_ceiling [d=100000] [N=40000000]
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ unsigned xs(unsigned &s) {
    s ^= s << 13; s ^= s >> 17; s ^= s << 5; return s;
}

template <bool CA>
__global__ void l2_k(double *v, unsigned V, long long n, double *sink) {
    unsigned s = 0x1234567u ^ (blockIdx.x * 1024 + threadIdx.x) * 3266489917u;
    double acc = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double x;
        if (CA) asm volatile("ld.global.ca.f64 %0, [%1];" : "=d"(x) : "l"(v + xs(s) % V));
        else asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(x) : "l"(v + xs(s) % V));
        acc += x;
        asm volatile("red.global.add.f64 [%0], %1;" ::"l"(v + xs(s) % V), "d"(1e-9) : "memory");
    }
    if (acc == 12345.678) sink[0] = acc;
}

// view sharded over the cluster: element i lives in CTA (i % C) at i / C
__global__ void dsmem_k(unsigned V, long long n_per_cluster, double *sink) {
    extern __shared__ double sv[];
    cg::cluster_group cl = cg::this_cluster();
    const unsigned C = cl.num_blocks();
    const unsigned me = cl.block_rank();
    const unsigned per = (V + C - 1) / C;
    for (unsigned i = threadIdx.x; i < per; i += blockDim.x) sv[i] = 0.0;
    cl.sync();
    double *base[16];
    for (unsigned r = 0; r < C; ++r) base[r] = cl.map_shared_rank(sv, r);
    unsigned s = 0x9E3779B9u ^ (blockIdx.x * 1024 + threadIdx.x) * 2654435761u;
    double acc = 0.0;
    const long long stride = (long long)C * blockDim.x;
    for (long long i = (long long)me * blockDim.x + threadIdx.x; i < n_per_cluster; i += stride) {
        const unsigned a = xs(s) % V, b = xs(s) % V;
        acc += base[a % C][a / C];
        atomicAdd(base[b % C] + b / C, 1e-9);
    }
    cl.sync();
    if (acc == 12345.678) sink[0] = acc;
}

__global__ void smem_k(unsigned V, long long n, double *sink) {
    extern __shared__ double sv[];
    for (unsigned i = threadIdx.x; i < V; i += blockDim.x) sv[i] = 0.0;
    __syncthreads();
    unsigned s = 0x7F4A7C15u ^ (blockIdx.x * 1024 + threadIdx.x) * 2246822519u;
    double acc = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned a = xs(s) % V, b = xs(s) % V;
        acc += sv[a];
        atomicAdd(sv + b, 1e-9);
    }
    __syncthreads();
    if (acc == 12345.678) sink[0] = acc;
}

template <class F>
float best_ms(F launch) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int i = 0; i < 2; ++i) launch();
    CK(cudaGetLastError());
    float best = 1e30f;
    for (int i = 0; i < 10; ++i) {
        CK(cudaEventRecord(a));
        launch();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (ms < best) best = ms;
    }
    return best;
}

int main(int argc, char **argv) {
    const unsigned V = argc > 1 ? (unsigned)atol(argv[1]) : 100000u;
    const long long N = argc > 2 ? atoll(argv[2]) : 40000000LL;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    double *v, *sink;
    CK(cudaMalloc(&v, sizeof(double) * V));
    CK(cudaMemset(v, 0, sizeof(double) * V));
    CK(cudaMalloc(&sink, 64));
    printf("{\"d\": %u, \"ops\": %lld", V, N);
    const float l2 = best_ms([&] { l2_k<false><<<sms * 8, 256>>>(v, V, N, sink); });
    const float l2ca = best_ms([&] { l2_k<true><<<sms * 8, 256>>>(v, V, N, sink); });
    printf(", \"l2_ms\": %.4f, \"l2_ca_ms\": %.4f", l2, l2ca);
    for (int C : {2, 4, 8, 16}) {
        const size_t smem = sizeof(double) * ((V + C - 1) / C);
        if (smem > 227 * 1024) continue;
        CK(cudaFuncSetAttribute(dsmem_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        if (C > 8)
            CK(cudaFuncSetAttribute(dsmem_k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        const int clusters = sms / C;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(clusters * C);
        cfg.blockDim = dim3(1024);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, dsmem_k, &cfg) != cudaSuccess || nc < 1) {
            cudaGetLastError();
            printf(", \"dsmem%d\": \"not schedulable\"", C);
            continue;
        }
        cfg.gridDim = dim3((nc < clusters ? nc : clusters) * C);
        const long long per = N / (cfg.gridDim.x / C);
        const float t = best_ms([&] { CK(cudaLaunchKernelEx(&cfg, dsmem_k, V, per, sink)); });
        printf(", \"dsmem%d_ms\": %.4f, \"dsmem%d_clusters\": %d", C, t, C, cfg.gridDim.x / C);
    }
    {
        const unsigned Vs = 27000;     // ~211 KB: the largest private view per SM
        const size_t smem = sizeof(double) * Vs;
        CK(cudaFuncSetAttribute(smem_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const float t = best_ms([&] { smem_k<<<sms, 1024, smem>>>(Vs, N, sink); });
        printf(", \"smem27k_ms\": %.4f", t);
    }
    printf("}\n");
    return 0;
}
