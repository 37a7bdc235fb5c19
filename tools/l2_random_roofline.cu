// l2_random_roofline.cu — the L2 random-access ceiling the TPA-SCD epoch runs
// against (C2: every nnz is one random 8-byte gather and one random f64 red
// into an 800 KB shared vector that lives in L2).
//
// Measures, on one B200, with CUDA events (best of 20 after warm-up):
//   gather : N random ld.global.cg.f64 from a V-double vector
//   red    : N random red.global.add.f64 into it
//   mixed  : N gathers + N reds (the epoch's shared-vector traffic)
//   stream : a 480 MB coalesced read (the epoch's column stream), for scale
// Random indices come from a per-thread xorshift (no index array traffic).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_random_roofline tools/l2_random_roofline.cu
//   ./l2_random_roofline [V=100000] [N=40000000]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ unsigned xs(unsigned &s) {
    s ^= s << 13; s ^= s >> 17; s ^= s << 5; return s;
}

__global__ void gather_k(const double *v, unsigned V, long long n, double *sink) {
    unsigned s = 0x9E3779B9u ^ (blockIdx.x * 1024 + threadIdx.x) * 2654435761u;
    double acc = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double x;
        asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(x) : "l"(v + xs(s) % V));
        acc += x;
    }
    if (acc == 12345.678) sink[0] = acc;
}

__global__ void red_k(double *v, unsigned V, long long n) {
    unsigned s = 0x7F4A7C15u ^ (blockIdx.x * 1024 + threadIdx.x) * 2246822519u;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        asm volatile("red.global.add.f64 [%0], %1;" ::"l"(v + xs(s) % V), "d"(1e-9) : "memory");
}

__global__ void mixed_k(double *v, unsigned V, long long n, double *sink) {
    unsigned s = 0x1234567u ^ (blockIdx.x * 1024 + threadIdx.x) * 3266489917u;
    double acc = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double x;
        asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(x) : "l"(v + xs(s) % V));
        acc += x;
        asm volatile("red.global.add.f64 [%0], %1;" ::"l"(v + xs(s) % V), "d"(1e-9) : "memory");
    }
    if (acc == 12345.678) sink[0] = acc;
}

__global__ void stream_k(const double2 *a, long long n2, double *sink) {
    double acc = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2;
         i += (long long)gridDim.x * blockDim.x) {
        double2 x = __ldg(a + i);
        acc += x.x + x.y;
    }
    if (acc == 12345.678) sink[0] = acc;
}

template <class F>
float best_ms(F launch) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int i = 0; i < 3; ++i) launch();
    float best = 1e30f;
    for (int i = 0; i < 20; ++i) {
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
    const long long SB = 480LL << 20;
    double2 *big;
    CK(cudaMalloc(&big, SB));
    CK(cudaMemset(big, 0, SB));
    const int grid = sms * 8, block = 256;
    float g = best_ms([&] { gather_k<<<grid, block>>>(v, V, N, sink); });
    float r = best_ms([&] { red_k<<<grid, block>>>(v, V, N); });
    float m = best_ms([&] { mixed_k<<<grid, block>>>(v, V, N, sink); });
    float s = best_ms([&] { stream_k<<<grid, block>>>(big, SB / 16, sink); });
    CK(cudaGetLastError());
    printf("{\"vector_doubles\": %u, \"ops\": %lld, \"gather_ms\": %.4f, \"red_ms\": %.4f, "
           "\"mixed_ms\": %.4f, \"stream480MB_ms\": %.4f, \"gather_Gops\": %.2f, "
           "\"red_Gops\": %.2f, \"mixed_Gpairs\": %.2f, \"stream_GBps\": %.1f}\n",
           V, N, g, r, m, s, N / g / 1e6, N / r / 1e6, N / m / 1e6, SB / s / 1e6);
    return 0;
}
