// Microbenchmark: random S-byte segments (S = 64 ... 1024) read by the SMs from
// pinned, mapped HOST memory -- does a wider interleave group (more instances
// per sample position, so a longer contiguous segment per request) move more
// bytes per second over PCIe than the 128-byte segments of the 16-wide group
// kernel?  Two issue flavours: (0) 16-byte ld.global.nc per lane, S/16 lanes
// per segment, 12 loads in flight per thread (the GroupGather pattern);
// (1) one cp.async.bulk (TMA, 1-D) of S bytes per segment into shared memory.
// Every CTA reads inside its own window of 65536 segments (one 256 x 256 group
// cube).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o seg_probe seg_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ float4 ld16(const void *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

template <int S>
__global__ void __launch_bounds__(256, 2) seg_ld(const char *__restrict__ a, unsigned long long nwin,
                                                  int rounds, float *out, unsigned seed) {
    constexpr int LPS = S / 16;        // lanes per segment
    constexpr int SPR = 256 / LPS;     // segments per CTA-wide load
    const int tid = threadIdx.x, c = tid % LPS, q = tid / LPS;
    unsigned long long w = ((unsigned long long)(seed * 7919u + blockIdx.x) * 0x9E3779B97F4A7C15ull >> 17) % nwin;
    const char *base = a + w * (65536ull * S);
    unsigned x = seed ^ (blockIdx.x * 977u + 13u);
    float acc = 0.f;
    for (int r = 0; r < rounds; ++r) {
        float4 v[12];
#pragma unroll
        for (int u = 0; u < 12; ++u) {
            x = x * 1664525u + 1013904223u;  // same stream in every thread of the CTA
            const unsigned pos = (((x >> 8) * 2654435761u) >> 8) + (unsigned)q * 40503u;
            v[u] = ld16(base + (unsigned long long)(pos & 65535u) * S + 16 * c);
        }
#pragma unroll
        for (int u = 0; u < 12; ++u) acc += v[u].x + v[u].w;
    }
    if (acc == 123.f) out[0] = acc + SPR;
}

template <int S>
__global__ void __launch_bounds__(256, 2) seg_bulk(const char *__restrict__ a, unsigned long long nwin,
                                                    int rounds, float *out, unsigned seed) {
    constexpr int NB = 96 * 1024 / S > 256 ? 256 : 96 * 1024 / S;  // copies in flight per CTA
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) unsigned long long mbar;
    const int tid = threadIdx.x;
    unsigned long long w = ((unsigned long long)(seed * 7919u + blockIdx.x) * 0x9E3779B97F4A7C15ull >> 17) % nwin;
    const char *base = a + w * (65536ull * S);
    const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(mb));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    unsigned x = seed ^ (blockIdx.x * 977u + 13u) ^ (tid * 2654435761u);
    float acc = 0.f;
    unsigned phase = 0;
    for (int r = 0; r < rounds; ++r) {
        if (tid == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(mb), "r"(NB * S) : "memory");
        __syncthreads();
        if (tid < NB) {
            x = x * 1664525u + 1013904223u;
            const unsigned pos = ((x >> 8) * 2654435761u) >> 8;
            const unsigned dst = (unsigned)__cvta_generic_to_shared(sm + tid * S);
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(dst), "l"(base + (unsigned long long)(pos & 65535u) * S), "r"(S), "r"(mb) : "memory");
        }
        unsigned done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(done) : "r"(mb), "r"(phase) : "memory");
        phase ^= 1;
        acc += ((const float *)sm)[tid];
        __syncthreads();
    }
    if (acc == 123.f) out[0] = acc;
}

int main() {
    const unsigned long long bytes = 2ull << 30;
    char *h = nullptr, *hd = nullptr;
    float *o;
    cudaMalloc(&o, 4);
    if (cudaHostAlloc(&h, bytes, cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(&hd, h, 0) != cudaSuccess) {
        printf("no mapped host memory\n");
        return 1;
    }
    for (unsigned long long i = 0; i < bytes; i += 4096) h[i] = 1;
    char *d;
    cudaMalloc(&d, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 32);
    const int ctas = 296;
#define RUN(NAME, KERN, S, SRC, SEGS_PER_ROUND, SMEM)                                              \
    for (int rep = 0; rep < 3; ++rep) {                                                            \
        const int rounds = 64;                                                                     \
        cudaFuncSetAttribute(KERN<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);          \
        cudaEventRecord(e0);                                                                       \
        KERN<S><<<ctas, 256, SMEM>>>(SRC, bytes / (65536ull * S), rounds, o, 31 + rep);            \
        cudaEventRecord(e1);                                                                       \
        cudaEventSynchronize(e1);                                                                  \
        float ms;                                                                                  \
        cudaEventElapsedTime(&ms, e0, e1);                                                         \
        const double segs = (double)ctas * rounds * (SEGS_PER_ROUND);                              \
        if (rep == 2)                                                                              \
            printf("%-6s %-5s S=%4d: %8.3f ms  %7.4f G segments/s  %7.2f GB/s  (%s)\n", NAME,      \
                   SRC == hd ? "HOST" : "HBM", S, ms, segs / ms / 1e6, segs * S / ms / 1e6,        \
                   cudaGetErrorString(cudaGetLastError()));                                        \
    }
#define ALL(SRC)                                                                                   \
    RUN("ld16", seg_ld, 64, SRC, 12 * 256 / 4, 0)                                                  \
    RUN("ld16", seg_ld, 128, SRC, 12 * 256 / 8, 0)                                                 \
    RUN("ld16", seg_ld, 256, SRC, 12 * 256 / 16, 0)                                                \
    RUN("ld16", seg_ld, 512, SRC, 12 * 256 / 32, 0)                                                \
    RUN("ld16", seg_ld, 1024, SRC, 12 * 256 / 64, 0)                                               \
    RUN("bulk", seg_bulk, 64, SRC, 256, 96 * 1024)                                                 \
    RUN("bulk", seg_bulk, 128, SRC, 256, 96 * 1024)                                                \
    RUN("bulk", seg_bulk, 256, SRC, 256, 96 * 1024)                                                \
    RUN("bulk", seg_bulk, 512, SRC, 192, 96 * 1024)                                                \
    RUN("bulk", seg_bulk, 1024, SRC, 96, 96 * 1024)
    ALL(hd)
    ALL(d)
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
