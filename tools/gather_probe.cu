// Microbenchmark: random 8-byte gathers from HBM with different load paths,
// array sizes and SM counts, to find what bounds the FPS-SFT line gather.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_probe gather_probe.cu
// run under ncu for dram__bytes_read.sum / lts__t_sectors_srcunit_tex_op_read.sum.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

template <int V>
__device__ __forceinline__ float2 ld(const float2 *p) {
    float2 v;
    if (V == 0) v = *p;
    else if (V == 1) asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    else asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    return v;
}

template <int V>
__global__ void probe(const float2 *__restrict__ a, unsigned long long mask, int per_thread,
                      float *out, unsigned seed) {
    __shared__ __align__(16) float2 sm[256 * 8 + 16];
    __shared__ __align__(8) unsigned long long bar;
    unsigned x = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
    float acc = 0.f;
    if (V == 4 && threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)), "r"(blockDim.x));
    }
    __syncthreads();
    unsigned phase = 0;
    for (int i = 0; i < per_thread; i += 8) {
        if (V <= 2) {
            float2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                x = x * 1664525u + 1013904223u;
                const unsigned long long j = ((unsigned long long)x * 2654435761ull) & mask;
                v[u] = ld<V>(a + j);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y;
        } else if (V == 3) {  // cp.async.ca 8B -> smem
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                x = x * 1664525u + 1013904223u;
                const unsigned long long j = ((unsigned long long)x * 2654435761ull) & mask;
                const unsigned s = (unsigned)__cvta_generic_to_shared(&sm[threadIdx.x * 8 + u]);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(a + j) : "memory");
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += sm[threadIdx.x * 8 + u].x;
        } else {  // TMA 1-D bulk copy of the 16-byte chunk holding the sample
            const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(16 * 4) : "memory");
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                x = x * 1664525u + 1013904223u;
                const unsigned long long j = (((unsigned long long)x * 2654435761ull) & mask) & ~1ull;
                const unsigned s = (unsigned)__cvta_generic_to_shared(&sm[threadIdx.x * 8 + 2 * u]);
                asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];"
                             ::"r"(s), "l"(a + j), "r"(b) : "memory");
            }
            unsigned done = 0;
            while (!done)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                             : "=r"(done) : "r"(b), "r"(phase) : "memory");
            phase ^= 1;
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += sm[threadIdx.x * 8 + u].x;
            __syncthreads();
        }
    }
    if (acc == 123.f) out[0] = acc;
}

int main(int argc, char **argv) {
    const unsigned long long n = 1ull << 28;  // 2 GiB of float2
    float2 *a;
    float *o;
    cudaMalloc(&a, n * sizeof(float2));
    cudaMalloc(&o, 4);
    cudaMemset(a, 0, n * sizeof(float2));
    const int threads = 256, per = 64;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Case { int logn, sms; } cases[] = {{28, 148}, {28, 74}, {28, 37}, {25, 148}, {22, 148}};
    for (auto c : cases) {
        const unsigned long long mask = (1ull << c.logn) - 1;
        const int blocks = c.sms * 8;
        const double loads = (double)blocks * threads * per;
        for (int rep = 0; rep < 2; ++rep) {
#define RUN(V)                                                                            \
    {                                                                                     \
        cudaEventRecord(e0);                                                              \
        probe<V><<<blocks, threads>>>(a, mask, per, o, 17 + rep);                         \
        cudaEventRecord(e1);                                                              \
        cudaEventSynchronize(e1);                                                         \
        float ms;                                                                         \
        cudaEventElapsedTime(&ms, e0, e1);                                                \
        if (rep) printf("array 2^%d x8B  ctas %4d  variant %d: %.3f ms  %.2f Gsamples/s\n", \
                        c.logn, blocks, V, ms, loads / ms / 1e6);                         \
    }
            RUN(0) RUN(2) RUN(3) RUN(4)
        }
    }
    // zero-copy: the same random 8-byte gathers from pinned, mapped host memory
    {
        float2 *h = nullptr, *hd = nullptr;
        if (cudaHostAlloc(&h, n * sizeof(float2), cudaHostAllocMapped) == cudaSuccess &&
            cudaHostGetDevicePointer(&hd, h, 0) == cudaSuccess) {
            memset(h, 0, n * sizeof(float2));
            const unsigned long long mask = n - 1;
            for (int sms : {148, 74}) {
                const int blocks = sms * 8;
                const double loads = (double)blocks * threads * per;
                for (int rep = 0; rep < 2; ++rep) {
#define RUNH(V)                                                                            \
    {                                                                                      \
        cudaEventRecord(e0);                                                               \
        probe<V><<<blocks, threads>>>(hd, mask, per, o, 29 + rep);                         \
        cudaEventRecord(e1);                                                               \
        cudaEventSynchronize(e1);                                                          \
        float ms;                                                                          \
        cudaEventElapsedTime(&ms, e0, e1);                                                 \
        if (rep) printf("HOST-MAPPED 2^28 x8B  ctas %4d  variant %d: %.3f ms  %.3f Gsamples/s\n", \
                        blocks, V, ms, loads / ms / 1e6);                                  \
    }
                    RUNH(0) RUNH(3)
                }
            }
            cudaFreeHost(h);
        } else {
            printf("no mapped host memory\n");
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
