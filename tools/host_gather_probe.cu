// Microbenchmark: random gathers from pinned, mapped HOST memory (zero copy
// over the host link), the path BatchRunner.run takes for a pinned host cube.
// Which load flavour / request size / concurrency moves the most random
// samples per second across PCIe?
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o host_gather_probe host_gather_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
#include <sys/mman.h>

// V: 0 ld.global 8B, 1 ld.global.nc.L1::no_allocate 8B, 2 same + .L2::64B,
//    3 cp.async.ca 8B, 5 cp.async.cg 16B .L2::64B, 6 cp.async.cg 16B,
//    7 ld.global.nc.v4 16B, 8 ld.global.nc 32B (2 x v4, same sector)
template <int V>
__global__ void probe(const float2 *__restrict__ a, unsigned long long mask, int per_thread,
                      float *out, unsigned seed, int wlog) {
    __shared__ __align__(16) float2 sm[256 * 16];
    unsigned x = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
    if (wlog) {  // every warp gathers inside one random window of 2^wlog samples
        const unsigned long long w = ((unsigned long long)(seed * 7919u + (blockIdx.x * blockDim.x + threadIdx.x) / 32) * 0x9E3779B97F4A7C15ull >> 20) & mask & ~((1ull << wlog) - 1);
        a += w;
        mask = (1ull << wlog) - 1;
    }
    float acc = 0.f;
    for (int i = 0; i < per_thread; i += 8) {
        if (V <= 2 || V == 7 || V == 8) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                x = x * 1664525u + 1013904223u;
                unsigned long long j = ((unsigned long long)x * 2654435761ull) & mask;
                const float2 *p = a + j;
                if (V == 0) { float2 t = *p; v[u] = make_float4(t.x, t.y, 0, 0); }
                else if (V == 1) asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(v[u].x), "=f"(v[u].y) : "l"(p));
                else if (V == 2) asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v2.f32 {%0,%1}, [%2];" : "=f"(v[u].x), "=f"(v[u].y) : "l"(p));
                else if (V == 7) {
                    p = a + (j & ~1ull);
                    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w) : "l"(p));
                } else {
                    p = a + (j & ~3ull);
                    float4 w;
                    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w) : "l"(p));
                    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(w.x), "=f"(w.y), "=f"(w.z), "=f"(w.w) : "l"(p + 2));
                    v[u].x += w.x;
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z;
        } else {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                x = x * 1664525u + 1013904223u;
                const unsigned long long j = ((unsigned long long)x * 2654435761ull) & mask;
                const unsigned s = (unsigned)__cvta_generic_to_shared(&sm[threadIdx.x * 16 + 2 * u]);
                if (V == 3)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(a + j) : "memory");
                else if (V == 5)
                    asm volatile("cp.async.cg.shared.global.L2::64B [%0], [%1], 16;" ::"r"(s), "l"(a + (j & ~1ull)) : "memory");
                else
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(a + (j & ~1ull)) : "memory");
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += sm[threadIdx.x * 16 + 2 * u].x;
        }
    }
    if (acc == 123.f) out[0] = acc;
}

int main(int argc, char **argv) {
    const unsigned long long n = 1ull << 28;  // 2 GiB of float2
    // argv[1]: "alloc" (cudaHostAlloc, default), "thp" (mmap + MADV_HUGEPAGE +
    // cudaHostRegister), "hugetlb" (mmap MAP_HUGETLB + cudaHostRegister)
    const char *how = argc > 1 ? argv[1] : "alloc";
    float *o;
    cudaMalloc(&o, 4);
    float2 *h = nullptr, *hd = nullptr;
    if (!strcmp(how, "alloc")) {
        if (cudaHostAlloc(&h, n * sizeof(float2), cudaHostAllocMapped) != cudaSuccess) h = nullptr;
    } else {
        const size_t bytes = n * sizeof(float2);
        int fl = MAP_PRIVATE | MAP_ANONYMOUS | (!strcmp(how, "hugetlb") ? MAP_HUGETLB : 0);
        void *m = mmap(nullptr, bytes + (2 << 20), PROT_READ | PROT_WRITE, fl, -1, 0);
        if (m == MAP_FAILED) { printf("mmap %s failed\n", how); return 1; }
        char *al = (char *)(((unsigned long long)m + (2 << 20) - 1) & ~((2ull << 20) - 1));
        if (!strcmp(how, "thp")) madvise(al, bytes, MADV_HUGEPAGE);
        memset(al, 0, bytes);
        cudaError_t e = cudaHostRegister(al, bytes, cudaHostRegisterMapped);
        printf("cudaHostRegister(%s): %s\n", how, cudaGetErrorString(e));
        h = e == cudaSuccess ? (float2 *)al : nullptr;
    }
    if (!h || cudaHostGetDevicePointer(&hd, h, 0) != cudaSuccess) {
        printf("no mapped host memory\n");
        return 1;
    }
    memset(h, 0, n * sizeof(float2));
    printf("host ptr %p device ptr %p (same under UVA: %d)\n", (void *)h, (void *)hd, h == hd);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int threads = 256;
    const unsigned long long mask = n - 1;
    for (int wlog : {0, 16})
    for (int gran : {32}) {
        cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
        for (int ctas : {1184}) {
            const int per = 16;
            const double loads = (double)ctas * threads * per;
            for (int rep = 0; rep < 2; ++rep) {
#define RUNH(V)                                                                                   \
    {                                                                                             \
        cudaEventRecord(e0);                                                                      \
        probe<V><<<ctas, threads>>>(hd, mask, per, o, 29 + rep, wlog);                            \
        cudaEventRecord(e1);                                                                      \
        cudaEventSynchronize(e1);                                                                 \
        float ms;                                                                                 \
        cudaEventElapsedTime(&ms, e0, e1);                                                        \
        if (rep) printf("HOST window 2^%2d l2gran %3d ctas %4d variant %d: %8.3f ms  %.3f G requests/s\n", \
                        wlog ? wlog : 28, gran, ctas, V, ms, loads / ms / 1e6);                   \
    }
                RUNH(3) RUNH(5)
            }
        }
    }
    // bulk H2D copy rate for comparison
    {
        void *d;
        cudaMalloc(&d, n * sizeof(float2));
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            cudaMemcpyAsync(d, h, n * sizeof(float2), cudaMemcpyHostToDevice);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep) printf("H2D memcpy 2 GiB: %.3f ms  %.2f GB/s\n", ms, n * 8.0 / ms / 1e6);
        }
        cudaFree(d);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    if (!strcmp(how, "alloc")) cudaFreeHost(h);
    return 0;
}
