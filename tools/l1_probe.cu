// Microbenchmark: does the L1 share of the SM's unified L1/shared memory bound
// the rate of random 8-byte gathers?  Same random-gather loop as
// gather_probe.cu, with dynamic shared memory padded so that S KB per SM are
// carved out as shared memory (4 CTAs of 256 threads per SM), for several load
// flavours:
//   0 ld.global                    2 ld.global.nc.L1::no_allocate
//   3 cp.async.ca 8 B -> smem       5 ld.global.cg (L2 only)
//   6 cp.async.cg 16 B (the aligned chunk holding the sample) -> smem
//   8 ld.global.nc.L1::no_allocate.v4 (aligned 16 B chunk)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l1_probe l1_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__global__ void __launch_bounds__(256) probe(const float2 *__restrict__ a, unsigned long long mask,
                                             int per_thread, float *out, unsigned seed) {
    extern __shared__ __align__(16) float4 st[];  // cp.async staging, then padding
    unsigned x = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
    float acc = 0.f;
    for (int i = 0; i < per_thread; i += 8) {
        if (V == 3 || V == 6) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                x = x * 1664525u + 1013904223u;
                unsigned long long j = ((unsigned long long)x * 2654435761ull) & mask;
                const unsigned s = (unsigned)__cvta_generic_to_shared(&st[threadIdx.x * 8 + u]);
                if (V == 3)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(a + j)
                                 : "memory");
                else
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s),
                                 "l"(a + (j & ~1ull))
                                 : "memory");
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += st[threadIdx.x * 8 + u].x;
        } else {
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                x = x * 1664525u + 1013904223u;
                const unsigned long long j = ((unsigned long long)x * 2654435761ull) & mask;
                const float2 *p = a + j;
                float2 r;
                if (V == 0) {
                    r = *p;
                } else if (V == 2) {
                    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];"
                                 : "=f"(r.x), "=f"(r.y) : "l"(p));
                } else if (V == 5) {
                    asm volatile("ld.global.cg.v2.f32 {%0,%1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
                } else {
                    float4 q;
                    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                                 : "=f"(q.x), "=f"(q.y), "=f"(q.z), "=f"(q.w)
                                 : "l"(a + (j & ~1ull)));
                    r = make_float2(q.x + q.z, q.y + q.w);
                }
                v[u] = r.x + r.y;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += v[u];
        }
    }
    if (acc == 123.f) out[0] = acc;
}

template <int V>
void run(const float2 *a, unsigned long long mask, float *o, int smem_kb_per_sm, int sms) {
    const int threads = 256, per = 64, ctas_per_sm = 4;
    const int blocks = sms * ctas_per_sm;
    const int need = (V == 3 || V == 6) ? 256 * 8 * 16 : 0;  // staging per CTA
    int dyn = smem_kb_per_sm * 1024 / ctas_per_sm - 1024;
    if (dyn < 0) dyn = 0;
    if (dyn < need) return;
    cudaFuncSetAttribute(probe<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, probe<V>, threads, dyn);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        probe<V><<<blocks, threads, dyn>>>(a, mask, per, o, 17 + rep);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
    }
    const double loads = (double)blocks * threads * per;
    printf("variant %d  smem/SM %3d KB (dyn %6d B/CTA, %d CTAs/SM resident): %.3f ms  %.2f G loads/s\n",
           V, smem_kb_per_sm, dyn, occ, ms, loads / ms / 1e6);
}

int main() {
    const unsigned long long n = 1ull << 28;  // 2 GiB of float2
    float2 *a;
    float *o;
    cudaMalloc(&a, n * sizeof(float2));
    cudaMalloc(&o, 4);
    cudaMemset(a, 0, n * sizeof(float2));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const unsigned long long mask = n - 1;
    for (int kb : {0, 64, 100, 132, 164, 196, 220}) {
        run<0>(a, mask, o, kb, sms);
        run<2>(a, mask, o, kb, sms);
        run<3>(a, mask, o, kb, sms);
        run<5>(a, mask, o, kb, sms);
        run<6>(a, mask, o, kb, sms);
        run<8>(a, mask, o, kb, sms);
    }
    printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
