// HBM write-bandwidth probe for the re-synthesis store pattern (run under gpurun):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/write_probe tools/write_probe.cu
// Modes: 0 = 16-byte stores, a warp writes 512 contiguous bytes; 1 = 8-byte stores, 256
// contiguous bytes per warp store; 2 = the synth512 pattern (each half-warp one 128-byte line,
// the two lines 4 KB apart, successive stores 128 B on); 3 = mode 2 with default (non-streaming)
// stores.  One CTA of 256 threads per 2 MiB frame, 2 CTAs per SM, like synth512_kernel.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(256, 2) wr(float2 *out) {
    float2 *img = out + (size_t)blockIdx.x * 512 * 512;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float2 v = make_float2((float)threadIdx.x, (float)blockIdx.x);
    if (MODE == 0) {
        float4 *p = (float4 *)img;
        for (int i = threadIdx.x; i < 512 * 512 / 2; i += 256) __stcs(p + i, make_float4(v.x, v.y, v.x, v.y));
    } else if (MODE == 1) {
        for (int i = threadIdx.x; i < 512 * 512; i += 256) __stcs(img + i, v);
    } else {
        const int cc = lane & 15, q = lane >> 4;
        for (int r0 = 0; r0 < 512; r0 += 16) {
            float2 *row = img + (size_t)(r0 + warp * 2 + q) * 512 + cc;
#pragma unroll
            for (int d = 0; d < 32; ++d) {
                if (MODE == 2) __stcs(row + 16 * d, v);
                else row[16 * d] = v;
            }
        }
    }
}
int main() {
    const int B = 2048;
    float2 *out;
    cudaMalloc(&out, (size_t)B * 512 * 512 * 8);
    cudaEvent_t s, e;
    cudaEventCreate(&s); cudaEventCreate(&e);
    for (int mode = 0; mode < 4; ++mode) {
        float best = 1e9;
        for (int rep = 0; rep < 6; ++rep) {
            cudaEventRecord(s);
            if (mode == 0) wr<0><<<B, 256>>>(out);
            if (mode == 1) wr<1><<<B, 256>>>(out);
            if (mode == 2) wr<2><<<B, 256>>>(out);
            if (mode == 3) wr<3><<<B, 256>>>(out);
            cudaEventRecord(e); cudaEventSynchronize(e);
            float ms; cudaEventElapsedTime(&ms, s, e);
            if (rep && ms < best) best = ms;
        }
        printf("mode %d: %.3f ms  %.0f GB/s written\n", mode, best, (double)B * 512 * 512 * 8 / best / 1e6);
    }
    cudaMemset(out, 0, (size_t)B * 512 * 512 * 8);
    cudaEventRecord(s);
    cudaMemsetAsync(out, 1, (size_t)B * 512 * 512 * 8);
    cudaEventRecord(e); cudaEventSynchronize(e);
    float ms; cudaEventElapsedTime(&ms, s, e);
    printf("cudaMemset: %.3f ms  %.0f GB/s\n", ms, (double)B * 512 * 512 * 8 / ms / 1e6);
    return 0;
}
