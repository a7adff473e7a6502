// FP32 pipe probe (run under gpurun): warp-instructions per cycle per SM partition for
// FFMA (3 registers), FADD, FMUL by an immediate, FFMA2 / FADD2 (packed) and a FADD + FFMA mix.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp32_probe tools/fp32_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
template <int MODE>
__global__ void __launch_bounds__(256) k(float *out, float a, float b, int iters) {
    float x[8];
    u64 p[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x + i; p[i] = ((u64)__float_as_uint(x[i]) << 32) | __float_as_uint(a + i); }
    u64 pa = ((u64)__float_as_uint(a) << 32) | __float_as_uint(b), pb = ((u64)__float_as_uint(b) << 32) | __float_as_uint(a);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (MODE == 0) x[i] = fmaf(x[i], a, b);
                if (MODE == 1) x[i] = x[i] + a;
                if (MODE == 2) x[i] = x[i] * 1.0001f;
                if (MODE == 3) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(pa), "l"(pb));
                if (MODE == 4) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(pa));
                if (MODE == 5) x[i] = (i & 1) ? fmaf(x[i], a, b) : x[i] + a;
                if (MODE == 6) x[i] = fmaf(x[i], 1.0001f, b);
            }
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i] + __uint_as_float((unsigned)p[i]) + __uint_as_float((unsigned)(p[i] >> 32));
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float *out; cudaMalloc(&out, 148 * 8 * 256 * 4);
    cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
    const char *names[] = {"FFMA 3-reg", "FADD", "FMUL imm", "FFMA2", "FADD2", "FADD+FFMA mix", "FFMA imm"};
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int wpsm = 4; wpsm <= 32; wpsm *= 2)
    for (int mode = 0; mode < 7; ++mode) {
        const int iters = 20000, blocks = 148 * wpsm / 8; float ms = 0;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(s);
            if (mode == 0) k<0><<<blocks, 256>>>(out, 1.0001f, 0.5f, iters);
            if (mode == 1) k<1><<<blocks, 256>>>(out, 1.0001f, 0.5f, iters);
            if (mode == 2) k<2><<<blocks, 256>>>(out, 1.0001f, 0.5f, iters);
            if (mode == 3) k<3><<<blocks, 256>>>(out, 1.0001f, 0.5f, iters);
            if (mode == 4) k<4><<<blocks, 256>>>(out, 1.0001f, 0.5f, iters);
            if (mode == 5) k<5><<<blocks, 256>>>(out, 1.0001f, 0.5f, iters);
            if (mode == 6) k<6><<<blocks, 256>>>(out, 1.0001f, 0.5f, iters);
            cudaEventRecord(e); cudaEventSynchronize(e); cudaEventElapsedTime(&ms, s, e);
        }
        const double winstr = (double)iters * 32 * wpsm;  // per SM
        printf("%2d warps/SM %-14s %.3f warp-instr / cycle / SMSP (at %d MHz)\n", wpsm, names[mode],
               winstr / 4 / (ms * 1e-3 * clk * 1e3), clk / 1000);
    }
    return 0;
}
