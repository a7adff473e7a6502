// Device building blocks of the B200-native FPS-SFT recovery loop.
//
// One CTA owns one instance (one cube) and keeps everything of its recovery
// on chip: the D+1 line spectra, the L-entry root table, the recovered set
// (slot table + open-addressing hash), and per-bin scratch.  The building
// blocks below are shared by the fused loop kernel and by the per-function
// kernels that mirror the reference's individual functions.
//
// Reference map (paths under /root/reference/pkg/src/fps_sft/):
//   gather_lines      lines.py:36-64, core.py:236-238
//   fft_lines         transform.py:17-22 (numpy pocketfft, 1/L normalised)
//   project_bins      decoder.py:172-191, numtheory.py:139-153, decoder.py:34-46
//   classify_bin      decoder.py:127-169 + driver.py:166-176 (bin guard)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fpssft {

constexpr int MAXD = 4;

// Debug builds (-DFPSSFT_DEBUG_BOUNDS=1, tools/bounds_check.sh): every
// shared-memory scatter / slot / hash index is checked and a violation traps
// (the GPU pool has no compute-sanitizer).  Compiled out otherwise.
#ifndef FPSSFT_DEBUG_BOUNDS
#define FPSSFT_DEBUG_BOUNDS 0
#endif
#if FPSSFT_DEBUG_BOUNDS
#define FPSSFT_CHECK(cond)                                                                    \
    do {                                                                                      \
        if (!(cond)) {                                                                        \
            printf("FPSSFT_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, \
                   #cond, (int)blockIdx.x, (int)threadIdx.x);                                \
            __trap();                                                                         \
        }                                                                                     \
    } while (0)
#else
#define FPSSFT_CHECK(cond) do {} while (0)
#endif
#ifndef FPSSFT_R16_256
#define FPSSFT_R16_256 1  // 256-point lines: radix 16x16 (1) or 8x8x4 (0)
#endif
constexpr int MAXSTAGES = 16;
constexpr unsigned FULL = 0xffffffffu;

// ----------------------------------------------------------------- complex
template <class R>
struct cpx {
    R re, im;
};
template <class R>
__device__ __forceinline__ cpx<R> operator+(cpx<R> a, cpx<R> b) { return {a.re + b.re, a.im + b.im}; }
template <class R>
__device__ __forceinline__ cpx<R> operator-(cpx<R> a, cpx<R> b) { return {a.re - b.re, a.im - b.im}; }
template <class R>
__device__ __forceinline__ cpx<R> operator*(cpx<R> a, cpx<R> b) {
    return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
// a * conj(b)
template <class R>
__device__ __forceinline__ cpx<R> mulc(cpx<R> a, cpx<R> b) {
    return {a.re * b.re + a.im * b.im, a.im * b.re - a.re * b.im};
}
// |z|: hypot in float64 (what np.abs computes); sqrt(x^2 + y^2) in float32,
// whose inputs never approach overflow here.  (FPSSFT_CABS_HYPOT=0: the
// float64 sqrt form, A/B only -- mixed, within +-4 %.)
#ifndef FPSSFT_CABS_HYPOT
#define FPSSFT_CABS_HYPOT 1
#endif
template <class R>
__device__ __forceinline__ R cabs(cpx<R> a) {
    if constexpr (FPSSFT_CABS_HYPOT) return hypot(a.re, a.im);
    else return sqrt(fma(a.re, a.re, a.im * a.im));
}
__device__ __forceinline__ float cabs(cpx<float> a) { return sqrtf(a.re * a.re + a.im * a.im); }
template <class R>
__device__ __forceinline__ R cabs2(cpx<R> a) { return a.re * a.re + a.im * a.im; }

// Padded spectra layout of the compile-time warp kernels: one spare complex
// after every 16, so the stride-16 writes of a radix-16 Stockham stage (and
// the stride-L line accesses) spread over the shared-memory banks.
template <bool PAD>
__device__ __forceinline__ int padi(int e) { return PAD ? e + (e >> 4) : e; }

// Synchronisation of the threads that own one instance: the whole CTA, or
// one warp (team of 32 lanes).
struct BlockTeam {
    __device__ __forceinline__ static void sync() { __syncthreads(); }
};
struct WarpTeam {
    __device__ __forceinline__ static void sync() { __syncwarp(); }
};

// ---------------------------------------------------------------- geometry
// CubeShape (core.py:26-73) as the kernels see it.
struct Geo {
    int D, L, nlines;               // nlines = D + 1
    int N[MAXD];                    // extents
    int cof[MAXD];                  // c_k = L / N_k
    long long stride[MAXD];         // element strides of one cube
    int stride32[MAXD];             // the same as int32 when off32
    int off32;                      // every element offset of a cube fits int32
    unsigned long long magic[MAXD]; // fastmod multipliers for N_k
    int nstages;                    // FFT plan, 16 bits per stage s in plan[s/4] >> 16(s%4):
    unsigned long long plan[4];     //   bits 0-4 radix {2,3,4,5,7,8,16} (0 = direct O(L^2)),
                                    //   bits 5-7 butterflies per thread {1,2,4},
                                    //   bits 8-15 lines transformed together (1..255)
    int threads;                    // threads per instance the plan was made for
    int key_shift[MAXD];            // packed frequency key: m_k << key_shift[k]
    int key_mask[MAXD];             //   (lexicographic order = key order)
    int key_bits_;                  // total bits of the packed key
};
__host__ __device__ __forceinline__ int stage_code(const Geo &g, int s) {
    const int q = s >> 2;  // selects, not dynamic indexing, keep g in registers
    const unsigned long long w = q == 0 ? g.plan[0] : q == 1 ? g.plan[1] : q == 2 ? g.plan[2]
                                                                              : g.plan[3];
    return (int)((w >> (16 * (s & 3))) & 0xFFFFULL);
}

// Tolerances / knobs (FpsSftConfig, driver.py:29-63).
struct Knobs {
    double mag_tol, verify_tol, round_tol, amp_prune_tol;
    double energy_floor, energy_floor_abs, residual_stop;
    double noise_coef;  // float32 rounding floor: coef * sqrt(sum |x|^2 over the D+1 lines)
    double guard_coef;  // guarded float32: transform error bound coef * sqrt(sum |x|^2)
    int t_max, stall_limit, k_cap;
    int group;  // instances interleaved per sample (batch layout [B/group, *dims, group])
    // staged lines (fpssft_stage.cuh): iterations t < stage_T of a group read
    // their line samples from staged[group][t][line][l][group] instead of the cube
    const float2 *staged;
    long long staged_group_stride;
    int stage_T;
};

// Base of instance `inst`'s cube: batch layout [B/G, *dims, G] (G = kn.group
// instances interleaved sample by sample; G = 1 is the plain [B, *dims]).
template <class T>
__device__ __forceinline__ const T *cube_base(const T *cubes, long long inst,
                                              long long group_stride, int group) {
    if (group == 1) return cubes + inst * group_stride;
    return cubes + (inst / group) * group_stride + (inst % group);
}

// v mod n for v in [-n, 2n) without division: the rounded phase ratio
// rint(N angle / 2 pi) lies in [-N/2, N/2] (decoder.py:153-158).
__device__ __forceinline__ int wrap_index(int v, int n) {
    v = v < 0 ? v + n : v;
    return v >= n ? v - n : v;
}

// a mod d without division (Lemire): valid for any 32-bit a, d >= 1.
__device__ __forceinline__ unsigned fastmod(unsigned a, unsigned long long M, unsigned d) {
    return (unsigned)__umul64hi(M * (unsigned long long)a, (unsigned long long)d);
}

// ----------------------------------------------------- block primitives
// blockDim.x is a multiple of 32, <= 1024.  Reductions combine the per-warp
// partials in a fixed order, so results are bit-deterministic for a given
// block size.
template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}
template <class T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
    return v;
}
template <class T>
__device__ __forceinline__ T block_sum(T v, T *red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    T r = red[0];
    for (int i = 1; i < nw; ++i) r += red[i];
    return r;
}
template <class T>
__device__ __forceinline__ T block_max(T v, T *red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    T r = red[0];
    for (int i = 1; i < nw; ++i) r = max(r, red[i]);
    return r;
}
// exclusive scan of one int per thread, in thread order; *total = sum.
__device__ __forceinline__ int block_exscan(int v, int *red, int *total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) red[w] = x;
    __syncthreads();
    int off = 0, tot = 0;
    for (int i = 0; i < nw; ++i) {
        int s = red[i];
        off += (i < w) ? s : 0;
        tot += s;
    }
    *total = tot;
    return off + x - v;
}

// ------------------------------------------------------------ root table
// roots[j] = exp(+2 pi i j / L), evaluated in double (sincospi) and rounded
// once to R: the exact integer-phase table of decoder.py:34-38/core.py:195.
template <class R>
__device__ __forceinline__ void build_roots(cpx<R> *roots, int L) {
    for (int j = threadIdx.x; j < L; j += blockDim.x) {
        double s, c;
        sincospi(2.0 * (double)j / (double)L, &s, &c);
        roots[j] = {(R)c, (R)s};
    }
}

// float64 roots as a float32 pair: hi = the float32 table (build_roots),
// lo = float32(root - hi); hi + lo carries ~2^-49 relative error, against
// 2^-53 for a float64 table, at half its shared memory.
struct Roots64Split {
    const cpx<float> *hi, *lo;
    __device__ __forceinline__ cpx<double> operator[](int j) const {
        const cpx<float> h = hi[j], l = lo[j];
        return {(double)h.re + (double)l.re, (double)h.im + (double)l.im};
    }
};
// A float64 table e^{+2 pi i j / L} (one 16-byte load per root).
struct Roots64Full {
    const cpx<double> *t;
    __device__ __forceinline__ cpx<double> operator[](int j) const { return t[j]; }
};
__device__ __forceinline__ void build_roots64(cpx<double> *t, int L) {
    for (int j = threadIdx.x; j < L; j += blockDim.x) {
        double s, c;
        sincospi(2.0 * (double)j / (double)L, &s, &c);
        t[j] = {c, s};
    }
}
__device__ __forceinline__ void build_roots_lo(cpx<float> *lo, int L) {
    for (int j = threadIdx.x; j < L; j += blockDim.x) {
        double s, c;
        sincospi(2.0 * (double)j / (double)L, &s, &c);
        lo[j] = {(float)(c - (double)(float)c), (float)(s - (double)(float)s)};
    }
}

// ------------------------------------------------------------------ gather
// Line samples x[(alpha*l + tau) mod N] for the D+1 offsets tau, tau+e_k
// (lines.py:36-64).  Row l of offset k+1 differs from offset 0 only in
// coordinate k, advanced by one with wrap, so each thread issues its D+1
// loads from one base address.  Index math is fastmod, no division.
// Returns this thread's share of sum |x|^2 over the gathered samples.
template <class R, bool PAD = false>
__device__ __forceinline__ R gather_lines(cpx<R> *spec, const float2 *__restrict__ cube,
                                          const Geo &g, const int *al, const int *ta, int tid,
                                          int nth) {
    const int L = g.L, D = g.D;
    R energy = (R)0;
    for (int l = tid; l < L; l += nth) {
        long long base = 0;
        long long delta[MAXD];
#pragma unroll
        for (int k = 0; k < MAXD; ++k) {
            if (k < D) {
                unsigned n = fastmod((unsigned)al[k] * (unsigned)l + (unsigned)ta[k], g.magic[k],
                                     (unsigned)g.N[k]);
                base += (long long)n * g.stride[k];
                delta[k] = (n + 1 == (unsigned)g.N[k]) ? -(long long)n * g.stride[k] : g.stride[k];
            }
        }
        float2 v[MAXD + 1];
        v[0] = __ldcs(cube + base);
#pragma unroll
        for (int k = 0; k < MAXD; ++k)
            if (k < D) v[k + 1] = __ldcs(cube + base + delta[k]);
        spec[padi<PAD>(l)] = {(R)v[0].x, (R)v[0].y};
        energy += (R)v[0].x * (R)v[0].x + (R)v[0].y * (R)v[0].y;
#pragma unroll
        for (int k = 0; k < MAXD; ++k)
            if (k < D) {
                spec[padi<PAD>((k + 1) * L + l)] = {(R)v[k + 1].x, (R)v[k + 1].y};
                energy += (R)v[k + 1].x * (R)v[k + 1].x + (R)v[k + 1].y * (R)v[k + 1].y;
            }
    }
    return energy;
}

// float32 path: the gather as asynchronous 8-byte global->shared copies
// (cp.async, LDGSTS): every sample of every line of an iteration is in flight
// at once, no registers held, so one warp per instance still has its whole
// line set outstanding against DRAM.  Caller: cp_async_wait_all(), team sync,
// then line_energy() if the rounding floor is needed.
#ifndef FPSSFT_GATHER_L2_64B
#define FPSSFT_GATHER_L2_64B 1
#endif
__device__ __forceinline__ void cp_async8(void *smem_dst, const void *gsrc) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
#if FPSSFT_GATHER_L2_64B
    // .L2::64B: an L2 miss fetches 64 B instead of a 128-byte line
    // (tools/gather_probe.cu: half the DRAM bytes, ~14% more random loads/s)
    asm volatile("cp.async.ca.shared.global.L2::64B [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc)
                 : "memory");
#else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc) : "memory");
#endif
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
}
template <int LC = 0, int NTC = 32>
__device__ __forceinline__ void gather_lines_async(cpx<float> *spec,
                                                   const float2 *__restrict__ cube, const Geo &g,
                                                   const int *al, const int *ta, int tid,
                                                   int nth) {
    const int L = g.L, D = g.D;
    if (LC && g.off32) {  // compile-time line length, one warp: fixed trip count
        int n[MAXD], step[MAXD];
#pragma unroll
        for (int k = 0; k < MAXD; ++k) {
            n[k] = k < D ? (int)fastmod((unsigned)al[k] * (unsigned)tid + (unsigned)ta[k],
                                        g.magic[k], (unsigned)g.N[k])
                         : 0;
            step[k] = k < D ? (int)fastmod((unsigned)al[k] * (unsigned)NTC, g.magic[k],
                                           (unsigned)g.N[k])
                            : 0;
        }
#pragma unroll 4
        for (int j = 0; j < (LC + NTC - 1) / NTC; ++j) {
            const int l = tid + NTC * j;
            if (LC % NTC != 0 && l >= LC) break;
            int base = 0;
#pragma unroll
            for (int k = 0; k < MAXD; ++k)
                if (k < D) base += n[k] * g.stride32[k];
            cp_async8(spec + padi<true>(l), cube + base);
#pragma unroll
            for (int k = 0; k < MAXD; ++k) {
                if (k < D) {
                    const int d = (n[k] + 1 == g.N[k]) ? -n[k] * g.stride32[k] : g.stride32[k];
                    cp_async8(spec + padi<true>((k + 1) * LC + l), cube + (base + d));
                    n[k] += step[k];
                    if (n[k] >= g.N[k]) n[k] -= g.N[k];
                }
            }
        }
        return;
    }
    if (g.off32) {
        // n_k(l) advanced incrementally by alpha_k * nth mod N_k: no division,
        // 32-bit offsets
        int n[MAXD], step[MAXD];
#pragma unroll
        for (int k = 0; k < MAXD; ++k) {
            n[k] = k < D ? (int)fastmod((unsigned)al[k] * (unsigned)tid + (unsigned)ta[k],
                                        g.magic[k], (unsigned)g.N[k])
                         : 0;
            step[k] = k < D ? (int)fastmod((unsigned)al[k] * (unsigned)nth, g.magic[k],
                                           (unsigned)g.N[k])
                            : 0;
        }
        for (int l = tid; l < L; l += nth) {
            int base = 0;
#pragma unroll
            for (int k = 0; k < MAXD; ++k)
                if (k < D) base += n[k] * g.stride32[k];
            cp_async8(spec + l, cube + base);
#pragma unroll
            for (int k = 0; k < MAXD; ++k) {
                if (k < D) {
                    const int d = (n[k] + 1 == g.N[k]) ? -n[k] * g.stride32[k] : g.stride32[k];
                    cp_async8(spec + (k + 1) * L + l, cube + (base + d));
                    n[k] += step[k];
                    if (n[k] >= g.N[k]) n[k] -= g.N[k];
                }
            }
        }
        return;
    }
    for (int l = tid; l < L; l += nth) {
        long long base = 0;
        long long delta[MAXD];
#pragma unroll
        for (int k = 0; k < MAXD; ++k) {
            if (k < D) {
                unsigned n = fastmod((unsigned)al[k] * (unsigned)l + (unsigned)ta[k], g.magic[k],
                                     (unsigned)g.N[k]);
                base += (long long)n * g.stride[k];
                delta[k] = (n + 1 == (unsigned)g.N[k]) ? -(long long)n * g.stride[k] : g.stride[k];
            }
        }
        cp_async8(spec + l, cube + base);
#pragma unroll
        for (int k = 0; k < MAXD; ++k)
            if (k < D) cp_async8(spec + (k + 1) * L + l, cube + base + delta[k]);
    }
}
// Register gather for compile-time shapes (LC, DC, NTC threads): batches of
// up to 24 samples per thread are all in flight before the first shared
// store.  ld.global.nc.L1::no_allocate keeps the random lines out of L1 --
// cp.async.ca stages every sample through an L1 line, and with most of the
// SM's 256 KB carved out as shared memory those in-flight lines back up the
// load pipe.
#ifndef FPSSFT_GATHER_NC
#define FPSSFT_GATHER_NC 1
#endif
__device__ __forceinline__ float2 ld_nc8(const float2 *p) {
    float2 v;
#if FPSSFT_GATHER_L2_64B
    asm("ld.global.nc.L1::no_allocate.L2::64B.v2.f32 {%0, %1}, [%2];"
        : "=f"(v.x), "=f"(v.y) : "l"(p));
#else
    asm("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
#endif
    return v;
}
template <int LC, int DC, int NTC = 32>
__device__ __forceinline__ void gather_lines_nc(cpx<float> *spec, const float2 *__restrict__ cube,
                                                const Geo &g, const int *al, const int *ta,
                                                int tid) {
    constexpr int NL = DC + 1, J = (LC + NTC - 1) / NTC;
    constexpr int JB = 24 / NL < J ? 24 / NL : J;
    int n[DC], step[DC];
#pragma unroll
    for (int k = 0; k < DC; ++k) {
        n[k] = (int)fastmod((unsigned)al[k] * (unsigned)tid + (unsigned)ta[k], g.magic[k],
                            (unsigned)g.N[k]);
        step[k] = (int)fastmod((unsigned)al[k] * (unsigned)NTC, g.magic[k], (unsigned)g.N[k]);
    }
#pragma unroll
    for (int j0 = 0; j0 < J; j0 += JB) {
        float2 v[JB][NL];
#pragma unroll
        for (int jj = 0; jj < JB; ++jj) {
            const int l = tid + NTC * (j0 + jj);
            if (j0 + jj < J && (LC % NTC == 0 || l < LC)) {
                int base = 0;
#pragma unroll
                for (int k = 0; k < DC; ++k) base += n[k] * g.stride32[k];
                v[jj][0] = ld_nc8(cube + base);
#pragma unroll
                for (int k = 0; k < DC; ++k) {
                    // tau + e_k: the next index along axis k, wrapping
                    const int d = (n[k] + 1 == g.N[k]) ? -n[k] * g.stride32[k] : g.stride32[k];
                    v[jj][k + 1] = ld_nc8(cube + (base + d));
                    n[k] += step[k];
                    if (n[k] >= g.N[k]) n[k] -= g.N[k];
                }
            }
        }
#pragma unroll
        for (int jj = 0; jj < JB; ++jj) {
            const int l = tid + NTC * (j0 + jj);
            if (j0 + jj < J && (LC % NTC == 0 || l < LC)) {
#pragma unroll
                for (int i = 0; i < NL; ++i) spec[padi<true>(i * LC + l)] = {v[jj][i].x, v[jj][i].y};
            }
        }
    }
}
// 16-byte gather that bypasses L1 (compile-time shapes, one warp): each
// sample is fetched as the aligned 16-byte chunk holding it with
// cp.async.cg into a 16-byte staging slot; bit t of the returned mask says
// which half is the sample (t = line * LC/32 + j for l = lane + 32 j).  The
// cp.async.ca 8-byte form stages every in-flight sample in an L1 line, and L1
// is what the shared-memory carveout leaves (92 KB at config 2's 162 KB of
// shared memory per SM), which caps the misses in flight.
#ifndef FPSSFT_GATHER_CG
#define FPSSFT_GATHER_CG 1
#endif
// Staging applies to float spectra with compile-time shapes whose NL x J
// samples per thread fit one 32-bit mask (J = L / nt samples per line).
#ifndef FPSSFT_STAGE16_TEAM
#define FPSSFT_STAGE16_TEAM 1
#endif
#ifndef FPSSFT_STAGE16_W64
#define FPSSFT_STAGE16_W64 1
#endif
__host__ __device__ constexpr bool stage16_ok(int D, int L, int cs, int nt) {
    return FPSSFT_GATHER_CG && cs == 8 && D >= 2 && L % nt == 0 && (D + 1) * (L / nt) <= 32 &&
           (nt == 32 ? ((L == 256 && D == 2) || (FPSSFT_STAGE16_W64 && L == 64 && D == 3))
                      : FPSSFT_STAGE16_TEAM != 0);
}
__device__ __forceinline__ void cp_async16_cg(void *smem_dst, const void *gsrc) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global.L2::64B [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ unsigned stage16(float4 *dst, const float2 *src, int bit) {
    const unsigned long long a = (unsigned long long)src;
    cp_async16_cg(dst, (const void *)(a & ~15ull));
    return (unsigned)((a >> 3) & 1ull) << bit;
}
// Thread tid stages l = tid + NTC j of every line into slot line * LC + l;
// returns the half-select mask (bit line * J + j) and in *dup the samples of
// the last-axis line (unit stride, no wrap) that sit in the upper half of
// tau's own chunk and so need no request of their own.
template <int LC, int DC, int NTC = 32>
__device__ __forceinline__ unsigned gather_lines_cg16(float4 *stage, const float2 *__restrict__ cube,
                                                      const Geo &g, const int *al, const int *ta,
                                                      int tid, unsigned *dup) {
    constexpr int J = LC / NTC;
    static_assert(LC % NTC == 0 && (DC + 1) * J <= 32, "one mask bit per staged sample");
    int n[DC], step[DC];
#pragma unroll
    for (int k = 0; k < DC; ++k) {
        n[k] = (int)fastmod((unsigned)al[k] * (unsigned)tid + (unsigned)ta[k], g.magic[k],
                            (unsigned)g.N[k]);
        step[k] = (int)fastmod((unsigned)al[k] * (unsigned)NTC, g.magic[k], (unsigned)g.N[k]);
    }
    unsigned par = 0, dp = 0;
    const bool unit_last = g.stride32[DC - 1] == 1;
#pragma unroll 4
    for (int j = 0; j < J; ++j) {
        const int l = tid + NTC * j;
        int base = 0;
#pragma unroll
        for (int k = 0; k < DC; ++k) base += n[k] * g.stride32[k];
        const unsigned p0 = stage16(stage + l, cube + base, j);
        par |= p0;
#pragma unroll
        for (int k = 0; k < DC; ++k) {
            const bool wrap = n[k] + 1 == g.N[k];
            const int d = wrap ? -n[k] * g.stride32[k] : g.stride32[k];
            if (k == DC - 1 && unit_last && !wrap && p0 == 0u)
                dp |= 1u << j;  // tau + e_last: the upper half of tau's chunk
            else
                par |= stage16(stage + (k + 1) * LC + l, cube + (base + d), (k + 1) * J + j);
            n[k] += step[k];
            if (n[k] >= g.N[k]) n[k] -= g.N[k];
        }
    }
    *dup = dp;
    return par;
}
// Staging slots -> padded spectra, in place (the spectra start at the
// staging base), one line per batch.  Sample f = NTC t + tid moves from
// 16-byte slot f (staged by this same thread) to complex padi(f), byte
// ~8.5 f: inside slots < 0.54 f, all read by the end of f's batch -- so one
// team barrier per batch, between its reads and its writes.  Last-axis
// samples flagged in dup are carried in registers from the line-0 batch.
template <int LC, int NL, int NTC, class Team>
__device__ __forceinline__ void compact_stage16(cpx<float> *spec, unsigned par, unsigned dup,
                                                int tid, cpx<double> *x0d = nullptr) {
    constexpr int J = LC / NTC;
    const float4 *stage = (const float4 *)spec;
    float2 hold[J];
#pragma unroll
    for (int i = 0; i < NL; ++i) {
        float2 v[J];
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int t = i * J + j;
            if (i == NL - 1 && ((dup >> j) & 1u)) {
                v[j] = hold[j];
            } else {
                const float4 q = stage[NTC * t + tid];
                v[j] = ((par >> t) & 1u) ? make_float2(q.z, q.w) : make_float2(q.x, q.y);
                if (i == 0) hold[j] = make_float2(q.z, q.w);
            }
        }
        Team::sync();
#pragma unroll
        for (int j = 0; j < J; ++j) spec[padi<true>(NTC * (i * J + j) + tid)] = {v[j].x, v[j].y};
        if (i == 0 && x0d != nullptr)  // guarded mode: line 0 also in float64
#pragma unroll
            for (int j = 0; j < J; ++j) x0d[padi<true>(NTC * j + tid)] = {(double)v[j].x, (double)v[j].y};
    }
}
// Group gather (interleaved batch layout [B/G, *dims, G]): the WG warps of a
// CTA own WG consecutive members of one interleave group, which share the
// schedule, so at every sample position their WG samples are contiguous
// (WG * 8 bytes) and are fetched once for all of them -- as 16-byte chunks,
// one thread per chunk, with L1-bypassing register loads -- and scattered
// into the owners' padded spectra.  Thread tid takes chunk c = tid % CH
// (members 2c, 2c + 1) of positions q = tid / CH + QS j (q = line * LC + l).
// The index arithmetic of a position is done once per group, not once per
// instance, and no 16-byte staging area is needed.
__device__ __forceinline__ float4 ld_nc16(const float2 *p) {
    float4 v;
    asm("ld.global.nc.L1::no_allocate.L2::64B.v4.f32 {%0, %1, %2, %3}, [%4];"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
template <int LC, int DC, int WG>
struct GroupGather {
    static constexpr int NL = DC + 1, CH = WG / 2, NTH = WG * 32, QS = NTH / CH;
    static constexpr int PPT = NL * LC * CH / NTH;  // chunks per thread
    static constexpr int LQ = LC / QS;              // distinct l per thread
    static_assert(WG % 2 == 0 && LC % QS == 0 && PPT * NTH == NL * LC * CH,
                  "group gather: whole lines per thread");
    float4 v[PPT];
    // gbase: the CTA's first member's sample 0 (group block + member0);
    // strides include the factor G of the interleaved layout
    __device__ __forceinline__ void load(const float2 *__restrict__ gbase, const Geo &g,
                                         const int *al, const int *ta, int tid) {
        const int c = tid % CH, q0 = tid / CH;
        int n[LQ][DC];
#pragma unroll
        for (int j = 0; j < LQ; ++j)
#pragma unroll
            for (int k = 0; k < DC; ++k)
                n[j][k] = (int)fastmod((unsigned)al[k] * (unsigned)(q0 + QS * j) + (unsigned)ta[k],
                                       g.magic[k], (unsigned)g.N[k]);
#pragma unroll
        for (int i = 0; i < NL; ++i) {
#pragma unroll
            for (int j = 0; j < LQ; ++j) {
                int off = 0;
#pragma unroll
                for (int k = 0; k < DC; ++k) {
                    int nk = n[j][k];
                    if (k == i - 1) nk = nk + 1 == g.N[k] ? 0 : nk + 1;  // tau + e_k
                    off += nk * g.stride32[k];
                }
                v[i * LQ + j] = ld_nc16(gbase + off + 2 * c);
            }
        }
    }
    // iteration `it` from the staging buffer (fpssft_stage.cuh): sbase = the
    // team's first member in staged[group], positions in line order, G
    // instances per position
    __device__ __forceinline__ void load_staged(const float2 *__restrict__ sbase, int it, int G,
                                                int tid) {
        const int c = tid % CH, q0 = tid / CH;
        const float2 *p = sbase + ((long long)it * (NL * LC) + q0) * G + 2 * c;
#pragma unroll
        for (int t = 0; t < PPT; ++t) v[t] = ld_nc16(p + (long long)(QS * t) * G);
    }
    // the same segments into L2 only (one request per 64-byte segment: the
    // thread that loads the segment's first chunk)
    __device__ __forceinline__ void prefetch_l2(const float2 *__restrict__ gbase, const Geo &g,
                                                const int *al, const int *ta, int tid) const {
        const int c = tid % CH, q0 = tid / CH;
        if (c != 0) return;
        int n[LQ][DC];
#pragma unroll
        for (int j = 0; j < LQ; ++j)
#pragma unroll
            for (int k = 0; k < DC; ++k)
                n[j][k] = (int)fastmod((unsigned)al[k] * (unsigned)(q0 + QS * j) + (unsigned)ta[k],
                                       g.magic[k], (unsigned)g.N[k]);
#pragma unroll
        for (int i = 0; i < NL; ++i) {
#pragma unroll
            for (int j = 0; j < LQ; ++j) {
                int off = 0;
#pragma unroll
                for (int k = 0; k < DC; ++k) {
                    int nk = n[j][k];
                    if (k == i - 1) nk = nk + 1 == g.N[k] ? 0 : nk + 1;
                    off += nk * g.stride32[k];
                }
                asm volatile("prefetch.global.L2 [%0];" ::"l"(gbase + off));
            }
        }
    }
    // owner spectra: warp w's at spec0 + w * warp_stride (complex units)
    __device__ __forceinline__ void store(cpx<float> *spec0, int warp_stride, int tid) const {
        const int c = tid % CH, q0 = tid / CH;
        cpx<float> *a = spec0 + (2 * c) * warp_stride, *b = a + warp_stride;
#pragma unroll
        for (int t = 0; t < PPT; ++t) {
            const int q = q0 + QS * t;  // position t: line t / LQ, l = q0 + QS (t % LQ)
            const int e = padi<true>(q);
            a[e] = {v[t].x, v[t].y};
            b[e] = {v[t].z, v[t].w};
        }
    }
};

// L2 prefetch of a future iteration's line samples (compile-time line
// length, one warp): the same addresses as gather_lines_async, no data moved
// on chip.
template <int LC, int NTC = 32>
__device__ __forceinline__ void prefetch_lines_l2(const float2 *__restrict__ cube, const Geo &g,
                                                  const int *al, const int *ta, int tid) {
    const int D = g.D;
    int n[MAXD], step[MAXD];
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
        n[k] = k < D ? (int)fastmod((unsigned)al[k] * (unsigned)tid + (unsigned)ta[k], g.magic[k],
                                    (unsigned)g.N[k])
                     : 0;
        step[k] = k < D ? (int)fastmod((unsigned)al[k] * (unsigned)NTC, g.magic[k],
                                       (unsigned)g.N[k])
                        : 0;
    }
#pragma unroll 4
    for (int j = 0; j < (LC + NTC - 1) / NTC; ++j) {
        if (LC % NTC != 0 && tid + NTC * j >= LC) break;
        int base = 0;
#pragma unroll
        for (int k = 0; k < MAXD; ++k)
            if (k < D) base += n[k] * g.stride32[k];
        asm volatile("prefetch.global.L2 [%0];" ::"l"(cube + base));
#pragma unroll
        for (int k = 0; k < MAXD; ++k) {
            if (k < D) {
                // tau + e_k shares a line with tau unless it is a different row
                if (k < D - 1) {
                    const int d = (n[k] + 1 == g.N[k]) ? -n[k] * g.stride32[k] : g.stride32[k];
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(cube + (base + d)));
                }
                n[k] += step[k];
                if (n[k] >= g.N[k]) n[k] -= g.N[k];
            }
        }
    }
}

template <class R>
__device__ __forceinline__ R line_energy(const cpx<R> *spec, int n, int tid, int nth) {
    R e = (R)0;
    for (int i = tid; i < n; i += nth) e += spec[i].re * spec[i].re + spec[i].im * spec[i].im;
    return e;
}

// ------------------------------------------------------------------- FFT
// Self-sorting (Stockham) mixed-radix DIT FFT on `nlines` contiguous lines of
// length L held in shared memory, in place: each stage pulls its butterflies
// into registers, barriers, and stores.  Twiddles come from the root table
// (exact integer phase indices).  The last stage divides by L
// (dft_forward = fft(s)/L, transform.py:22).
template <class R, int RAD>
struct Bfly {
    // generic odd radix: y_q = sum_j v_j * conj(root[(j*q mod RAD) * L/RAD])
    static __device__ __forceinline__ void run(cpx<R> *v, const cpx<R> *roots, int L) {
        const int s = L / RAD;
        cpx<R> y[RAD];
#pragma unroll
        for (int q = 0; q < RAD; ++q) {
            cpx<R> acc = v[0];
#pragma unroll
            for (int j = 1; j < RAD; ++j) acc = acc + mulc(v[j], roots[((j * q) % RAD) * s]);
            y[q] = acc;
        }
#pragma unroll
        for (int q = 0; q < RAD; ++q) v[q] = y[q];
    }
};
template <class R>
struct Bfly<R, 2> {
    static __device__ __forceinline__ void run(cpx<R> *v, const cpx<R> *, int) {
        cpx<R> a = v[0], b = v[1];
        v[0] = a + b;
        v[1] = a - b;
    }
};
template <class R>
__device__ __forceinline__ void dft4(cpx<R> &a0, cpx<R> &a1, cpx<R> &a2, cpx<R> &a3) {
    cpx<R> t0 = a0 + a2, t1 = a0 - a2, t2 = a1 + a3, d = a1 - a3;
    cpx<R> t3 = {d.im, -d.re};  // -i * (a1 - a3)
    a0 = t0 + t2;
    a2 = t0 - t2;
    a1 = t1 + t3;
    a3 = t1 - t3;
}
template <class R>
struct Bfly<R, 4> {
    static __device__ __forceinline__ void run(cpx<R> *v, const cpx<R> *, int) {
        dft4(v[0], v[1], v[2], v[3]);
    }
};
template <class R>
struct Bfly<R, 8> {
    static __device__ __forceinline__ void run(cpx<R> *v, const cpx<R> *, int) {
        const R c = (R)0.70710678118654752440;
        cpx<R> e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
        cpx<R> o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
        dft4(e0, e1, e2, e3);
        dft4(o0, o1, o2, o3);
        cpx<R> w1 = {c * (o1.re + o1.im), c * (o1.im - o1.re)};  // e^{-i pi/4} o1
        cpx<R> w2 = {o2.im, -o2.re};                            // -i o2
        cpx<R> w3 = {c * (o3.im - o3.re), -c * (o3.re + o3.im)}; // e^{-3i pi/4} o3
        v[0] = e0 + o0;
        v[4] = e0 - o0;
        v[1] = e1 + w1;
        v[5] = e1 - w1;
        v[2] = e2 + w2;
        v[6] = e2 - w2;
        v[3] = e3 + w3;
        v[7] = e3 - w3;
    }
};

template <class R>
struct Bfly<R, 16> {
    // 4 x 4: DFT4 over n1 of x[4 n1 + n2], twiddle W16^(n2 k1), DFT4 over n2.
    static __device__ __forceinline__ void run(cpx<R> *v, const cpx<R> *, int) {
        const R c1 = (R)0.92387953251128675613, s1 = (R)0.38268343236508977173;
        const R h = (R)0.70710678118654752440;
        cpx<R> a[4][4];
#pragma unroll
        for (int n2 = 0; n2 < 4; ++n2) {
#pragma unroll
            for (int n1 = 0; n1 < 4; ++n1) a[n2][n1] = v[4 * n1 + n2];
            dft4(a[n2][0], a[n2][1], a[n2][2], a[n2][3]);
        }
        // W16^p = (cos(2 pi p/16), -sin(2 pi p/16)) for p = n2 * k1
        const cpx<R> w[10] = {{(R)1, (R)0}, {c1, -s1}, {h, -h},   {s1, -c1}, {(R)0, (R)-1},
                              {-s1, -c1},   {-h, -h}, {-c1, -s1}, {(R)-1, (R)0}, {-c1, s1}};
#pragma unroll
        for (int n2 = 1; n2 < 4; ++n2)
#pragma unroll
            for (int k1 = 1; k1 < 4; ++k1) a[n2][k1] = a[n2][k1] * w[n2 * k1];
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) {
            dft4(a[0][k1], a[1][k1], a[2][k1], a[3][k1]);
#pragma unroll
            for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = a[k2][k1];
        }
    }
};

// One Stockham stage: butterfly q (of G*L/RAD for a group of G lines) reads
// x[line][j + k L/RAD], twiddles by W_{Ns RAD}^{(j mod Ns) k}, and writes
// x[line][(j - j mod Ns) RAD + j mod Ns + k Ns].  Each of the team's `nth`
// threads owns up to MB butterflies of a group; lines are processed G at a
// time so that a group's butterflies fit the team's registers.
template <class R, int RAD, int MB, class Team>
__device__ __forceinline__ void fft_stage(cpx<R> *x, int nlines, int G, int L, int Ns,
                                          const cpx<R> *roots, bool last, int tid, int nth) {
    const int m = L / RAD, step = L / (Ns * RAD);
    const R inv = (R)1 / (R)L;
    const bool pow2 = (L & (L - 1)) == 0;  // then x * (1/L) == x / L exactly
    for (int l0 = 0; l0 < nlines; l0 += G) {
        const int total = min(G, nlines - l0) * m;
        cpx<R> v[MB][RAD];
        int ob[MB];
#pragma unroll
        for (int j = 0; j < MB; ++j) {
            const int q = tid + j * nth;
            ob[j] = -1;
            if (q < total) {
                const int line = l0 + q / m, jj = q % m;
                const cpx<R> *xl = x + line * L;
#pragma unroll
                for (int k = 0; k < RAD; ++k) v[j][k] = xl[jj + k * m];
                const int jm = jj % Ns;
                if (jm) {
#pragma unroll
                    for (int k = 1; k < RAD; ++k) v[j][k] = mulc(v[j][k], roots[jm * k * step]);
                }
                Bfly<R, RAD>::run(v[j], roots, L);
                ob[j] = line * L + (jj - jm) * RAD + jm;
            }
        }
        Team::sync();
#pragma unroll
        for (int j = 0; j < MB; ++j) {
            if (ob[j] >= 0) {
#pragma unroll
                for (int k = 0; k < RAD; ++k) {
                    cpx<R> o = v[j][k];
                    if (last && pow2) o = {o.re * inv, o.im * inv};
                    x[ob[j] + k * Ns] = o;
                }
            }
        }
        Team::sync();
    }
}

// Direct O(L^2) pass for lengths with a prime factor > 7 (test-size L only).
template <class R, int MB, class Team>
__device__ __forceinline__ void dft_direct(cpx<R> *x, int nlines, int G, int L,
                                          const cpx<R> *roots, int tid, int nth) {
    const R fl = (R)L;
    for (int l0 = 0; l0 < nlines; l0 += G) {
        const int total = min(G, nlines - l0) * L;
        cpx<R> acc[MB];
#pragma unroll
        for (int j = 0; j < MB; ++j) {
            const int q = tid + j * nth;
            if (q < total) {
                const int line = l0 + q / L, k = q % L;
                const cpx<R> *xl = x + line * L;
                cpx<R> a = {(R)0, (R)0};
                int idx = 0;
                for (int l = 0; l < L; ++l) {
                    a = a + mulc(xl[l], roots[idx]);
                    idx += k;
                    if (idx >= L) idx -= L;
                }
                acc[j] = a;
            }
        }
        Team::sync();
#pragma unroll
        for (int j = 0; j < MB; ++j) {
            const int q = tid + j * nth;
            if (q < total) x[l0 * L + q] = {acc[j].re / fl, acc[j].im / fl};
        }
        Team::sync();
    }
}

// 1/L for lengths that are not powers of two, as a true division (what
// fft(s)/L computes); kept out of the butterfly code so the division's slow
// path does not force the butterfly registers to spill.
template <class R, class Team>
__device__ __noinline__ void divide_by_length(cpx<R> *x, int n, int L, int tid, int nth) {
    const R fl = (R)L;
    for (int i = tid; i < n; i += nth) x[i] = {x[i].re / fl, x[i].im / fl};
    Team::sync();
}

template <class R, int RAD, class Team>
__device__ __forceinline__ void fft_stage_mb(cpx<R> *x, int nlines, int G, int L, int Ns,
                                             int mb, const cpx<R> *roots, bool last, int tid,
                                             int nth) {
    // register budget (matches plan_fft's caps): complex values per thread
    // <= 16 (float) / 8 (double)
    constexpr int CAP = sizeof(R) == 4 ? (RAD <= 4 ? 4 : (RAD <= 8 ? 2 : 1))
                                       : (RAD <= 2 ? 4 : (RAD <= 4 ? 2 : 1));
    if (mb <= 1) fft_stage<R, RAD, 1, Team>(x, nlines, G, L, Ns, roots, last, tid, nth);
    else if (mb <= 2 || CAP < 4)
        fft_stage<R, RAD, (CAP < 2 ? 1 : 2), Team>(x, nlines, G, L, Ns, roots, last, tid, nth);
    else fft_stage<R, RAD, CAP, Team>(x, nlines, G, L, Ns, roots, last, tid, nth);
}

// Forward DFT (1/L normalised) of `nlines` contiguous lines per the plan in g.
template <class R, class Team>
__device__ __forceinline__ void fft_lines(cpx<R> *x, int nlines, const Geo &g,
                                          const cpx<R> *roots, int tid, int nth) {
    int Ns = 1;
    for (int s = 0; s < g.nstages; ++s) {
        const int code = stage_code(g, s);
        const int r = code & 31, mb = (code >> 5) & 7, G = max(1, (code >> 8) & 255);
        const bool last = (s == g.nstages - 1);
        switch (r) {
            case 16: fft_stage_mb<R, 16, Team>(x, nlines, G, g.L, Ns, mb, roots, last, tid, nth); break;
            case 8: fft_stage_mb<R, 8, Team>(x, nlines, G, g.L, Ns, mb, roots, last, tid, nth); break;
            case 4: fft_stage_mb<R, 4, Team>(x, nlines, G, g.L, Ns, mb, roots, last, tid, nth); break;
            case 2: fft_stage_mb<R, 2, Team>(x, nlines, G, g.L, Ns, mb, roots, last, tid, nth); break;
            case 3: fft_stage_mb<R, 3, Team>(x, nlines, G, g.L, Ns, mb, roots, last, tid, nth); break;
            case 5: fft_stage_mb<R, 5, Team>(x, nlines, G, g.L, Ns, mb, roots, last, tid, nth); break;
            case 7: fft_stage_mb<R, 7, Team>(x, nlines, G, g.L, Ns, mb, roots, last, tid, nth); break;
            default:
                if (mb <= 1) dft_direct<R, 1, Team>(x, nlines, G, g.L, roots, tid, nth);
                else if (mb <= 2) dft_direct<R, 2, Team>(x, nlines, G, g.L, roots, tid, nth);
                else dft_direct<R, 4, Team>(x, nlines, G, g.L, roots, tid, nth);
                break;
        }
        Ns *= (r > 0 ? r : g.L);
    }
    if (g.nstages == 0) Team::sync();  // L == 1: the DFT of one sample is itself
    const int r0 = stage_code(g, 0) & 31;
    if (g.nstages > 0 && r0 != 0 && (g.L & (g.L - 1)) != 0)
        divide_by_length<R, Team>(x, nlines * g.L, g.L, tid, nth);
}

// Warp-team FFT for power-of-two L: radices 8/4/2 only, each stage with its
// full register batch (guarded), which keeps the warp kernel's code small.
template <class R>
__device__ __forceinline__ void fft_lines_warp(cpx<R> *x, int nlines, const Geo &g,
                                               const cpx<R> *roots, int lane) {
    constexpr bool F = sizeof(R) == 4;
    int Ns = 1;
    for (int s = 0; s < g.nstages; ++s) {
        const int code = stage_code(g, s);
        const int r = code & 31, G = max(1, (code >> 8) & 255);
        const bool last = (s == g.nstages - 1);
        if (F && r == 16) fft_stage<R, 16, 1, WarpTeam>(x, nlines, G, g.L, Ns, roots, last, lane, 32);
        else if (r == 8) fft_stage<R, 8, F ? 2 : 1, WarpTeam>(x, nlines, G, g.L, Ns, roots, last, lane, 32);
        else if (r == 4) fft_stage<R, 4, F ? 4 : 2, WarpTeam>(x, nlines, G, g.L, Ns, roots, last, lane, 32);
        else fft_stage<R, 2, 4, WarpTeam>(x, nlines, G, g.L, Ns, roots, last, lane, 32);
        Ns *= r;
    }
    if (g.nstages == 0) __syncwarp();
}

// Compile-time FFT for the line lengths of the benchmark configs: every
// index, group and twiddle stride is a constant, so the stage loops fully
// unroll.  Team = one warp (NT = 32) or one CTA (NT = blockDim.x).  Stage:
// radix RAD after NS points have been combined; the spectra use the padded
// layout (padi).  The first stage (NS == 1) also returns this thread's share
// of sum |x|^2 over the raw samples it reads (each is read exactly once).
template <class R, int RAD>
struct StageCap {  // butterflies per thread that fit the register budget
    static constexpr int value = RAD == 16 ? 1 : (RAD == 8 ? 2 : 4);
};

template <class R, int L, int NL, int RAD, int NS, bool LAST, int NT, class Team,
          class RT = const cpx<R> *>
__device__ __forceinline__ R stage_static(cpx<R> *x, RT roots, int tid) {
    constexpr int M = L / RAD;                                   // butterflies per line
    constexpr int CAPB = StageCap<R, RAD>::value;
    constexpr int G0 = CAPB * NT / M;
    constexpr int G = G0 < 1 ? 1 : (G0 > NL ? NL : G0);          // lines per group
    constexpr int MB = (G * M + NT - 1) / NT;
    static_assert(MB <= CAPB, "stage does not fit the team's registers");
    constexpr int STEP = L / (NS * RAD);
    const R inv = (R)1 / (R)L;
    R energy = (R)0;
#pragma unroll
    for (int l0 = 0; l0 < NL; l0 += G) {
        const int total = (NL - l0 < G ? NL - l0 : G) * M;
        cpx<R> v[MB][RAD];
        int ob[MB];
#pragma unroll
        for (int j = 0; j < MB; ++j) {
            const int q = tid + NT * j;
            ob[j] = -1;
            if (q < total) {
                const int line = l0 + q / M, jj = q % M;
#pragma unroll
                for (int k = 0; k < RAD; ++k) v[j][k] = x[padi<true>(line * L + jj + k * M)];
                if (NS == 1) {
#pragma unroll
                    for (int k = 0; k < RAD; ++k) energy += cabs2(v[j][k]);
                }
                if (NS > 1) {
                    const int jm = jj % NS;
#pragma unroll
                    for (int k = 1; k < RAD; ++k) v[j][k] = mulc(v[j][k], roots[jm * k * STEP]);
                    ob[j] = line * L + (jj - jm) * RAD + jm;
                } else {
                    ob[j] = line * L + jj * RAD;
                }
                Bfly<R, RAD>::run(v[j], (const cpx<R> *)nullptr, L);  // radix 4/8/16: no table
            }
        }
        Team::sync();
#pragma unroll
        for (int j = 0; j < MB; ++j) {
            if (ob[j] >= 0) {
#pragma unroll
                for (int k = 0; k < RAD; ++k) {
                    cpx<R> o = v[j][k];
                    if (LAST) o = {o.re * inv, o.im * inv};  // L is a power of two: exact
                    x[padi<true>(ob[j] + k * NS)] = o;
                }
            }
        }
        Team::sync();
    }
    return energy;
}

template <int L>
struct HasStaticPlan {
    static constexpr bool value = L == 64 || L == 256 || L == 512 || L == 2048;
};

// Returns this thread's share of sum |x|^2 of the input samples.
template <class R, int L, int NL, int NT = 32, class Team = WarpTeam,
          class RT = const cpx<R> *>
__device__ __forceinline__ R fft_static(cpx<R> *x, RT roots, int tid) {
    constexpr bool F = sizeof(R) == 4;
    R e;
    if constexpr (L == 256 && F && FPSSFT_R16_256) {
        e = stage_static<R, L, NL, 16, 1, false, NT, Team, RT>(x, roots, tid);
        stage_static<R, L, NL, 16, 16, true, NT, Team, RT>(x, roots, tid);
    } else if constexpr (L == 256) {
        e = stage_static<R, L, NL, 8, 1, false, NT, Team, RT>(x, roots, tid);
        stage_static<R, L, NL, 8, 8, false, NT, Team, RT>(x, roots, tid);
        stage_static<R, L, NL, 4, 64, true, NT, Team, RT>(x, roots, tid);
    } else if constexpr (L == 512) {
        e = stage_static<R, L, NL, 8, 1, false, NT, Team, RT>(x, roots, tid);
        stage_static<R, L, NL, 8, 8, false, NT, Team, RT>(x, roots, tid);
        stage_static<R, L, NL, 8, 64, true, NT, Team, RT>(x, roots, tid);
    } else if constexpr (L == 64) {
        e = stage_static<R, L, NL, 8, 1, false, NT, Team, RT>(x, roots, tid);
        stage_static<R, L, NL, 8, 8, true, NT, Team, RT>(x, roots, tid);
    } else if constexpr (L == 2048 && F) {
        e = stage_static<R, L, NL, 16, 1, false, NT, Team, RT>(x, roots, tid);
        stage_static<R, L, NL, 16, 16, false, NT, Team, RT>(x, roots, tid);
        stage_static<R, L, NL, 8, 256, true, NT, Team, RT>(x, roots, tid);
    } else if constexpr (L == 2048) {
        e = stage_static<R, L, NL, 8, 1, false, NT, Team, RT>(x, roots, tid);
        stage_static<R, L, NL, 8, 8, false, NT, Team, RT>(x, roots, tid);
        stage_static<R, L, NL, 8, 64, false, NT, Team, RT>(x, roots, tid);
        stage_static<R, L, NL, 4, 512, true, NT, Team, RT>(x, roots, tid);
    } else {
        static_assert(HasStaticPlan<L>::value, "no static plan for this L");
    }
    return e;
}

// ------------------------------------------------------------- bin map
// bin(m) = sum_k c_k alpha_k m_k mod L (numtheory.py:139-153);
// u_tau(m) = sum_k c_k tau_k m_k mod L (decoder.py:41-46).  Every term is
// < L * N_k and the host guards D * L * max N_k < 2^31, so int32 is exact.
__device__ __forceinline__ int bin_of(const int *m, const Geo &g, const int *al) {
    int acc = 0;
#pragma unroll
    for (int k = 0; k < MAXD; ++k)
        if (k < g.D) acc += g.cof[k] * al[k] * m[k];
    return acc % g.L;
}
__device__ __forceinline__ int phase_of(const int *m, const Geo &g, const int *ta) {
    int acc = 0;
#pragma unroll
    for (int k = 0; k < MAXD; ++k)
        if (k < g.D) acc += g.cof[k] * ta[k] * m[k];
    return acc % g.L;
}
// Phase of offset i (0 = tau, i = tau + e_{i-1}) from u_0: the step adds
// c_{i-1} m_{i-1} < L (a wrap of tau adds L m, which vanishes mod L).
// (Selects instead of indexing with i keep m and g in registers.)
__device__ __forceinline__ int phase_step(int u0, int i, const int *m, const Geo &g) {
    int add = 0;
#pragma unroll
    for (int k = 0; k < MAXD; ++k)
        if (k == i - 1) add = g.cof[k] * m[k];
    const int u = u0 + add;
    return u >= g.L ? u - g.L : u;
}

// The magnitude half of the 1-sparse test (decoder.py:146-148): occupied
// (|S_0| > floor) and all D+1 magnitudes within mag_tol of the largest.
// Float64 evaluates it exactly as the reference (hypot magnitudes); float32
// compares squared magnitudes (no square roots): top - low <= t top  <=>
// low^2 >= (1 - t)^2 top^2 for t < 1.  `res` receives the bin's largest
// |S_i|^2 (float) / |S_i| (double) for the termination test.
template <class R, bool PAD = false>
__device__ __forceinline__ bool bin_is_candidate(const cpx<R> *spec, const Geo &g, int b,
                                                 R mag_tol, R floor, R *res) {
    if constexpr (sizeof(R) == 4) {
        const R q0 = cabs2(spec[padi<PAD>(b)]);
        R top = q0, low = q0;
#pragma unroll
        for (int i = 1; i < MAXD + 1; ++i) {
            if (i <= g.D) {
                const R qi = cabs2(spec[padi<PAD>(i * g.L + b)]);
                top = max(top, qi);
                low = min(low, qi);
            }
        }
        *res = top;
        const R c = (R)1 - mag_tol;
        return q0 > floor * floor && (mag_tol >= (R)1 || low >= c * c * top);
    } else {
        const R m0 = cabs(spec[padi<PAD>(b)]);
        R top = m0, low = m0;
#pragma unroll
        for (int i = 1; i < MAXD + 1; ++i) {
            if (i <= g.D) {
                const R mi = cabs(spec[padi<PAD>(i * g.L + b)]);
                top = max(top, mi);
                low = min(low, mi);
            }
        }
        *res = top;
        return m0 > floor && (top - low) <= mag_tol * top;
    }
}
// Largest |S_i[b]|^2 (float) or |S_i[b]| (double) over the D+1 lines.
template <class R, bool PAD = false>
__device__ __forceinline__ R bin_residual(const cpx<R> *spec, const Geo &g, int b) {
    R top = (R)0;
#pragma unroll
    for (int i = 0; i < MAXD + 1; ++i) {
        if (i <= g.D) {
            const cpx<R> v = spec[padi<PAD>(i * g.L + b)];
            top = max(top, sizeof(R) == 4 ? cabs2(v) : cabs(v));
        }
    }
    return top;
}

// ---------------------------------------------------------- classifier
// decode_spectra for one bin b (decoder.py:127-169) with the driver's guard
// (driver.py:166-176), on the bin's D+1 values s[0..D].  Returns 0 (not a
// candidate), 1 (candidate, rejected), 2 (accepted), 3 (decoded and verified
// but guard failed).  `roots` is any exact-phase table e^{+2 pi i j / L}.
template <class R, class RT = const cpx<R> *>
__device__ __forceinline__ int classify_values(const cpx<R> *s, const Geo &g, int b,
                                               const int *al, const int *ta,
                                               RT roots, R mag_tol, R round_tol,
                                               R verify_tol, R floor, int *m, cpx<R> *amp_out) {
    const int D = g.D;
    R mag[MAXD + 1];
#pragma unroll
    for (int i = 0; i < MAXD + 1; ++i)
        if (i <= D) mag[i] = cabs(s[i]);
    R top = mag[0], low = mag[0];
#pragma unroll
    for (int i = 1; i < MAXD + 1; ++i) {
        if (i <= D) {
            top = max(top, mag[i]);
            low = min(low, mag[i]);
        }
    }
    if (!(mag[0] > floor && (top - low) <= mag_tol * top)) return 0;
    const R two_pi = (R)6.283185307179586476925286766559;
    bool ok = true;
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
        if (k < D) {
            cpx<R> z = mulc(s[k + 1], s[0]);
            R theta = atan2(z.im, z.re);
            R raw = (R)g.N[k] * theta / two_pi;
            R near = rint(raw);
            ok = ok && (fabs(raw - near) <= round_tol);
            m[k] = wrap_index((int)near, g.N[k]);
        }
    }
    if (!ok) return 1;
    const int u0 = phase_of(m, g, ta);
    const cpx<R> amp = mulc(s[0], roots[u0]);
    const R lim = verify_tol * mag[0];
#pragma unroll
    for (int i = 0; i < MAXD + 1; ++i) {
        if (i <= D) {
            cpx<R> d = amp * roots[phase_step(u0, i, m, g)] - s[i];
            ok = ok && (cabs(d) <= lim);
        }
    }
    if (!ok) return 1;
    *amp_out = amp;
    if (al != nullptr && bin_of(m, g, al) != b) return 3;
    return 2;
}
template <class R>
__device__ __forceinline__ int classify_bin(const cpx<R> *spec, const Geo &g, int b,
                                            const int *al, const int *ta, const cpx<R> *roots,
                                            R mag_tol, R round_tol, R verify_tol, R floor,
                                            int *m, cpx<R> *amp_out) {
    cpx<R> s[MAXD + 1];
#pragma unroll
    for (int i = 0; i < MAXD + 1; ++i)
        if (i <= g.D) s[i] = spec[i * g.L + b];
    return classify_values(s, g, b, al, ta, roots, mag_tol, round_tol, verify_tol, floor, m,
                           amp_out);
}

// As classify_bin for a bin already known to pass the magnitude test.
// s_out / r_out (optional): the bin's D+1 values and, when verified, the D+1
// roots of the re-prediction (what the merge subtracts with).
template <class R, bool PAD = false>
__device__ __forceinline__ int decode_candidate(const cpx<R> *spec, const Geo &g, int b,
                                            const int *al, const int *ta, const cpx<R> *roots,
                                            R round_tol, R verify_tol,
                                            int *m, cpx<R> *amp_out, cpx<R> *s_out = nullptr,
                                            cpx<R> *r_out = nullptr) {
    const int L = g.L, D = g.D;
    cpx<R> s[MAXD + 1];
#pragma unroll
    for (int i = 0; i < MAXD + 1; ++i)
        if (i <= D) s[i] = spec[padi<PAD>(i * L + b)];
    if (s_out)
#pragma unroll
        for (int i = 0; i < MAXD + 1; ++i)
            if (i <= D) s_out[i] = s[i];
    const R mag0 = cabs(s[0]);
    const R two_pi = (R)6.283185307179586476925286766559;
    bool ok = true;
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
        if (k < D) {
            cpx<R> z = mulc(s[k + 1], s[0]);
            R theta = atan2(z.im, z.re);
            // float64: the reference's n * angle / (2 pi); float32 multiplies
            // by the reciprocal (no division slow path)
            R raw = sizeof(R) == 8 ? (R)g.N[k] * theta / two_pi
                                   : (R)g.N[k] * theta * (R)0.15915494309189533577;
            R near = rint(raw);
            ok = ok && (fabs(raw - near) <= round_tol);
            m[k] = wrap_index((int)near, g.N[k]);
        }
    }
    if (!ok) return 1;
    const int u0 = phase_of(m, g, ta);
    const cpx<R> amp = mulc(s[0], roots[u0]);
    const R lim = verify_tol * mag0;
#pragma unroll
    for (int i = 0; i < MAXD + 1; ++i) {
        if (i <= D) {
            const cpx<R> r = roots[phase_step(u0, i, m, g)];
            if (r_out) r_out[i] = r;
            cpx<R> d = amp * r - s[i];
            ok = ok && (sizeof(R) == 8 ? cabs(d) <= lim : cabs2(d) <= lim * lim);
        }
    }
    if (!ok) return 1;
    *amp_out = amp;
    if (al != nullptr && bin_of(m, g, al) != b) return 3;
    return 2;
}

}  // namespace fpssft
