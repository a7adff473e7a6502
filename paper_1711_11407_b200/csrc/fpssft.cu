// B200-native FPS-SFT: kernels and the C ABI declared in include/fpssft.h.
//
// recover_kernel is the product: one CTA per instance runs the whole
// projection-slice loop of fps_sft (reference driver.py:121-212) on chip --
// gather D+1 lines from the HBM-resident cube, FFT them in shared memory,
// peel the recovered set, classify/decode every bin, merge, test termination
// -- and writes the padded RecoveryReport.  The other kernels expose single
// steps (line spectra, DFT, classifier, projection) through the same device
// code so each reference function can be parity-tested on its own.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <functional>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>
#include <numeric>
#include <string>
#include <type_traits>

#include "../../include/fpssft.h"
#include "fpssft_device.cuh"

#ifndef FPSSFT_PREFETCH_FROM
#define FPSSFT_PREFETCH_FROM 4  // L2-prefetch iteration t+1 from iteration t >= this on
#endif
#ifndef FPSSFT_PREFETCH_SMEM
#define FPSSFT_PREFETCH_SMEM 0  // A/B: warp kernel, lines of <= 64 points: iteration t+1 samples
                                // copied into a second buffer (cp.async) during t (config 3
                                // guarded 1.21 -> 1.82 ms: a second wave; -1.6 % warp cycles)
#endif
#ifndef FPSSFT_TEAM_GATHER_NC
#define FPSSFT_TEAM_GATHER_NC FPSSFT_GATHER_NC
#endif
#ifndef FPSSFT_SYNTH_WARPFFT
#define FPSSFT_SYNTH_WARPFFT 1  // per-warp row FFTs in the static synthesis kernel
#endif
#ifndef FPSSFT_SYNTH_REG
#define FPSSFT_SYNTH_REG 1  // float32 512-point rows: register-FFT synthesis kernel
#endif
#ifndef FPSSFT_SYNTH_RC
#define FPSSFT_SYNTH_RC 16  // rows per chunk of synth512_kernel
#endif
#ifndef FPSSFT_SYNTH_PAIR
#define FPSSFT_SYNTH_PAIR 1  // synth512_kernel: row pairs per warp (second FFT stage without shuffles),
                             // bank-conflict-free column order
#endif
#ifndef FPSSFT_SYNTH_NT
#define FPSSFT_SYNTH_NT 256  // threads per CTA of synth512_kernel (512 / NT CTAs per SM)
#endif
#ifndef FPSSFT_SYNTH_PACKED
#define FPSSFT_SYNTH_PACKED 0  // synth512_kernel: packed float32 pairs (FADD2 / FMUL2 / FFMA2); A/B: same time
#endif
#ifndef FPSSFT_SYNTH_QUAD
#define FPSSFT_SYNTH_QUAD 1  // synth512_kernel: a chunk is 4 rows of each quarter of the image, whose sparse
                             // parts share one phasor recurrence (quarter-period shift = i^(m0 q))
#endif
#ifndef FPSSFT_SYNTH_SPARSE
#define FPSSFT_SYNTH_SPARSE 0  // A/B: 1 = packed pairs in the sparse part only, 2 = two phasor chains
#endif
#ifndef FPSSFT_SYNTH_DB
#define FPSSFT_SYNTH_DB 0  // synth512_kernel: double-buffered chunks (measured slower)
#endif
#ifndef SYNTH_RC
#define SYNTH_RC 16  // rows per chunk of the static 512-point synthesis kernel
#endif
#ifndef SYNTH_NT
#define SYNTH_NT 256
#endif
#ifndef FPSSFT_WARP_FFT_JOINT
#define FPSSFT_WARP_FFT_JOINT 0  // A/B: warp kernel, 256-point lines transformed together (measured slower: spills)
#endif
#ifndef FPSSFT_GUARD_FFT64
#define FPSSFT_GUARD_FFT64 1  // guarded warp kernel, 64-point lines: register/shuffle float64 FFT
#endif
#ifndef FPSSFT_GUARD_R64
#define FPSSFT_GUARD_R64 1  // guarded warp kernel: float64 root table (not a float32 hi/lo pair)
#endif
#ifndef FPSSFT_CLASSIFY_SPLIT
#define FPSSFT_CLASSIFY_SPLIT 1  // group kernel: all bins tested before the ballots (ILP; measured
                                 // -2 % there, +3 % on the batch-major kernel and config 3)
#endif
#ifndef FPSSFT_DECODE_PIPE
#define FPSSFT_DECODE_PIPE 0  // A/B: decode of chunk i+1 ahead of merge i (measured +2 %: off)
#endif
#ifndef FPSSFT_PROJ_LANE
#define FPSSFT_PROJ_LANE 1  // warp kernel float32: projection from per-lane contributions
#endif
#ifndef FPSSFT_WARP_MINB_SHORT
#define FPSSFT_WARP_MINB_SHORT 1  // lines of <= 64 points: registers for ILP (config 3 has ~7
                                  // instances per SM anyway; guarded 1.344 -> 1.221 ms)
#endif
#ifndef FPSSFT_PROJ_X2
#define FPSSFT_PROJ_X2 0  // A/B: lines of <= 64 points, projection two chunks at a time (+2 %: off)
#endif
#ifndef FPSSFT_WARP_FFT_JOINT2
#define FPSSFT_WARP_FFT_JOINT2 0  // A/B: group kernel, 256-point lines 0 and 1 transformed together
#endif
#ifndef FPSSFT_DECODE_KEEP
#define FPSSFT_DECODE_KEEP 1  // group kernel: decode values/roots reused by the merge (-1.4 %;
                              // batch-major +1.6 %, config 3 +10 %: group kernel only)
#endif
#ifndef FPSSFT_OUT_BITONIC
#define FPSSFT_OUT_BITONIC 1  // warp kernel, k_cap <= 128: output order by a register bitonic sort
#endif
#ifndef FPSSFT_TEAM256
#define FPSSFT_TEAM256 0  // A/B: team kernels for 256-point lines
#endif
#ifndef FPSSFT_GROUP_ASSIST
#define FPSSFT_GROUP_ASSIST 1  // group kernel: idle warps transform the last members' lines
#endif
#ifndef FPSSFT_GROUP_MINB
#define FPSSFT_GROUP_MINB 2  // group kernel: CTAs per SM its registers must allow (3: compact layout)
#endif
#ifndef FPSSFT_GROUP_LATE
#define FPSSFT_GROUP_LATE 1  // group kernel: finished warps gather after the barrier (0: A/B)
#endif
#ifndef FPSSFT_GROUP_PF
#define FPSSFT_GROUP_PF 0  // group kernel: L2-prefetch iteration t+1 during t for t + 1 < this
#endif
#ifndef FPSSFT_WARP_NT
#define FPSSFT_WARP_NT 256  // largest CTA of the warp kernel (FPSSFT_WARP_NT / 32 instances)
#endif
#ifndef FPSSFT_WARP_REGFFT256
#define FPSSFT_WARP_REGFFT256 1  // warp kernel, 256-point lines: register FFT (regfft::fft256)
#endif
#ifndef FPSSFT_WARP_W
#define FPSSFT_WARP_W 0  // A/B builds only: force the warp kernel's instances per CTA (0 = planner)
#endif
#ifndef FPSSFT_TEAM_NT
#define FPSSFT_TEAM_NT 0  // A/B builds only: force the team kernel's CTA size (0 = planner)
#endif
#ifndef FPSSFT_WARP_MINB
#define FPSSFT_WARP_MINB 2  // CTAs of FPSSFT_WARP_NT threads per SM its registers must allow
#endif

namespace fpssft {

// ------------------------------------------------------------ smem layout
struct Layout {
    size_t spec, roots, slot_amp, slot_m, slot_key, slot_live, hash;
    size_t bin_start, bin_fill, seg, slot_bin, slot_u0;  // projection scratch (union A)
    size_t dec_amp, dec_m, dec_lin, dec_slot;            // classifier scratch (union B)
    size_t red, total;
    int H;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline Layout make_layout(int D, int L, int k_cap, int cs) {
    Layout y;
    const int nl = D + 1;
    size_t o = 0;
    y.H = 2 * k_cap;
    y.spec = o;      o = align16(o + (size_t)nl * L * cs);
    y.roots = o;     o = align16(o + (size_t)L * cs);
    y.slot_amp = o;  o = align16(o + (size_t)k_cap * cs);
    y.slot_m = o;    o = align16(o + (size_t)k_cap * D * 4);
    y.slot_key = o;  o = align16(o + (size_t)k_cap * 4);
    y.slot_live = o; o = align16(o + (size_t)k_cap * 4);
    y.hash = o;      o = align16(o + (size_t)y.H * 4);
    const size_t u = o;
    y.bin_start = u; size_t a = align16(u + (size_t)(L + 1) * 4);
    y.bin_fill = a;  a = align16(a + (size_t)L * 4);
    y.seg = a;       a = align16(a + (size_t)k_cap * 4);
    y.slot_bin = a;  a = align16(a + (size_t)k_cap * 4);
    y.slot_u0 = a;   a = align16(a + (size_t)k_cap * 4);
    y.dec_amp = u;   size_t b = align16(u + (size_t)L * cs);
    y.dec_m = b;     b = align16(b + (size_t)L * D * 4);
    y.dec_lin = b;   b = align16(b + (size_t)L * 4);
    y.dec_slot = b;  b = align16(b + (size_t)L * 4);
    o = a > b ? a : b;
    y.red = o;       o = align16(o + 64 * 8);
    y.total = o;
    return y;
}

struct OutPtrs {
    int *freqs;
    double *amps;
    int *count, *iterations;
    long long *samples_used;
    int *terminated_by, *iter_stats;
};

__device__ __forceinline__ unsigned hash32(int key) { return (unsigned)key * 2654435761u; }

__device__ __forceinline__ int hash_find(const int *hash, const int *slot_key, int H, int key) {
    unsigned h = hash32(key) & (unsigned)(H - 1);
    while (true) {
        const int s = hash[h];
        if (s < 0) return -1;
        if (slot_key[s] == key) return s;
        h = (h + 1) & (unsigned)(H - 1);
    }
}
__device__ __forceinline__ void hash_insert(int *hash, int H, int key, int slot) {
    unsigned h = hash32(key) & (unsigned)(H - 1);
    while (atomicCAS(&hash[h], -1, slot) != -1) h = (h + 1) & (unsigned)(H - 1);
}

__device__ __forceinline__ int linear_index(const int *m, const Geo &g) {
    int lin = 0;
#pragma unroll
    for (int k = 0; k < MAXD; ++k)
        if (k < g.D) lin = lin * g.N[k] + m[k];
    return lin;
}

__device__ __forceinline__ bool line_params_ok(const Geo &g, const int *al, const int *ta) {
    bool ok = true;
#pragma unroll
    for (int k = 0; k < MAXD; ++k)
        if (k < g.D) ok = ok && al[k] >= 0 && al[k] < g.N[k] && ta[k] >= 0 && ta[k] < g.N[k];
    return ok;
}

// ------------------------------------------------------------ projection
// Line spectrum of the recovered set (project_onto_bins, decoder.py:172-191)
// for `nl` offsets, either subtracted from spec (driver.py:150-154) or
// stored.  Per-bin sums run in slot order (= insertion order, like
// np.bincount over the dict arrays) via a counting sort, so the result is
// deterministic -- no floating-point atomics.
template <class R>
__device__ void project_bins(cpx<R> *spec, int nl, const Geo &g, const int *al, const int *ta,
                             int n_slots, const int *slot_m, const cpx<R> *slot_amp,
                             const int *slot_live, int *bin_start, int *bin_fill, int *seg,
                             int *slot_bin, int *slot_u0, const cpx<R> *roots, int *ired,
                             bool subtract) {
    const int L = g.L, D = g.D, NT = blockDim.x, tid = threadIdx.x;
    for (int b = tid; b < L; b += NT) bin_fill[b] = 0;
    __syncthreads();
    for (int s = tid; s < n_slots; s += NT) {
        if (slot_live == nullptr || slot_live[s]) {
            int m[MAXD];
#pragma unroll
            for (int k = 0; k < MAXD; ++k) m[k] = k < D ? slot_m[s * D + k] : 0;
            const int b = bin_of(m, g, al);
            slot_bin[s] = b;
            slot_u0[s] = phase_of(m, g, ta);
            atomicAdd(&bin_fill[b], 1);
        } else {
            slot_bin[s] = -1;
        }
    }
    __syncthreads();
    int carry = 0;
    for (int j0 = 0; j0 < L; j0 += NT) {
        const int b = j0 + tid;
        const int c = b < L ? bin_fill[b] : 0;
        int tot;
        const int pre = block_exscan(c, ired, &tot);
        if (b < L) {
            bin_start[b] = carry + pre;
            bin_fill[b] = 0;
        }
        carry += tot;
    }
    if (tid == 0) bin_start[L] = carry;
    __syncthreads();
    for (int s = tid; s < n_slots; s += NT) {
        const int b = slot_bin[s];
        if (b >= 0) seg[bin_start[b] + atomicAdd(&bin_fill[b], 1)] = s;
    }
    __syncthreads();
    for (int b = tid; b < L; b += NT) {
        const int st = bin_start[b], en = bin_start[b + 1];
        for (int i = st + 1; i < en; ++i) {  // segments are short: insertion sort
            const int v = seg[i];
            int j = i - 1;
            while (j >= st && seg[j] > v) {
                seg[j + 1] = seg[j];
                --j;
            }
            seg[j + 1] = v;
        }
        for (int i = 0; i < nl; ++i) {
            cpx<R> P = {(R)0, (R)0};
            for (int p = st; p < en; ++p) {
                const int s = seg[p];
                int m[MAXD];
#pragma unroll
                for (int k = 0; k < MAXD; ++k) m[k] = k < D ? slot_m[s * D + k] : 0;
                P = P + slot_amp[s] * roots[phase_step(slot_u0[s], i, m, g)];
            }
            if (subtract) {
                if (en > st) spec[i * L + b] = spec[i * L + b] - P;
            } else {
                spec[i * L + b] = P;
            }
        }
    }
    __syncthreads();
}

// ------------------------------------------------------------ fused loop
template <class R>
__global__ void __launch_bounds__(1024, 1) recover_kernel(const float2 *__restrict__ cubes,
                                                       long long batch_stride, Geo g, Knobs kn,
                                                       const int *__restrict__ schedule,
                                                       const int *__restrict__ sched_index,
                                                       int n_sched, OutPtrs out) {
    extern __shared__ __align__(16) unsigned char sm[];
    const Layout lay = make_layout(g.D, g.L, kn.k_cap, (int)sizeof(cpx<R>));
    cpx<R> *spec = (cpx<R> *)(sm + lay.spec);
    cpx<R> *roots = (cpx<R> *)(sm + lay.roots);
    cpx<R> *slot_amp = (cpx<R> *)(sm + lay.slot_amp);
    int *slot_m = (int *)(sm + lay.slot_m);
    int *slot_key = (int *)(sm + lay.slot_key);
    int *slot_live = (int *)(sm + lay.slot_live);
    int *hash = (int *)(sm + lay.hash);
    int *bin_start = (int *)(sm + lay.bin_start);
    int *bin_fill = (int *)(sm + lay.bin_fill);
    int *seg = (int *)(sm + lay.seg);
    int *slot_bin = (int *)(sm + lay.slot_bin);
    int *slot_u0 = (int *)(sm + lay.slot_u0);
    cpx<R> *dec_amp = (cpx<R> *)(sm + lay.dec_amp);
    int *dec_m = (int *)(sm + lay.dec_m);
    int *dec_lin = (int *)(sm + lay.dec_lin);
    int *dec_slot = (int *)(sm + lay.dec_slot);
    int *ired = (int *)(sm + lay.red);
    R *rred = (R *)(sm + lay.red + 256);

    const int L = g.L, D = g.D, nl = g.nlines, NT = blockDim.x, tid = threadIdx.x;
    const int inst = blockIdx.x;
    const float2 *cube = cube_base(cubes, (long long)inst, batch_stride, kn.group);
    int sidx = sched_index ? sched_index[inst] : 0;
    const bool sched_ok = sidx >= 0 && sidx < n_sched;
    if (!sched_ok) sidx = 0;
    const int *sched = schedule + (long long)sidx * kn.t_max * 2 * D;
    const int H = lay.H;
    const R mag_tol = (R)kn.mag_tol, round_tol = (R)kn.round_tol, verify_tol = (R)kn.verify_tol;
    const R prune = (R)kn.amp_prune_tol;

    build_roots(roots, L);
    for (int h = tid; h < H; h += NT) hash[h] = -1;
    __syncthreads();

    int n_slots = 0, stall = 0, it_run = 0;
    int term = sched_ok ? FPSSFT_TERM_MAX_ITERATIONS : -1;
    R amp_sum = (R)0;

    for (int it = 0; it < kn.t_max && term != -1; ++it) {
        int al[MAXD], ta[MAXD];
#pragma unroll
        for (int k = 0; k < MAXD; ++k) {
            al[k] = k < D ? sched[(long long)it * 2 * D + k] : 0;
            ta[k] = k < D ? sched[(long long)it * 2 * D + D + k] : 0;
        }
        if (!line_params_ok(g, al, ta)) {
            term = -1;
            break;
        }
        it_run = it + 1;

        // (1) gather + (2) DFT of the D+1 lines           driver.py:146-154
        R my_energy;
        if constexpr (sizeof(R) == 4) {
            gather_lines_async(spec, cube, g, al, ta, tid, NT);
            cp_async_wait_all();
            __syncthreads();
            my_energy = kn.noise_coef > 0 ? line_energy(spec, nl * L, tid, NT) : (R)0;
        } else {
            my_energy = gather_lines(spec, cube, g, al, ta, tid, NT);
            __syncthreads();
        }
        fft_lines<R, BlockTeam>(spec, nl, g, roots, tid, NT);
        // float32 only: bins below the transform's own rounding floor are
        // numerically empty ("precision floor")
        R noise_floor = (R)0;
        if (sizeof(R) == 4 && kn.noise_coef > 0)
            noise_floor = (R)kn.noise_coef * sqrt(block_sum(my_energy, rred));
        // (3) construction-subtraction of the recovered set
        if (n_slots > 0)
            project_bins(spec, nl, g, al, ta, n_slots, slot_m, slot_amp, slot_live, bin_start,
                         bin_fill, seg, slot_bin, slot_u0, roots, ired, true);

        // (4) classify every bin                            driver.py:156-176
        const R floor =
            max(max((R)kn.energy_floor_abs, (R)kn.energy_floor * amp_sum), noise_floor);
        int my_cand = 0, my_acc = 0;
        for (int b = tid; b < L; b += NT) {
            int m[MAXD];
            cpx<R> a;
            const int st = classify_bin(spec, g, b, al, ta, roots, mag_tol, round_tol,
                                        verify_tol, floor, m, &a);
            my_cand += st > 0;
            if (st == 2) {
                ++my_acc;
                dec_lin[b] = linear_index(m, g);
#pragma unroll
                for (int k = 0; k < MAXD; ++k)
                    if (k < D) dec_m[b * D + k] = m[k];
                dec_amp[b] = a;
            } else {
                dec_lin[b] = -1;
            }
        }
        const int n_cand = block_sum(my_cand, ired);
        const int n_acc = block_sum(my_acc, ired);

        // (5) merge-by-sum into the recovered set, ascending bin order
        //     (driver.py:103-108)
        if (n_acc > 0) {
            int total_new = 0;
            for (int j0 = 0; j0 < L; j0 += NT) {
                const int b = j0 + tid;
                int isnew = 0;
                if (b < L && dec_lin[b] >= 0) {
                    const int s = hash_find(hash, slot_key, H, dec_lin[b]);
                    isnew = s < 0;
                    dec_slot[b] = s;
                }
                int tot;
                const int pre = block_exscan(isnew, ired, &tot);
                if (isnew) dec_slot[b] = (1 << 30) | (n_slots + total_new + pre);
                total_new += tot;
            }
            if (n_slots + total_new > kn.k_cap) {
                term = FPSSFT_TERM_K_CAP_OVERFLOW;
                if (tid == 0 && out.iter_stats) {
                    int *st = out.iter_stats + ((long long)inst * kn.t_max + it) * 3;
                    st[0] = n_cand;
                    st[1] = 0;
                    st[2] = n_cand;
                }
                break;
            }
            for (int b = tid; b < L; b += NT) {
                if (dec_lin[b] < 0) continue;
                const int code = dec_slot[b];
                const int s = code & ((1 << 30) - 1);
                const cpx<R> a = dec_amp[b];
                int m[MAXD];
#pragma unroll
                for (int k = 0; k < MAXD; ++k) m[k] = k < D ? dec_m[b * D + k] : 0;
                cpx<R> v;
                if (code >> 30) {
                    slot_key[s] = dec_lin[b];
#pragma unroll
                    for (int k = 0; k < MAXD; ++k)
                        if (k < D) slot_m[s * D + k] = m[k];
                    hash_insert(hash, H, dec_lin[b], s);
                    v = a;
                } else {
                    v = slot_amp[s] + a;  // a pruned slot holds 0: entries.get(f, 0) + a
                }
                const bool keep = !(cabs(v) <= prune);
                slot_amp[s] = keep ? v : cpx<R>{(R)0, (R)0};
                slot_live[s] = keep;
                // remove the new sinusoid from this iteration's spectra
                // (driver.py:189-194); its bin holds no other new entry
                const int u0 = phase_of(m, g, ta);
                for (int i = 0; i < nl; ++i)
                    spec[i * L + b] = spec[i * L + b] - a * roots[phase_step(u0, i, m, g)];
            }
            n_slots += total_new;
            __syncthreads();
        }

        // (6) amp_sum = sum |a| over the recovered set        driver.py:108
        R my = (R)0;
        for (int s = tid; s < n_slots; s += NT)
            if (slot_live[s]) my += cabs(slot_amp[s]);
        amp_sum = block_sum(my, rred);
        stall = n_acc > 0 ? 0 : stall + 1;

        // (7) termination                                     driver.py:196-204
        R mx = (R)0;
        for (int e = tid; e < nl * L; e += NT) mx = max(mx, cabs(spec[e]));
        mx = block_max(mx, rred);
        if (tid == 0 && out.iter_stats) {
            int *st = out.iter_stats + ((long long)inst * kn.t_max + it) * 3;
            st[0] = n_cand;
            st[1] = n_acc;
            st[2] = n_cand - n_acc;
        }
        const R clean = max((R)kn.energy_floor_abs, (R)kn.residual_stop * amp_sum);
        __syncthreads();
        if (mx <= clean) {
            term = FPSSFT_TERM_RESIDUAL_CLEAN;
            break;
        }
        if (stall >= kn.stall_limit) {
            term = FPSSFT_TERM_STALL;
            break;
        }
    }

    // ---- RecoveryReport: live entries in lexicographic (= linear) order
    __syncthreads();
    const int P = kn.k_cap;  // power of two
    int my_live = 0;
    for (int s = tid; s < P; s += NT) {
        const bool live = s < n_slots && slot_live[s];
        my_live += live;
        seg[s] = live ? slot_key[s] : INT_MAX;
        slot_bin[s] = s;
    }
    const int count = block_sum(my_live, ired);
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = tid; i < P; i += NT) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool up = (i & size) == 0;
                    const int ki = seg[i], kj = seg[j];
                    if ((ki > kj) == up) {
                        seg[i] = kj;
                        seg[j] = ki;
                        const int t = slot_bin[i];
                        slot_bin[i] = slot_bin[j];
                        slot_bin[j] = t;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int r = tid; r < count; r += NT) {
        const int s = slot_bin[r];
        int *fo = out.freqs + ((long long)inst * kn.k_cap + r) * D;
        for (int k = 0; k < D; ++k) fo[k] = slot_m[s * D + k];
        double *ao = out.amps + ((long long)inst * kn.k_cap + r) * 2;
        ao[0] = (double)slot_amp[s].re;
        ao[1] = (double)slot_amp[s].im;
    }
    if (tid == 0) {
        out.count[inst] = count;
        out.iterations[inst] = it_run;
        out.samples_used[inst] = (long long)it_run * nl * L;
        out.terminated_by[inst] = term;
    }
}

#include "fpssft_guard.cuh"
#include "fpssft_regfft.cuh"

// ------------------------------------------------------ warp-per-instance
// For short lines ((D+1) L <= 2048) one warp owns one instance: the same loop
// as recover_kernel, but every step is warp-synchronous (__syncwarp, ballots,
// match_any) and a CTA hosts several independent instances that share one
// root table.  Many more instances are in flight per SM, which is what hides
// the gather latency of this short, latency-bound loop.
//
// Per-warp shared memory: spectra (or the final sort's scratch, whichever is
// larger), the slot table (packed key, amplitude, live flag), a 16-bit
// open-addressing hash, and 32-entry scratch for the projection step.
struct WarpLayout {
    size_t spec, slot_amp, slot_key, hash, slot_live, cand, scr_u, scr_amp;
    size_t x0d, pabs;  // GUARD only
    size_t spec_nx;    // warp_prefetch_smem(): the next iteration's samples
    size_t per_warp, roots, roots64;
    int H;
};

// Warp kernel shapes whose next iteration's line samples are prefetched into
// a second spectra buffer (short lines: the loop runs tens of iterations and
// the gather latency is a fixed share of each).
__host__ __device__ constexpr bool warp_prefetch_smem(int L, int cs, bool grouped) {
    return FPSSFT_PREFETCH_SMEM && cs == 8 && !grouped && L <= 64 && L % 32 == 0;
}
__host__ __device__ inline WarpLayout make_warp_layout(int D, int L, int k_cap, int cs,
                                                       bool guard = false, bool grouped = false) {
    WarpLayout y;
    const int acs = guard ? 16 : cs;  // slot amplitude bytes (complex128 when guarded)
    size_t spec_bytes = (size_t)(D + 1) * (L + L / 16 + 1) * cs;  // room for padi()
    if (!grouped && stage16_ok(D, L, cs, 32) && spec_bytes < (size_t)(D + 1) * L * 16)
        spec_bytes = (size_t)(D + 1) * L * 16;  // 16-byte staging slots (gather_lines_cg16)
    const size_t sort_bytes = 1024 + (size_t)k_cap * 4;
    // compact (group kernel at FPSSFT_GROUP_MINB 3 CTAs/SM): hash of k_cap
    // entries, candidate list inside the projection staging (not live together)
    const bool compact = grouped && FPSSFT_GROUP_MINB >= 3 && !guard && cs == 8 &&
                         (size_t)L * 2 <= 32 * (size_t)cs * (size_t)(D + 1);
    size_t o = 0;
    y.H = compact ? k_cap : 2 * k_cap;
    y.spec = o;      o = align16(o + (spec_bytes > sort_bytes ? spec_bytes : sort_bytes));
    y.spec_nx = y.spec;
    if (warp_prefetch_smem(L, cs, grouped)) {
        y.spec_nx = o; o = align16(o + (spec_bytes > sort_bytes ? spec_bytes : sort_bytes));
    }
    y.slot_amp = o;  o = align16(o + (size_t)k_cap * acs);
    y.slot_key = o;  o = align16(o + (size_t)k_cap * 4);
    y.hash = o;      o = align16(o + (size_t)y.H * 2);
    y.slot_live = o; o = align16(o + (size_t)k_cap);
    y.cand = o;      if (!compact) o = align16(o + (size_t)L * 2);
    // projection staging: per lane, its slot's contribution on every line
    // (and, guarded, the float64 line-0 one and |a|)
    // (float64: the slots' phases and amplitudes instead)
    y.scr_u = o;     o = align16(o + 32 * (size_t)(cs == 16 ? 4 : cs) * (size_t)(D + 1));
    y.scr_amp = o;   o = align16(o + (guard ? 32 * (16 + 4) : (cs == 16 ? 32 * 16 : 0)));
    y.x0d = y.pabs = o;
    if (guard) {
        y.x0d = o;   o = align16(o + (size_t)(L + L / 16 + 1) * 16);
        y.pabs = o;  o = align16(o + (size_t)L * 4);
    }
    y.per_warp = o;
    // per CTA: the float32 root table, then (guarded) the float64 one
    y.roots64 = align16((size_t)L * cs);  // lo half of Roots64Split (guarded)
    y.roots = y.roots64 + (guard ? align16((size_t)L * (FPSSFT_GUARD_R64 ? 16 : 8)) : 0);
    return y;
}

__device__ __forceinline__ void unpack_key(int key, const Geo &g, int *m) {
#pragma unroll
    for (int k = 0; k < MAXD; ++k) m[k] = k < g.D ? (key >> g.key_shift[k]) & g.key_mask[k] : 0;
}
__device__ __forceinline__ int pack_key(const int *m, const Geo &g) {
    int key = 0;
#pragma unroll
    for (int k = 0; k < MAXD; ++k)
        if (k < g.D) key |= m[k] << g.key_shift[k];
    return key;
}

constexpr unsigned short HASH_EMPTY = 0xFFFF;

__device__ __forceinline__ int hash16_find(const unsigned short *hash, const int *slot_key, int H,
                                           int key) {
    unsigned h = hash32(key) & (unsigned)(H - 1);
    [[maybe_unused]] int probes = 0;
    while (true) {
        const unsigned short s = hash[h];
        FPSSFT_CHECK(++probes <= H);
        if (s == HASH_EMPTY) return -1;
        FPSSFT_CHECK((int)s < H);  // H = 2 k_cap (k_cap in the compact layout)
        if (slot_key[s] == key) return s;
        h = (h + 1) & (unsigned)(H - 1);
    }
}
__device__ __forceinline__ void hash16_insert(unsigned short *hash, int H, int key, int slot) {
    unsigned h = hash32(key) & (unsigned)(H - 1);
    FPSSFT_CHECK(slot >= 0 && slot < H);
    [[maybe_unused]] int probes = 0;
    while (atomicCAS(hash + h, HASH_EMPTY, (unsigned short)slot) != HASH_EMPTY) {
        FPSSFT_CHECK(++probes < H);
        h = (h + 1) & (unsigned)(H - 1);
    }
}

// FPSSFT_PHASE_CLOCK builds: per-phase clock cycles of the warp kernel
// (lane 0 of every warp), summed over the launch (fpssft_debug_phase_cycles)
#ifndef FPSSFT_PHASE_CLOCK
#define FPSSFT_PHASE_CLOCK 0
#endif
#if FPSSFT_PHASE_CLOCK
__device__ unsigned long long g_phase_cycles[16];
#define PCLK_DECL() long long pclk_t = clock64(); long long pclk_acc[12] = {0}; int pclk_last = 8
#define PCLK(n) do { const long long t_ = clock64(); pclk_acc[pclk_last] += t_ - pclk_t; pclk_t = t_; pclk_last = (n); } while (0)
#define PCLK_FLUSH() do { if (lane == 0) for (int i_ = 0; i_ < 12; ++i_) atomicAdd(&g_phase_cycles[i_], (unsigned long long)pclk_acc[i_]); } while (0)
#else
#define PCLK_DECL() do {} while (0)
#define PCLK(n) do {} while (0)
#define PCLK_FLUSH() do {} while (0)
#endif

// Named barrier `id` over `n` threads (a gather team), plain and OR-reducing.
__device__ __forceinline__ void team_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ bool team_bar_or(int id, int n, bool p) {
    int r;
    asm volatile(
        "{\n\t.reg .pred pi, po;\n\tsetp.ne.s32 pi, %1, 0;\n\t"
        "bar.red.or.pred po, %2, %3, pi;\n\tselp.s32 %0, 1, 0, po;\n\t}"
        : "=r"(r) : "r"((int)p), "r"(id), "r"(n) : "memory");
    return r != 0;
}

// LC / DC: compile-time line length and dimensionality (0 = runtime), so the
// benchmark shapes get fully unrolled gathers, FFTs and bin loops.  GUARD
// (float32, compile-time shapes): the float64 reference's decisions
// (fpssft_guard.cuh) -- float64 slot amplitudes and line-0 transform, guard
// flags on every float32 decision statistic, flagged bins re-evaluated in
// float64 by the whole warp.
// STG: the instance that reads staged lines (fpssft_stage.cuh, Knobs::staged);
// a separate instantiation, so the device-resident kernels carry none of it.
template <class R, int LC, int DC, bool GUARD = false, int WG = 0, int KC = 0, bool STG = false>
__global__ void __launch_bounds__(WG > 8 ? 32 * WG : FPSSFT_WARP_NT,
                                  WG > 8 ? 1
                                         : (WG ? FPSSFT_GROUP_MINB
                                               : (LC != 0 && LC <= 64 ? FPSSFT_WARP_MINB_SHORT
                                                                      : FPSSFT_WARP_MINB)))
    recover_warp_kernel(const float2 *__restrict__ cubes,
                                                           long long batch, long long batch_stride,
                                                           Geo g_in, Knobs kn,
                                                           const int *__restrict__ schedule,
                                                           const int *__restrict__ sched_index,
                                                           int n_sched, OutPtrs out) {
    static_assert(!GUARD || (sizeof(R) == 4 && LC != 0 && DC != 0),
                  "guarded mode: float32 with a compile-time shape");
    static_assert(!WG || (sizeof(R) == 4 && LC != 0 && DC != 0 && !GUARD),
                  "group gather: float32 with a compile-time shape");
    extern __shared__ __align__(16) unsigned char sm[];
    constexpr bool PAD = LC != 0;  // padded spectra layout (see padi)
    using A = typename std::conditional<GUARD, double, R>::type;  // slot amplitude type
    Geo g = g_in;
    if (LC) g.L = LC;
    if (DC) {
        g.D = DC;
        g.nlines = DC + 1;
    }
    // KC: compile-time capacity, so the per-warp layout is constant-folded
    const int k_cap = KC ? KC : kn.k_cap;
    const WarpLayout lay = make_warp_layout(g.D, g.L, k_cap, (int)sizeof(cpx<R>), GUARD, WG != 0);
    cpx<R> *roots = (cpx<R> *)sm;
    [[maybe_unused]] cpx<float> *roots_lo = (cpx<float> *)(sm + lay.roots64);
#if FPSSFT_GUARD_R64
    using Roots64 = Roots64Full;  // guarded: a float64 root table
    [[maybe_unused]] const Roots64 roots64{(const cpx<double> *)(sm + lay.roots64)};
#else
    using Roots64 = Roots64Split;
    [[maybe_unused]] const Roots64 roots64{(const cpx<float> *)roots, roots_lo};
#endif
    build_roots(roots, g.L);
    if constexpr (GUARD) {
        if (FPSSFT_GUARD_R64) build_roots64((cpx<double> *)(sm + lay.roots64), g.L);
        else build_roots_lo(roots_lo, g.L);
    }
    __syncthreads();  // the only block-wide barrier: warps run independently below

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // WG: the CTA's warps form teams of WG consecutive instances (members of
    // one interleave group); a team gathers its members' shared line samples
    // together and meets at its own barrier (the CTA-wide one when the team is
    // the whole CTA, else named barrier 1 + team)
    [[maybe_unused]] const int team = WG ? warp / WG : 0;
    [[maybe_unused]] const int team_tid = WG ? (int)threadIdx.x - team * WG * 32 : 0;
    [[maybe_unused]] const bool team_is_cta = WG && (int)blockDim.x == WG * 32;
    const long long inst0 = (long long)blockIdx.x * (blockDim.x >> 5) + (WG ? team * WG : 0);
    const long long inst = (long long)blockIdx.x * (blockDim.x >> 5) + warp;
    // WG: the CTA's warps gather together every iteration, so a warp without
    // an instance (the batch's last group) stays to the end, inactive
    if (!WG && inst >= batch) return;
    const bool has_inst = inst < batch;
    unsigned char *base = sm + lay.roots + (size_t)warp * lay.per_warp;
    cpx<R> *spec = (cpx<R> *)(base + lay.spec);
    // PFS: iteration t+1's samples land in spec_nx (cp.async) while t runs;
    // the two buffers swap roles at the top of each iteration
    constexpr bool PFS = sizeof(R) == 4 && !WG && LC != 0 && DC != 0 && warp_prefetch_smem(LC, 8, false);
    [[maybe_unused]] cpx<R> *spec_nx = (cpx<R> *)(base + lay.spec_nx);
    [[maybe_unused]] bool pf_ok = false;  // spec_nx holds the coming iteration's samples
    cpx<A> *slot_amp = (cpx<A> *)(base + lay.slot_amp);
    int *slot_key = (int *)(base + lay.slot_key);
    unsigned short *hash = (unsigned short *)(base + lay.hash);
    unsigned char *slot_live = base + lay.slot_live;
    unsigned short *cand = (unsigned short *)(base + lay.cand);
    cpx<R> *scr_c = (cpx<R> *)(base + lay.scr_u);
    [[maybe_unused]] cpx<double> *scr_c0 = (cpx<double> *)(base + lay.scr_amp);
    [[maybe_unused]] float *scr_ca = (float *)(base + lay.scr_amp + 32 * 16);
    [[maybe_unused]] cpx<double> *x0d = (cpx<double> *)(base + lay.x0d);
    [[maybe_unused]] float *pabs = (float *)(base + lay.pabs);

    const int L = g.L, D = g.D, nl = g.nlines, H = lay.H;
    const float2 *cube = cube_base(cubes, (long long)inst, batch_stride, kn.group);
    // WG: the group shares schedule 0 (the launcher passes no sched_index)
    int sidx = (sched_index && !WG && has_inst) ? sched_index[inst] : 0;
    const bool sched_ok = sidx >= 0 && sidx < n_sched;
    if (!sched_ok) sidx = 0;
    const int *sched = schedule + (long long)sidx * kn.t_max * 2 * D;
    const R mag_tol = (R)kn.mag_tol, round_tol = (R)kn.round_tol, verify_tol = (R)kn.verify_tol;
    const unsigned lt_mask = (1u << lane) - 1u;
    [[maybe_unused]] const float2 *gbase =
        cube_base(cubes, inst0, batch_stride, kn.group);  // the CTA's first member
    [[maybe_unused]] cpx<float> *spec0 =
        (cpx<float> *)(sm + lay.roots + (WG ? (size_t)team * WG : 0) * lay.per_warp + lay.spec);

    for (int h = lane; h < H; h += 32) hash[h] = HASH_EMPTY;
    __syncwarp();
    // staged lines (fpssft_stage.cuh): this instance's (WG: the team's first
    // member's) sample 0 of iteration 0 in staged[group][t][line][l][group]
    const int sinst = (int)(WG ? inst0 : inst);
    [[maybe_unused]] const float2 *sbase =
        (STG && kn.staged != nullptr)
            ? kn.staged + (long long)(sinst / kn.group) * kn.staged_group_stride +
                  (sinst % kn.group)
            : nullptr;

    int n_slots = 0, stall = 0, it_run = 0;
    int term = sched_ok ? FPSSFT_TERM_MAX_ITERATIONS : -1;
    A amp_sum = (A)0;

    // the schedule is data-independent: iteration t+1's (alpha, tau) load
    // while iteration t runs
    int nal[MAXD], nta[MAXD];
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
        nal[k] = k < D ? sched[k] : 0;
        nta[k] = k < D ? sched[D + k] : 0;
    }
    bool active = sched_ok && has_inst;
    if constexpr (PFS) {
        if (active && g.off32 && line_params_ok(g, nal, nta)) {
            gather_lines_async<LC>((cpx<float> *)spec_nx, cube, g, nal, nta, lane, 32);
            pf_ok = true;
        }
    }
    // FPSSFT_GROUP_ASSIST: group kernel of 256-point lines, unguarded float32
    constexpr bool ASSIST = FPSSFT_GROUP_ASSIST && WG != 0 && LC == 256 && DC + 1 <= 3 &&
                            sizeof(R) == 4 && !GUARD && FPSSFT_WARP_REGFFT256;
    [[maybe_unused]] __shared__ int s_act[ASSIST ? 32 : 1];
    [[maybe_unused]] bool assisted = false;
    PCLK_DECL();
    for (int it = 0; it < kn.t_max; ++it) {
        int al[MAXD], ta[MAXD];
#pragma unroll
        for (int k = 0; k < MAXD; ++k) {
            al[k] = nal[k];
            ta[k] = nta[k];
        }
        if constexpr (WG != 0) {
            // (1) group gather: loads in flight across the barrier that waits
            // for every warp to finish the previous iteration with its spectra
            const bool lines_ok = line_params_ok(g, al, ta);
            PCLK(0);
            GroupGather<LC, DC, WG> gg;
            auto group_load = [&]() {
                if (STG && sbase != nullptr && it < kn.stage_T)
                    gg.load_staged(sbase, it, kn.group, team_tid);
                else
                    gg.load(gbase, g, al, ta, team_tid);
            };
            // a warp whose instance has finished sends its share of the gather
            // only once the barrier has shown that some member continues: the
            // team's last pass (nobody left) then reads nothing.  (A running
            // member is the last to arrive, so its own share already exposes
            // one memory latency in a straggler iteration: no longer path.)
            const bool early = !FPSSFT_GROUP_LATE || active;
            if (lines_ok && early) group_load();
            if constexpr (ASSIST)
                if (lane == 0) s_act[warp] = (int)(active && lines_ok);
            const bool any = team_is_cta ? __syncthreads_or(active && lines_ok)
                                         : team_bar_or(1 + team, WG * 32, active && lines_ok);
            if (!any) {
                if (active) term = -1;  // invalid schedule: the whole team stops
                break;
            }
            PCLK(1);
            if (!early) group_load();
            gg.store(spec0, (int)(lay.per_warp / sizeof(cpx<float>)), team_tid);
            if (it + 1 < kn.t_max) {
#pragma unroll
                for (int k = 0; k < MAXD; ++k) {
                    nal[k] = k < D ? sched[(long long)(it + 1) * 2 * D + k] : 0;
                    nta[k] = k < D ? sched[(long long)(it + 1) * 2 * D + D + k] : 0;
                }
            }
            if (team_is_cta) __syncthreads();
            else team_bar(1 + team, WG * 32);
            if constexpr (ASSIST) {
                // straggler iterations (at most 2 members still running): the
                // group's idle warps transform the active members' lines, one
                // line per warp (the same per-line code and energy order as
                // fft256_lines_warp), results and per-lane energies in place
                if (team_is_cta) {
                    unsigned amask = 0;
#pragma unroll
                    for (int w2 = 0; w2 < WG; ++w2) amask |= (unsigned)(s_act[w2] != 0) << w2;
                    const int n_act = __popc(amask);
                    assisted = n_act > 0 && n_act <= 2;
                    if (assisted) {
                        if (warp < (DC + 1) * n_act) {
                            unsigned rest = amask;
                            for (int q = warp / (DC + 1); q > 0; --q) rest &= rest - 1;
                            const int mem = __ffs(rest) - 1, line = warp % (DC + 1);
                            unsigned char *mb = sm + lay.roots + (size_t)mem * lay.per_warp;
                            cpx<float> *ml = (cpx<float> *)(mb + lay.spec) + line * 272;
                            const float e = regfft::fft256_lines_warp(ml, 1,
                                                                      (const cpx<float> *)roots, lane);
                            ((float *)(mb + lay.scr_u))[line * 32 + lane] = e;
                        }
                        __syncthreads();
                    }
                }
            }
            // L2 prefetch of the next iteration's segments (one request per
            // segment) while this one computes: only for the leading
            // iterations nearly every instance runs (FPSSFT_GROUP_PF)
            if (FPSSFT_GROUP_PF && it + 1 < FPSSFT_GROUP_PF && it + 1 < kn.t_max &&
                line_params_ok(g, nal, nta))
                gg.prefetch_l2(gbase, g, nal, nta, team_tid);
        } else if (!active) {
            break;
        }
        do {  // one iteration of this warp's instance; `break` ends its recovery
        if (!active) break;
        if (!line_params_ok(g, al, ta)) {
            term = -1;
            active = false;
            break;
        }
        it_run = it + 1;
        // staged lines: this iteration's samples of this instance (else nullptr)
        [[maybe_unused]] const float2 *sline =
            (STG && !PFS && !WG && sbase != nullptr && it < kn.stage_T)
                ? sbase + (long long)it * (nl * L) * kn.group
                : nullptr;

        // (1) gather + (2) DFT of the D+1 lines           driver.py:146-154
        R my_energy = (R)0;
        bool staged = false;
        unsigned par = 0, dup = 0;
        if constexpr (WG != 0) {
            // the group gather above filled the spectra
        } else if constexpr (sizeof(R) == 4) {
            bool reg_gather = false, pf_used = false;
            // staged lines (fpssft_stage.cuh): this iteration's samples sit in
            // line order in HBM, kn.group instances per position
            const bool from_hbm = sline != nullptr;
            if (from_hbm) {
                for (int q = lane; q < nl * L; q += 32)
                    cp_async8((cpx<float> *)spec + padi<PAD>(q), sline + (long long)q * kn.group);
            }
            if constexpr (PFS) {
                if (pf_ok) {  // prefetched during the previous iteration
                    cpx<R> *t = spec;
                    spec = spec_nx;
                    spec_nx = t;
                    pf_used = true;
                }
            }
            // register gather for short lines (config 3: 1.2% faster), cp.async
            // for L >= 256 (config 2: 1% faster) -- measured, profiles/README.md
            if constexpr (FPSSFT_GATHER_NC && LC != 0 && LC < 256 && DC != 0 &&
                          !stage16_ok(DC, LC, 8, 32)) {
                reg_gather = g.off32 && !pf_used && !from_hbm;
                if (reg_gather) gather_lines_nc<LC, DC>(spec, cube, g, al, ta, lane);
            }
            if constexpr (LC != 0 && stage16_ok(DC, LC, 8, 32)) {
                staged = g.off32 && !reg_gather && !pf_used && !from_hbm;
                if (staged)
                    par = gather_lines_cg16<LC, DC>((float4 *)spec, cube, g, al, ta, lane, &dup);
            }
            if (!reg_gather && !staged && !pf_used && !from_hbm)
                gather_lines_async<LC>(spec, cube, g, al, ta, lane, 32);
            if (it + 1 < kn.t_max) {
#pragma unroll
                for (int k = 0; k < MAXD; ++k) {
                    nal[k] = k < D ? sched[(long long)(it + 1) * 2 * D + k] : 0;
                    nta[k] = k < D ? sched[(long long)(it + 1) * 2 * D + D + k] : 0;
                }
                // long-running instances (noisy configs: tens of iterations)
                // L2-prefetch the next iteration's lines; short ones do not --
                // on config 2 (~3 iterations) the extra random DRAM fetches of
                // a last-iteration prefetch cost more than the latency saved
                if (!PFS && LC != 0 && it >= FPSSFT_PREFETCH_FROM && g.off32 &&
                    !(STG && sbase != nullptr && it + 1 < kn.stage_T) &&
                    line_params_ok(g, nal, nta))
                    prefetch_lines_l2<LC>(cube, g, nal, nta, lane);
            }
            if constexpr (GUARD)
                for (int b = lane; b < L; b += 32) pabs[b] = 0.f;
            cp_async_wait_all();
            __syncwarp();
            if constexpr (PFS) {
                // the next iteration's lines into the buffer this one left
                // (every lane's reads of it ended before the last __syncwarp)
                pf_ok = false;
                if (it + 1 < kn.t_max && g.off32 && line_params_ok(g, nal, nta)) {
                    gather_lines_async<LC>((cpx<float> *)spec_nx, cube, g, nal, nta, lane, 32);
                    pf_ok = true;
                }
            }
            if constexpr (LC != 0 && stage16_ok(DC, LC, 8, 32)) {
                if (staged) {
                    compact_stage16<LC, DC + 1, 32, WarpTeam>(spec, par, dup, lane,
                                                              GUARD ? x0d : nullptr);
                    __syncwarp();
                }
            }
            if constexpr (GUARD) {
                if (!staged) {  // line 0's samples into the float64 buffer
                    for (int l = lane; l < L; l += 32) {
                        const cpx<R> v = spec[padi<PAD>(l)];
                        x0d[padi<PAD>(l)] = {(double)v.re, (double)v.im};
                    }
                    __syncwarp();
                }
            }
            my_energy = (LC == 0 && kn.noise_coef > 0) ? line_energy(spec, nl * L, lane, 32) : (R)0;
        } else {
            my_energy = gather_lines<R, PAD>(spec, cube, g, al, ta, lane, 32);
            if (it + 1 < kn.t_max) {
#pragma unroll
                for (int k = 0; k < MAXD; ++k) {
                    nal[k] = k < D ? sched[(long long)(it + 1) * 2 * D + k] : 0;
                    nta[k] = k < D ? sched[(long long)(it + 1) * 2 * D + D + k] : 0;
                }
            }
            __syncwarp();
        }
        PCLK(2);
        if constexpr (LC == 256 && sizeof(R) == 4 && FPSSFT_WARP_REGFFT256) {
            // 256-point lines in registers (regfft::fft256_lines_warp)
            if constexpr (FPSSFT_WARP_FFT_JOINT && DC + 1 <= 3)
                my_energy = (R)regfft::fft256_lines_joint<DC + 1>((cpx<float> *)spec,
                                                                  (const cpx<float> *)roots, lane);
            else if constexpr (FPSSFT_WARP_FFT_JOINT2 && WG != 0 && DC + 1 == 3) {
                // lines 0 and 1 together, then line 2
                my_energy = (R)regfft::fft256_lines_joint<2>((cpx<float> *)spec,
                                                             (const cpx<float> *)roots, lane);
                my_energy += (R)regfft::fft256_lines_warp((cpx<float> *)spec + 2 * 272, 1,
                                                          (const cpx<float> *)roots, lane);
            } else if (ASSIST && assisted) {  // transformed by the group's idle warps
                const float *es = (const float *)scr_c;
                float e = es[lane];
#pragma unroll
                for (int i = 1; i < DC + 1; ++i) e += es[i * 32 + lane];
                my_energy = (R)e;
            } else
                my_energy = (R)regfft::fft256_lines_warp((cpx<float> *)spec, DC + 1,
                                                         (const cpx<float> *)roots, lane);
            if constexpr (GUARD) fft_static<double, LC, 1, 32, WarpTeam, Roots64>(x0d, roots64, lane);
        } else if constexpr (LC != 0) {
            const R e = fft_static<R, LC, DC + 1>(spec, roots, lane);
            if (sizeof(R) == 4) my_energy = e;
            if constexpr (GUARD && LC == 64 && FPSSFT_GUARD_FFT64)
                regfft::fft64_line_f64(x0d, roots64, lane);
            else if constexpr (GUARD)
                fft_static<double, LC, 1, 32, WarpTeam, Roots64>(x0d, roots64, lane);
        } else
            fft_lines_warp<R>(spec, nl, g, roots, lane);
        PCLK(3);
        R noise_floor = (R)0;
        [[maybe_unused]] float Ef = 0.f;  // GUARD: transform part of the error bound
        if constexpr (GUARD) {
            Ef = (float)(kn.guard_coef *
                         sqrt((double)__shfl_sync(FULL, warp_sum(my_energy), 0)));
        } else if (sizeof(R) == 4 && kn.noise_coef > 0) {
            noise_floor = (R)kn.noise_coef * sqrt(__shfl_sync(FULL, warp_sum(my_energy), 0));
        }

        // (3) construction-subtraction, 32 slots at a time in slot order:
        //     each lane computes its slot's contribution on every line; slots
        //     sharing a bin are summed by their lowest lane in lane (= slot)
        //     order, through shared memory only when a bin is hit twice.
        //     GUARD: also the float64 line-0 projection and the bins' sum |a|
        if constexpr (sizeof(R) == 8 || (!GUARD && !FPSSFT_PROJ_LANE)) {
            // float64: slot phases staged, the group's lowest lane forms the
            // sums (fewer live registers than per-lane contributions:
            // measured 1.75 vs 2.12 ms on config 3)
            int *scr_u = (int *)scr_c;
            cpx<R> *scr_amp = sizeof(R) == 8 ? (cpx<R> *)(base + lay.scr_amp)
                                             : scr_c + 16 * nl;  // after nl x 32 ints
            for (int c0 = 0; c0 < n_slots; c0 += 32) {
                const int s = c0 + lane;
                const bool valid = s < n_slots && slot_live[s];
                int b = -1 - lane;
                if (valid) {
                    int m[MAXD];
                    unpack_key(slot_key[s], g, m);
                    b = bin_of(m, g, al);
                    const int u0 = phase_of(m, g, ta);
#pragma unroll
                    for (int i = 0; i < MAXD + 1; ++i)
                        if (i < nl) scr_u[i * 32 + lane] = phase_step(u0, i, m, g);
                    scr_amp[lane] = {(R)slot_amp[s].re, (R)slot_amp[s].im};
                }
                __syncwarp();
                const unsigned grp = __match_any_sync(FULL, b);
                if (valid && lane == __ffs(grp) - 1) {
                    cpx<R> P[MAXD + 1];
#pragma unroll
                    for (int i = 0; i < MAXD + 1; ++i) P[i] = {(R)0, (R)0};
                    for (unsigned rest = grp; rest; rest &= rest - 1) {
                        const int j = __ffs(rest) - 1;
                        const cpx<R> ar = scr_amp[j];
#pragma unroll
                        for (int i = 0; i < MAXD + 1; ++i)
                            if (i < nl) P[i] = P[i] + ar * roots[scr_u[i * 32 + j]];
                    }
#pragma unroll
                    for (int i = 0; i < MAXD + 1; ++i)
                        if (i < nl) spec[padi<PAD>(i * L + b)] = spec[padi<PAD>(i * L + b)] - P[i];
                }
                __syncwarp();
            }
        } else {
            // every lane: its slot's contribution a root[u_i] on each line
            auto contrib = [&](int s, bool &valid, int &b, cpx<R> *C, cpx<double> &C0, float &ca) {
                valid = s < n_slots && slot_live[s];
                b = -1 - lane;
                C0 = {0.0, 0.0};
                ca = 0.f;
                if (valid) {
                    int m[MAXD];
                    unpack_key(slot_key[s], g, m);
                    b = bin_of(m, g, al);
                    const int u0 = phase_of(m, g, ta);
                    const cpx<A> aj = slot_amp[s];
                    const cpx<R> ar = {(R)aj.re, (R)aj.im};
#pragma unroll
                    for (int i = 0; i < MAXD + 1; ++i)
                        if (i < nl) C[i] = ar * roots[phase_step(u0, i, m, g)];
                    if constexpr (GUARD) {
                        C0 = cpx<double>{(double)aj.re, (double)aj.im} * roots64[u0];
                        ca = cabs(ar);
                    }
                }
            };
            // slots sharing a bin are summed by their lowest lane in lane
            // (= slot) order; a bin hit once is updated by its own lane
            auto apply = [&](bool valid, int b, cpx<R> *C, cpx<double> C0, float ca) {
                const unsigned grp = __match_any_sync(FULL, b);
                const bool multi = (grp & (grp - 1)) != 0;
                const bool lead = valid && lane == __ffs(grp) - 1;
                if (__any_sync(FULL, valid && multi)) {
                    if (valid && multi && !lead) {
#pragma unroll
                        for (int i = 0; i < MAXD + 1; ++i)
                            if (i < nl) scr_c[i * 32 + lane] = C[i];
                        if constexpr (GUARD) {
                            scr_c0[lane] = C0;
                            scr_ca[lane] = ca;
                        }
                    }
                    __syncwarp();
                    if (lead && multi) {
                        for (unsigned rest = grp & (grp - 1); rest; rest &= rest - 1) {
                            const int j = __ffs(rest) - 1;
#pragma unroll
                            for (int i = 0; i < MAXD + 1; ++i)
                                if (i < nl) C[i] = C[i] + scr_c[i * 32 + j];
                            if constexpr (GUARD) {
                                C0 = C0 + scr_c0[j];
                                ca += scr_ca[j];
                            }
                        }
                    }
                }
                if (lead) {
#pragma unroll
                    for (int i = 0; i < MAXD + 1; ++i)
                        if (i < nl) spec[padi<PAD>(i * L + b)] = spec[padi<PAD>(i * L + b)] - C[i];
                    if constexpr (GUARD) {
                        x0d[padi<PAD>(b)] = x0d[padi<PAD>(b)] - C0;
                        pabs[b] += ca;
                    }
                }
                __syncwarp();
            };
            // short lines (few instances per SM, registers to spare): two
            // chunks' contributions computed together, applied in slot order
            constexpr bool X2 = FPSSFT_PROJ_X2 && LC != 0 && LC <= 64;
            for (int c0 = 0; c0 < n_slots; c0 += X2 ? 64 : 32) {
                bool va, vb = false;
                int ba, bb = 0;
                cpx<R> Ca[MAXD + 1], Cb[MAXD + 1];
                cpx<double> C0a, C0b;
                float caa, cab;
                contrib(c0 + lane, va, ba, Ca, C0a, caa);
                if constexpr (X2) contrib(c0 + 32 + lane, vb, bb, Cb, C0b, cab);
                apply(va, ba, Ca, C0a, caa);
                if constexpr (X2)
                    if (c0 + 32 < n_slots) apply(vb, bb, Cb, C0b, cab);
            }
        }

        // (4) classify + (5) merge, 32 bins at a time in ascending order
        const A floor_a = max(max((A)kn.energy_floor_abs, (A)kn.energy_floor * amp_sum),
                              (A)noise_floor);
        const R floor = (R)floor_a;
        // 1-sparse magnitude test on every bin, candidates compacted in
        // ascending order so the decode runs on dense batches of 32.  The
        // termination residual (max |S|) is folded in: non-candidate bins keep
        // their values, candidates are re-read after the merge below.
        // GUARD: bins inside the guard band join the list, flagged.
        int n_cand = 0, n_acc = 0;
        R resid = (R)0;
        constexpr int NCH = (LC + 31) / 32;  // compile-time shapes: the chunks' tests
        if constexpr (LC != 0 && WG != 0 && NCH >= 4 && NCH <= 16 && FPSSFT_CLASSIFY_SPLIT) {
            // first every chunk's test (loads and arithmetic only, independent
            // chains), then the ballots and compaction
            unsigned okb = 0, flb = 0;
#pragma unroll
            for (int j = 0; j < NCH; ++j) {
                const int b = 32 * j + lane;
                R top = (R)0;
                bool ok = false, fl = false;
                if (LC % 32 == 0 || b < L) {
                    if constexpr (GUARD)
                        ok = bin_is_candidate_guarded<PAD>((const cpx<float> *)spec, g, b,
                                                           (float)mag_tol, (float)floor,
                                                           Ef + GUARD_KP * pabs[b], (float *)&top,
                                                           &fl);
                    else
                        ok = bin_is_candidate<R, PAD>(spec, g, b, mag_tol, floor, &top);
                }
                if (!ok && !fl) resid = max(resid, top);
                okb |= (unsigned)ok << j;
                flb |= (unsigned)fl << j;
            }
#pragma unroll
            for (int j = 0; j < NCH; ++j) {
                const bool c = ((okb | flb) >> j) & 1u;
                const unsigned msk = __ballot_sync(FULL, c);
                FPSSFT_CHECK(!c || n_cand + __popc(msk & lt_mask) < L);
                if (c)
                    cand[n_cand + __popc(msk & lt_mask)] =
                        (unsigned short)(32 * j + lane) |
                        (unsigned short)(((flb >> j) & 1u) ? CAND_FLAG : 0);
                n_cand += __popc(msk);
            }
        } else
        for (int c0 = 0; c0 < L; c0 += 32) {
            const int b = c0 + lane;
            R top = (R)0;
            bool ok = false, fl = false;
            if (b < L) {
                if constexpr (GUARD)
                    ok = bin_is_candidate_guarded<PAD>((const cpx<float> *)spec, g, b,
                                                       (float)mag_tol, (float)floor,
                                                       Ef + GUARD_KP * pabs[b], (float *)&top, &fl);
                else
                    ok = bin_is_candidate<R, PAD>(spec, g, b, mag_tol, floor, &top);
            }
            if (!ok && !fl) resid = max(resid, top);
            const unsigned msk = __ballot_sync(FULL, ok || fl);
            FPSSFT_CHECK(!(ok || fl) || n_cand + __popc(msk & lt_mask) < L);
            if (ok || fl)
                cand[n_cand + __popc(msk & lt_mask)] =
                    (unsigned short)b | (unsigned short)(fl ? CAND_FLAG : 0);
            n_cand += __popc(msk);
        }
        __syncwarp();
        PCLK(5);
        bool overflow = false;
        int n_cand_x = 0;
        A d_amp = (A)0;  // this lane's change of amp_sum
        // unguarded: the next chunk is decoded before this one merges (its
        // loads and arithmetic overlap the merge's dependent chain; distinct
        // bins, so no hazard)
        constexpr bool PIPE = !GUARD && FPSSFT_DECODE_PIPE;
        [[maybe_unused]] int nx_b = -1, nx_st = 0, nx_m[MAXD];
        [[maybe_unused]] cpx<R> nx_a;
        if constexpr (PIPE) {
            nx_b = lane < n_cand ? (int)(cand[lane] & ~CAND_FLAG) : -1;
            if (nx_b >= 0)
                nx_st = decode_candidate<R, PAD>(spec, g, nx_b, al, ta, roots, round_tol,
                                                 verify_tol, nx_m, &nx_a);
        }
        // unguarded float32: the decode's bin values and roots stay in
        // registers for the merge and the residual (no re-reads)
        constexpr bool KEEP = !GUARD && sizeof(R) == 4 && FPSSFT_DECODE_KEEP && !PIPE && WG != 0;
        for (int c0 = 0; c0 < n_cand; c0 += 32) {
            const int ce = c0 + lane < n_cand ? cand[c0 + lane] : -1;
            const int b = ce >= 0 ? (ce & ~(int)CAND_FLAG) : -1;
            int m[MAXD];
            cpx<R> a;
            int st = 0;
            [[maybe_unused]] cpx<R> sv[MAXD + 1], rv[MAXD + 1];
            if constexpr (PIPE) {
                st = nx_st;
                a = nx_a;
#pragma unroll
                for (int k = 0; k < MAXD; ++k) m[k] = nx_m[k];
                const int c1 = c0 + 32 + lane;
                nx_b = c1 < n_cand ? (int)(cand[c1] & ~CAND_FLAG) : -1;
                nx_st = 0;
                if (nx_b >= 0)
                    nx_st = decode_candidate<R, PAD>(spec, g, nx_b, al, ta, roots, round_tol,
                                                     verify_tol, nx_m, &nx_a);
            } else if constexpr (GUARD) {
                const bool mflag = ce >= 0 && ((ce & CAND_FLAG) || FPSSFT_GUARD_CALIB == 1);
                if (b >= 0 && !mflag)
                    st = decode_candidate_guarded<PAD>((const cpx<float> *)spec, g, b, al, ta,
                                                       (const cpx<float> *)roots,
                                                       (float)round_tol, (float)verify_tol,
                                                       Ef + GUARD_KP * pabs[b], m);
                const unsigned need = __ballot_sync(FULL, b >= 0 && (mflag || st == ST_FLAG));
#if FPSSFT_GUARD_CALIB == 2
                if (lane == 0 && need) atomicAdd(&g_guard_calib_count, (unsigned long long)__popc(need));
#endif
                // exact float64 re-evaluation of the flagged bins, one at a
                // time by the whole warp
                for (unsigned rest = need; rest; rest &= rest - 1) {
                    const int owner = __ffs(rest) - 1;
                    const int bf = __shfl_sync(FULL, b, owner);
                    int mx[MAXD];
                    [[maybe_unused]] cpx<double> S[MAXD + 1];
                    // every lane gets the same decision, the owner keeps it
                    const int sx = exact_reeval_warp<A, Roots64, LC, DC>(
                        bf, cube, g, al, ta, roots64, n_slots, slot_key, slot_live, slot_amp,
                        x0d[padi<PAD>(bf)], kn, (double)floor_a, lane, mx,
                        FPSSFT_GUARD_CALIB == 1 ? S : nullptr, STG ? sline : nullptr);
                    if (lane == owner) {
                        st = sx;
#pragma unroll
                        for (int k = 0; k < MAXD; ++k) m[k] = mx[k];
#if FPSSFT_GUARD_CALIB == 1
                        const double unit = (double)Ef / GUARD_KF + U32 * pabs[bf];
                        double worst = 0.0;
                        for (int i = 0; i <= D; ++i) {
                            const cpx<R> v = spec[padi<PAD>(i * L + bf)];
                            worst = fmax(worst, hypot((double)v.re - S[i].re,
                                                      (double)v.im - S[i].im));
                        }
                        atomicMax(&g_guard_calib_max, __float_as_uint((float)(worst / unit)));
                        atomicAdd(&g_guard_calib_count, 1ull);
#endif
                    }
                }
            } else {
                if (b >= 0)
                    st = decode_candidate<R, PAD>(spec, g, b, al, ta, roots, round_tol,
                                                  verify_tol, m, &a, KEEP ? sv : nullptr,
                                                  KEEP ? rv : nullptr);
            }
            const unsigned acc = __ballot_sync(FULL, st == 2);
            if constexpr (GUARD) n_cand_x += __popc(__ballot_sync(FULL, st >= 1));
            int key = 0, found = -1;
            if (st == 2) {
                key = pack_key(m, g);
                found = hash16_find(hash, slot_key, H, key);
            }
            const unsigned fresh = __ballot_sync(FULL, st == 2 && found < 0);
            if (n_slots + __popc(fresh) > k_cap) {
                overflow = true;
                break;
            }
            n_acc += __popc(acc);
            if (st == 2) {
                cpx<A> av;
                if constexpr (GUARD) {  // the float64 amplitude (decoder.py:160)
                    av = mulc(x0d[padi<PAD>(b)], roots64[phase_of(m, g, ta)]);
                    a = {(R)av.re, (R)av.im};
                } else {
                    av = a;
                }
                cpx<A> v = av;
                int s;
                if (found < 0) {
                    s = n_slots + __popc(fresh & lt_mask);
                    FPSSFT_CHECK(s < k_cap);
                    slot_key[s] = key;
                    hash16_insert(hash, H, key, s);
                } else {
                    s = found;
                    v = slot_amp[s] + av;  // a pruned slot holds 0: entries.get(f, 0) + a
                }
                const A av_new = cabs(v);
                const bool keep = !(av_new <= (A)kn.amp_prune_tol);
                d_amp += (keep ? av_new : (A)0) - (found < 0 ? (A)0 : cabs(slot_amp[s]));
                slot_amp[s] = keep ? v : cpx<A>{(A)0, (A)0};
                slot_live[s] = keep;
                if constexpr (KEEP) {  // the decode's values and roots, in registers
#pragma unroll
                    for (int i = 0; i < MAXD + 1; ++i)
                        if (i < nl) {
                            sv[i] = sv[i] - a * rv[i];
                            spec[padi<PAD>(i * L + b)] = sv[i];
                        }
                } else {
                    const int u0 = phase_of(m, g, ta);  // driver.py:189-194
                    for (int i = 0; i < nl; ++i)
                        spec[padi<PAD>(i * L + b)] =
                            spec[padi<PAD>(i * L + b)] - a * roots[phase_step(u0, i, m, g)];
                }
            }
            if constexpr (KEEP) {
                if (b >= 0)
#pragma unroll
                    for (int i = 0; i < MAXD + 1; ++i)
                        if (i < nl) resid = max(resid, cabs2(sv[i]));
            } else if (b >= 0) {
                resid = max(resid, bin_residual<R, PAD>(spec, g, b));
            }
            n_slots += __popc(fresh);
            __syncwarp();
        }
        if constexpr (GUARD) n_cand = n_cand_x;
        if (overflow) {
            term = FPSSFT_TERM_K_CAP_OVERFLOW;
            if (lane == 0 && out.iter_stats) {
                int *st = out.iter_stats + (inst * kn.t_max + it) * 3;
                st[0] = n_cand;
                st[1] = 0;
                st[2] = n_cand;
            }
            active = false;
            break;
        }
        __syncwarp();

        PCLK(6);
        // (6) amp_sum = sum |a| over the recovered set        driver.py:108
        //     kept incrementally: every merge adds |new| - |old| of its slot
        amp_sum += __shfl_sync(FULL, warp_sum(d_amp), 0);
        stall = n_acc > 0 ? 0 : stall + 1;

        // (7) termination                                     driver.py:196-204
        const R clean = (R)max((A)kn.energy_floor_abs, (A)kn.residual_stop * amp_sum);
        const R worst = warp_max(resid);  // |S|^2 (float) or |S| (double)
        const bool is_clean = sizeof(R) == 8 ? worst <= clean : worst <= clean * clean;
        if (lane == 0 && out.iter_stats) {
            int *st = out.iter_stats + (inst * kn.t_max + it) * 3;
            st[0] = n_cand;
            st[1] = n_acc;
            st[2] = n_cand - n_acc;
        }
        __syncwarp();
        if (is_clean) {
            term = FPSSFT_TERM_RESIDUAL_CLEAN;
            active = false;
            break;
        }
        if (stall >= kn.stall_limit) {
            term = FPSSFT_TERM_STALL;
            active = false;
            break;
        }
        } while (0);
    }
    if (!has_inst) return;  // (WG: a padding warp of the batch's last group)
    if constexpr (PFS) cp_async_wait_all();  // a prefetch past the last iteration

    PCLK(7);
    // ---- RecoveryReport: live entries sorted by packed key (= lexicographic).
    __syncwarp();
    if constexpr (KC != 0 && KC <= 128 && FPSSFT_OUT_BITONIC) {
        // compile-time capacity <= 128: a bitonic sort of (key << 7 | slot)
        // in registers, 4 per lane (element i = 4 lane + j), shuffles only
        if (g.key_bits_ + 7 <= 31) {  // (block-uniform)
            unsigned v[4];
            int my = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int sl = 4 * lane + j;
                const bool live = sl < n_slots && slot_live[sl];
                my += live;
                v[j] = live ? ((unsigned)slot_key[sl] << 7) | (unsigned)sl : 0x7FFFFFFFu;
            }
            const int count = __shfl_sync(FULL, warp_sum(my), 0);
#pragma unroll
            for (int k = 2; k <= 128; k <<= 1) {
#pragma unroll
                for (int jj = k >> 1; jj > 0; jj >>= 1) {
                    if (jj >= 4) {
                        const bool lower = (lane & (jj >> 2)) == 0;
                        const bool asc = ((4 * lane) & k) == 0;
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const unsigned y = __shfl_xor_sync(FULL, v[j], jj >> 2);
                            v[j] = (lower == asc) ? min(v[j], y) : max(v[j], y);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            if ((j ^ jj) > j) {
                                const bool asc = ((4 * lane + j) & k) == 0;
                                const unsigned x = v[j], y = v[j ^ jj];
                                v[j] = asc ? min(x, y) : max(x, y);
                                v[j ^ jj] = asc ? max(x, y) : min(x, y);
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int r = 4 * lane + j;
                if (r < count) {
                    const int sl = (int)(v[j] & 127u);
                    int m[MAXD];
                    unpack_key((int)(v[j] >> 7), g, m);
                    int *fo = out.freqs + (inst * k_cap + r) * D;
#pragma unroll
                    for (int k = 0; k < MAXD; ++k)
                        if (k < D) fo[k] = m[k];
                    double *ao = out.amps + (inst * k_cap + r) * 2;
                    ao[0] = (double)slot_amp[sl].re;
                    ao[1] = (double)slot_amp[sl].im;
                }
            }
            if (lane == 0) {
                out.count[inst] = count;
                out.iterations[inst] = it_run;
                out.samples_used[inst] = (long long)it_run * nl * L;
                out.terminated_by[inst] = term;
            }
            PCLK(8);
            PCLK_FLUSH();
            return;
        }
    }
    // Counting sort on the key's top 8 bits (shared-memory histogram, warp
    // scan, scatter), then insertion sort inside the (short) buckets.
    int *hist = (int *)spec;          // 256 buckets
    int *sslot = hist + 256;          // n_slots entries
    const int kb = g.key_bits_;
    const int shift = kb > 8 ? kb - 8 : 0;
    for (int i = lane; i < 256; i += 32) hist[i] = 0;
    __syncwarp();
    int my_live = 0;
    for (int s = lane; s < n_slots; s += 32)
        if (slot_live[s]) {
            ++my_live;
            atomicAdd(&hist[slot_key[s] >> shift], 1);
        }
    const int count = __shfl_sync(FULL, warp_sum(my_live), 0);
    __syncwarp();
    {   // exclusive scan of the 256 bucket counts: 8 consecutive per lane
        int c[8], run = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            c[i] = hist[lane * 8 + i];
            run += c[i];
        }
        int incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        int start = incl - run;
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            hist[lane * 8 + i] = start;  // becomes the bucket's fill cursor
            start += c[i];
        }
    }
    __syncwarp();
    for (int s = lane; s < n_slots; s += 32)
        if (slot_live[s]) {
            const int pos = atomicAdd(&hist[slot_key[s] >> shift], 1);
            FPSSFT_CHECK(pos >= 0 && pos < count && (slot_key[s] >> shift) < 256);
            sslot[pos] = s;
        }
    __syncwarp();
    // buckets end at hist[b] (cursor after the scatter); sort each in place
    for (int bkt = lane; bkt < 256; bkt += 32) {
        const int en = hist[bkt], st = bkt ? hist[bkt - 1] : 0;
        for (int i = st + 1; i < en; ++i) {
            const int v = sslot[i], kv = slot_key[v];
            int j = i - 1;
            while (j >= st && slot_key[sslot[j]] > kv) {
                sslot[j + 1] = sslot[j];
                --j;
            }
            sslot[j + 1] = v;
        }
    }
    __syncwarp();
    for (int r = lane; r < count; r += 32) {
        const int s = sslot[r];
        int m[MAXD];
        unpack_key(slot_key[s], g, m);
        int *fo = out.freqs + (inst * k_cap + r) * D;
#pragma unroll
        for (int k = 0; k < MAXD; ++k)
            if (k < D) fo[k] = m[k];
        double *ao = out.amps + (inst * k_cap + r) * 2;
        ao[0] = (double)slot_amp[s].re;
        ao[1] = (double)slot_amp[s].im;
    }
    if (lane == 0) {
        out.count[inst] = count;
        out.iterations[inst] = it_run;
        out.samples_used[inst] = (long long)it_run * nl * L;
        out.terminated_by[inst] = term;
    }
    PCLK(8);
    PCLK_FLUSH();
}

#include "fpssft_team.cuh"
#include "fpssft_synth.cuh"

// ------------------------------------------------------------ re-synthesis
// x(n) = sum_i a_i exp(+2 pi j sum_k n_k m_ik / N_k) on the full grid of
// every instance (config 5's "inverse-synthesise each image"; the dense
// equivalent of SyntheticSource.sample_many, core.py:176-217, with the same
// exact integer-phase root table).  One CTA per instance; the grid is
// produced RC rows (last dimension = row) at a time:
//   V[r][m_last] = sum over entries with that m_last (in entry order) of
//                  a * root_L[sum_{k<D-1} c_k n_k m_k mod L]   (sparse part)
//   row = inverse FFT of V[r] along the last dimension        (dense part)
// and each finished row is written once, coalesced: the kernel is bound by
// the HBM write of the grid.
// Compile-time variant for 2-D grids with NL-point rows (config 5: 512 x 512):
// RC rows per chunk, compile-time padded FFT (fft_static), NT threads.
template <class R, int NL, int RC, int NT>
__global__ void __launch_bounds__(NT) synth_static_kernel(const int *__restrict__ freqs,
                                                          const double *__restrict__ amps,
                                                          const int *__restrict__ counts,
                                                          int k_cap, Geo gc, float2 *out,
                                                          long long out_stride) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int L = gc.L, N0 = gc.N[0], c0 = gc.cof[0];
    const int tid = threadIdx.x;
    const long long inst = blockIdx.x;
    const int n = min(counts[inst], k_cap);
    constexpr int VROW = NL + NL / 16 + 1;  // padded row stride (padi layout)
    size_t o = 0;
    cpx<R> *V = (cpx<R> *)(sm + o);       o = align16(o + (size_t)RC * VROW * sizeof(cpx<R>));
    cpx<R> *rootsL = (cpx<R> *)(sm + o);  o = align16(o + (size_t)L * sizeof(cpx<R>));
    cpx<R> *rootsN = (cpx<R> *)(sm + o);  o = align16(o + (size_t)NL * sizeof(cpx<R>));
    cpx<R> *eamp = (cpx<R> *)(sm + o);    o = align16(o + (size_t)k_cap * sizeof(cpx<R>));
    int *em0 = (int *)(sm + o);           o = align16(o + (size_t)k_cap * 4);
    int *col_start = (int *)(sm + o);     o = align16(o + (size_t)(NL + 1) * 4);
    int *col_fill = (int *)(sm + o);      o = align16(o + (size_t)NL * 4);
    int *order = (int *)(sm + o);         o = align16(o + (size_t)k_cap * 4);
    int *active = (int *)(sm + o);        o = align16(o + (size_t)NL * 4);
    int *ired = (int *)(sm + o);

    build_roots(rootsL, L);
    build_roots(rootsN, NL);
    for (int c = tid; c < NL; c += NT) col_fill[c] = 0;
    __syncthreads();
    for (int e = tid; e < n; e += NT) {
        const long long src = inst * k_cap + e;
        em0[e] = freqs[src * 2];
        eamp[e] = {(R)amps[src * 2], (R)amps[src * 2 + 1]};
        atomicAdd(&col_fill[freqs[src * 2 + 1]], 1);
    }
    __syncthreads();
    // column -> entry ranges, and the list of non-empty columns (ascending)
    int carry = 0, n_active = 0;
    for (int j0 = 0; j0 < NL; j0 += NT) {
        const int c = j0 + tid;
        const int cnt = c < NL ? col_fill[c] : 0;
        int tot;
        const int pre = block_exscan(cnt | ((cnt > 0) << 16), ired, &tot);
        if (c < NL) {
            col_start[c] = carry + (pre & 0xFFFF);
            col_fill[c] = 0;
            if (cnt) active[n_active + (pre >> 16)] = c;
        }
        carry += tot & 0xFFFF;
        n_active += tot >> 16;
    }
    if (tid == 0) col_start[NL] = carry;
    __syncthreads();
    for (int e = tid; e < n; e += NT) {
        const int c = freqs[(inst * k_cap + e) * 2 + 1];
        order[col_start[c] + atomicAdd(&col_fill[c], 1)] = e;
    }
    __syncthreads();
    for (int c = tid; c < NL; c += NT) {  // entry order inside a column: deterministic sums
        const int st = col_start[c], en = col_start[c + 1];
        for (int i = st + 1; i < en; ++i) {
            const int v = order[i];
            int j = i - 1;
            while (j >= st && order[j] > v) {
                order[j + 1] = order[j];
                --j;
            }
            order[j + 1] = v;
        }
    }
    __syncthreads();

    float2 *img = out + inst * out_stride;
    const R scale = (R)NL;
    const unsigned long long magicL = ~0ULL / (unsigned)L + 1ULL;
    constexpr int NW = NT / 32, RW = RC / NW;  // rows per warp in the FFT phase
    static_assert(!FPSSFT_SYNTH_WARPFFT || RC % NW == 0, "whole rows per warp");
    const int warp = tid >> 5, lane = tid & 31;
    if (FPSSFT_SYNTH_WARPFFT)
        for (int q = tid; q < RC * VROW; q += NT) V[q] = {(R)0, (R)0};
    for (int r0 = 0; r0 < N0; r0 += RC) {
        if (!FPSSFT_SYNTH_WARPFFT)
            for (int q = tid; q < RC * VROW; q += NT) V[q] = {(R)0, (R)0};
        __syncthreads();
        // sparse part: one thread per non-empty column, all RC rows of the
        // chunk, entries in order; phase c0 n0 m0 mod L advanced by c0 m0 per row
        for (int a = tid; a < n_active; a += NT) {
            const int c = active[a];
            cpx<R> acc[RC];
#pragma unroll
            for (int r = 0; r < RC; ++r) acc[r] = {(R)0, (R)0};
            for (int p = col_start[c]; p < col_start[c + 1]; ++p) {
                const int e = order[p];
                const unsigned m0 = (unsigned)em0[e];
                const cpx<R> am = eamp[e];
                const unsigned step = fastmod((unsigned)c0 * m0, magicL, (unsigned)L);
                unsigned u = fastmod((unsigned)c0 * (unsigned)r0 % (unsigned)L * m0, magicL,
                                     (unsigned)L);
#pragma unroll
                for (int r = 0; r < RC; ++r) {
                    acc[r] = acc[r] + am * rootsL[u];
                    u += step;
                    if (u >= (unsigned)L) u -= (unsigned)L;
                }
            }
#pragma unroll
            for (int r = 0; r < RC; ++r) V[padi<true>(r * NL + c)] = {acc[r].re, -acc[r].im};
        }
        __syncthreads();
        if constexpr (FPSSFT_SYNTH_WARPFFT) {
            // each warp transforms, writes and re-zeroes its own RW rows: the
            // only block barriers left are around the sparse phase
            cpx<R> *Vw = V + warp * RW * (NL + NL / 16);
            fft_static<R, NL, RW, 32, WarpTeam>(Vw, rootsN, lane);
            float2 *iw = img + (long long)(r0 + warp * RW) * NL;
#pragma unroll 4
            for (int q = lane; q < RW * NL; q += 32) {
                const cpx<R> x = Vw[padi<true>(q)];
                iw[q] = make_float2((float)(x.re * scale), (float)(-x.im * scale));
                Vw[padi<true>(q)] = {(R)0, (R)0};
            }
        } else {
            fft_static<R, NL, RC, NT, BlockTeam>(V, rootsN, tid);
#pragma unroll 4
            for (int q = tid; q < RC * NL; q += NT) {
                const cpx<R> x = V[padi<true>(q)];
                img[(long long)r0 * NL + q] =
                    make_float2((float)(x.re * scale), (float)(-x.im * scale));
            }
        }
        __syncthreads();
    }
}

template <class R>
__global__ void __launch_bounds__(256) synth_kernel(const int *__restrict__ freqs,
                                                    const double *__restrict__ amps,
                                                    const int *__restrict__ counts, int k_cap,
                                                    Geo gc, Geo gr, int rc, float2 *out,
                                                    long long out_stride) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int D = gc.D, L = gc.L, NL = gr.L;  // NL = N_{D-1} (row length)
    const int tid = threadIdx.x, NT = blockDim.x;
    const long long inst = blockIdx.x;
    const int n = min(counts[inst], k_cap);
    long long rows = 1;  // product of all but the last extent
    for (int k = 0; k < D - 1; ++k) rows *= gc.N[k];
    size_t o = 0;
    cpx<R> *V = (cpx<R> *)(sm + o);          o = align16(o + (size_t)rc * NL * sizeof(cpx<R>));
    cpx<R> *rootsL = (cpx<R> *)(sm + o);     o = align16(o + (size_t)L * sizeof(cpx<R>));
    cpx<R> *rootsN = (cpx<R> *)(sm + o);     o = align16(o + (size_t)NL * sizeof(cpx<R>));
    cpx<R> *eamp = (cpx<R> *)(sm + o);       o = align16(o + (size_t)k_cap * sizeof(cpx<R>));
    int *ekey = (int *)(sm + o);             o = align16(o + (size_t)k_cap * 4 * MAXD);
    int *col_start = (int *)(sm + o);        o = align16(o + (size_t)(NL + 1) * 4);
    int *col_fill = (int *)(sm + o);         o = align16(o + (size_t)NL * 4);
    int *order = (int *)(sm + o);            o = align16(o + (size_t)k_cap * 4);
    int *ired = (int *)(sm + o);

    build_roots(rootsL, L);
    build_roots(rootsN, NL);
    for (int c = tid; c < NL; c += NT) col_fill[c] = 0;
    __syncthreads();
    for (int e = tid; e < n; e += NT) {
        const long long src = inst * k_cap + e;
#pragma unroll
        for (int k = 0; k < MAXD; ++k) ekey[e * MAXD + k] = k < D ? freqs[src * D + k] : 0;
        eamp[e] = {(R)amps[src * 2], (R)amps[src * 2 + 1]};
        atomicAdd(&col_fill[freqs[src * D + D - 1]], 1);
    }
    __syncthreads();
    int carry = 0;
    for (int c0 = 0; c0 < NL; c0 += NT) {  // columns -> entry ranges
        const int c = c0 + tid;
        int tot;
        const int pre = block_exscan(c < NL ? col_fill[c] : 0, ired, &tot);
        if (c < NL) {
            col_start[c] = carry + pre;
            col_fill[c] = 0;
        }
        carry += tot;
    }
    if (tid == 0) col_start[NL] = carry;
    __syncthreads();
    for (int e = tid; e < n; e += NT) {
        const int c = ekey[e * MAXD + D - 1];
        order[col_start[c] + atomicAdd(&col_fill[c], 1)] = e;
    }
    __syncthreads();
    for (int c = tid; c < NL; c += NT) {  // entry order inside a column: deterministic sums
        const int st = col_start[c], en = col_start[c + 1];
        for (int i = st + 1; i < en; ++i) {
            const int v = order[i];
            int j = i - 1;
            while (j >= st && order[j] > v) {
                order[j + 1] = order[j];
                --j;
            }
            order[j + 1] = v;
        }
    }
    __syncthreads();

    float2 *img = out + inst * out_stride;
    const R scale = (R)NL;
    for (long long r0 = 0; r0 < rows; r0 += rc) {
        const int nr = (int)min((long long)rc, rows - r0);
        // sparse part: conj(V) so that the forward FFT below yields the
        // inverse transform: IFFT(v) = conj(FFT(conj(v))) * NL
        for (int r = 0; r < nr; ++r) {
            // w_k = c_k n_k mod L for this row (uniform across the block)
            long long row = r0 + r;
            int w[MAXD] = {0, 0, 0, 0};
            for (int k = D - 2; k >= 0; --k) {
                const int nk = (int)(row % gc.N[k]);
                row /= gc.N[k];
                w[k] = (int)((long long)gc.cof[k] * nk % L);
            }
            for (int c = tid; c < NL; c += NT) {
                cpx<R> acc = {(R)0, (R)0};
                for (int p = col_start[c]; p < col_start[c + 1]; ++p) {
                    const int e = order[p];
                    int u = 0;  // each term < L * N_k; the host guards D L max N < 2^31
#pragma unroll
                    for (int k = 0; k < MAXD - 1; ++k)
                        if (k < D - 1) u += w[k] * ekey[e * MAXD + k];
                    acc = acc + eamp[e] * rootsL[u % L];
                }
                V[r * NL + c] = {acc.re, -acc.im};
            }
        }
        __syncthreads();
        fft_lines<R, BlockTeam>(V, nr, gr, rootsN, tid, NT);
        for (int q = tid; q < nr * NL; q += NT) {
            const cpx<R> x = V[q];
            img[(r0 + q / NL) * NL + q % NL] = make_float2((float)(x.re * scale),
                                                          (float)(-x.im * scale));
        }
        __syncthreads();
    }
}


// ------------------------------------------------------- per-function kernels
template <class R>
__global__ void __launch_bounds__(1024, 1) line_spectra_kernel(const float2 *__restrict__ cubes,
                                                            long long batch_stride, Geo g,
                                                            const int *__restrict__ alpha_tau,
                                                            int per_instance, cpx<R> *out) {
    extern __shared__ __align__(16) unsigned char sm[];
    cpx<R> *spec = (cpx<R> *)sm;
    cpx<R> *roots = spec + (size_t)g.nlines * g.L;
    const int inst = blockIdx.x, D = g.D;
    const int *at = alpha_tau + (per_instance ? (long long)inst * 2 * D : 0);
    int al[MAXD], ta[MAXD];
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
        al[k] = k < D ? at[k] : 0;
        ta[k] = k < D ? at[D + k] : 0;
    }
    build_roots(roots, g.L);
    if (!line_params_ok(g, al, ta)) return;
    gather_lines(spec, cubes + (long long)inst * batch_stride, g, al, ta, threadIdx.x,
                 blockDim.x);
    __syncthreads();
    fft_lines<R, BlockTeam>(spec, g.nlines, g, roots, threadIdx.x, blockDim.x);
    cpx<R> *o = out + (long long)inst * g.nlines * g.L;
    for (int e = threadIdx.x; e < g.nlines * g.L; e += blockDim.x) o[e] = spec[e];
}

template <class R>
__global__ void __launch_bounds__(1024, 1) dft_kernel(const cpx<R> *__restrict__ in, Geo g,
                                                   cpx<R> *out) {
    extern __shared__ __align__(16) unsigned char sm[];
    cpx<R> *x = (cpx<R> *)sm;
    cpx<R> *roots = x + g.L;
    const long long off = (long long)blockIdx.x * g.L;
    build_roots(roots, g.L);
    for (int l = threadIdx.x; l < g.L; l += blockDim.x) x[l] = in[off + l];
    __syncthreads();
    fft_lines<R, BlockTeam>(x, 1, g, roots, threadIdx.x, blockDim.x);
    for (int l = threadIdx.x; l < g.L; l += blockDim.x) out[off + l] = x[l];
}

// GLOBAL: the spectra stay in global memory (lines too long for shared
// memory, e.g. the 512 x 576 imaging shape, L = 4608, in float64); only the
// root table is staged.
template <class R, bool GLOBAL = false>
__global__ void __launch_bounds__(1024, 1) decode_kernel(const cpx<R> *__restrict__ spectra, Geo g,
                                                      const int *__restrict__ alpha_tau,
                                                      int per_instance, Knobs kn, double floor,
                                                      int *status, int *freqs, double *amps,
                                                      int *n_candidates,
                                                      const double *floor_dev = nullptr) {
    extern __shared__ __align__(16) unsigned char sm[];
    cpx<R> *spec = GLOBAL ? nullptr : (cpx<R> *)sm;
    cpx<R> *roots = GLOBAL ? (cpx<R> *)sm : spec + (size_t)g.nlines * g.L;
    int *ired = (int *)(roots + g.L);
    const int inst = blockIdx.x, D = g.D, L = g.L;
    const int *at = alpha_tau + (per_instance ? (long long)inst * 2 * D : 0);
    int al[MAXD], ta[MAXD];
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
        al[k] = k < D ? at[k] : 0;
        ta[k] = k < D ? at[D + k] : 0;
    }
    build_roots(roots, L);
    const cpx<R> *src = spectra + (long long)inst * g.nlines * L;
    R my_e = (R)0;
    for (int e = threadIdx.x; e < g.nlines * L; e += blockDim.x) {
        const cpx<R> v = src[e];
        if (!GLOBAL) spec[e] = v;
        my_e += v.re * v.re + v.im * v.im;
    }
    __syncthreads();
    const cpx<R> *sp = GLOBAL ? src : spec;
    R fl = (R)(floor_dev ? *floor_dev : floor);  // the device loop keeps its floor on chip
    if (sizeof(R) == 4 && kn.noise_coef > 0)  // sum |x|^2 = L sum |S|^2 (Parseval)
        fl = max(fl, (R)kn.noise_coef * sqrt((R)L * block_sum(my_e, (R *)(ired + 32))));
    int my = 0;
    for (int b = threadIdx.x; b < L; b += blockDim.x) {
        int m[MAXD] = {0, 0, 0, 0};
        cpx<R> a = {(R)0, (R)0};
        const int st = classify_bin(sp, g, b, al, ta, roots, (R)kn.mag_tol, (R)kn.round_tol,
                                    (R)kn.verify_tol, fl, m, &a);
        my += st > 0;
        const long long o = (long long)inst * L + b;
        status[o] = st;
#pragma unroll
        for (int k = 0; k < MAXD; ++k)
            if (k < D) freqs[o * D + k] = m[k];
        amps[o * 2] = (double)a.re;
        amps[o * 2 + 1] = (double)a.im;
    }
    const int tot = block_sum(my, ired);
    if (threadIdx.x == 0) n_candidates[inst] = tot;
}

template <class R>
__global__ void __launch_bounds__(1024, 1) project_kernel(const int *__restrict__ freqs,
                                                       const double *__restrict__ amps,
                                                       const int *__restrict__ counts, int k_max,
                                                       Geo g, const int *__restrict__ alpha_tau,
                                                       int per_instance, double *out) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int inst = blockIdx.x, D = g.D, L = g.L, NT = blockDim.x, tid = threadIdx.x;
    const Layout lay = make_layout(D, L, k_max, (int)sizeof(cpx<R>));
    cpx<R> *spec = (cpx<R> *)(sm + lay.spec);
    cpx<R> *roots = (cpx<R> *)(sm + lay.roots);
    cpx<R> *slot_amp = (cpx<R> *)(sm + lay.slot_amp);
    int *slot_m = (int *)(sm + lay.slot_m);
    const int *at = alpha_tau + (per_instance ? (long long)inst * 2 * D : 0);
    int al[MAXD], ta[MAXD];
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
        al[k] = k < D ? at[k] : 0;
        ta[k] = k < D ? at[D + k] : 0;
    }
    const int n = min(counts[inst], k_max);
    build_roots(roots, L);
    for (int s = tid; s < n; s += NT) {
        const long long o = (long long)inst * k_max + s;
        for (int k = 0; k < D; ++k) slot_m[s * D + k] = freqs[o * D + k];
        slot_amp[s] = {(R)amps[o * 2], (R)amps[o * 2 + 1]};
    }
    __syncthreads();
    project_bins(spec, 1, g, al, ta, n, slot_m, slot_amp, (const int *)nullptr,
                 (int *)(sm + lay.bin_start), (int *)(sm + lay.bin_fill), (int *)(sm + lay.seg),
                 (int *)(sm + lay.slot_bin), (int *)(sm + lay.slot_u0), roots,
                 (int *)(sm + lay.red), false);
    for (int b = tid; b < L; b += NT) {
        out[((long long)inst * L + b) * 2] = (double)spec[b].re;
        out[((long long)inst * L + b) * 2 + 1] = (double)spec[b].im;
    }
}

#include "fpssft_large.cuh"
#include "fpssft_loop.cuh"
#include "fpssft_stage.cuh"

// ================================================================== host
namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char *where) {
    return fail(FPSSFT_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

long long lcm_ll(long long a, long long b) { return a / std::gcd(a, b) * b; }

// Fill Geo from a shape; validates like CubeShape (core.py:33-37, :49-55).
int make_geo(const fpssft_shape *shape, Geo *g) {
    if (!shape) return fail(FPSSFT_EINVAL, "shape is NULL");
    const int D = shape->ndim;
    if (D < 1 || D > FPSSFT_MAX_DIMS)
        return fail(FPSSFT_EUNSUPPORTED, "ndim must be in [1, " + std::to_string(FPSSFT_MAX_DIMS) + "]");
    std::memset(g, 0, sizeof(*g));
    g->D = D;
    g->nlines = D + 1;
    long long L = 1, Ntot = 1, maxN = 1;
    for (int k = 0; k < D; ++k) {
        const long long n = shape->dims[k];
        if (n < 1) return fail(FPSSFT_EINVAL, "dimension lengths must be >= 1");
        L = lcm_ll(L, n);
        Ntot *= n;
        maxN = std::max(maxN, n);
        if (L >= (1LL << 31) || Ntot >= (1LL << 31))
            return fail(FPSSFT_EOVERFLOW, "line length / grid size exceeds the int32 index range");
    }
    if ((long long)D * L * maxN >= (1LL << 31))
        return fail(FPSSFT_EOVERFLOW, "D*L*max(N) exceeds the int32 phase-arithmetic range");
    g->L = (int)L;
    for (int k = 0; k < D; ++k) {
        const unsigned n = (unsigned)shape->dims[k];
        g->N[k] = (int)n;
        g->cof[k] = (int)(L / n);
        g->stride[k] = shape->strides[k];
        g->magic[k] = (n == 1) ? 0ULL : (~0ULL / n + 1ULL);
    }
    // 32-bit element offsets when the whole cube is addressable with them
    long long span = 0;
    for (int k = 0; k < D; ++k) span += (long long)(shape->dims[k] - 1) * std::llabs(shape->strides[k]);
    g->off32 = span < (1LL << 31) ? 1 : 0;
    for (int k = 0; k < D; ++k) g->stride32[k] = g->off32 ? (int)shape->strides[k] : 0;
    // packed frequency key (warp mode): bit_length(N_k - 1) bits per dim,
    // dim 0 most significant, so key order is lexicographic order
    int shift = 0;
    for (int k = D - 1; k >= 0; --k) {
        int bits = 0;
        while ((1LL << bits) < shape->dims[k]) ++bits;
        g->key_shift[k] = shift;
        g->key_mask[k] = (int)((1LL << bits) - 1);
        shift += bits;
    }
    g->key_bits_ = shift;
    return FPSSFT_OK;
}

// FFT plan for `nlines` lines of length L owned by `team` threads (32 = one
// warp per instance; 0 = one CTA per instance, size chosen here).  Radices:
// the largest power of two allowed (16 in float, 8 in double or for warp
// teams), the leftover power of two as one stage, then 3s, 5s, 7s; a
// remaining prime factor > 7 means one direct O(L^2) pass.  A stage's
// butterflies are spread MB per thread with MB*radix complex values held in
// registers (<= 16 float / 8 double); lines are transformed G at a time so
// that fits.  Returns the thread count, or -1 if no plan fits.
int plan_fft(Geo *g, int nlines, int precision, int team) {
    const int L = g->L;
    const bool dbl = precision == FPSSFT_F64;
    auto cap = [dbl](int r) {
        if (r == 0) return 4;
        if (dbl) return r <= 2 ? 4 : (r <= 4 ? 2 : 1);
        return r <= 4 ? 4 : (r <= 8 ? 2 : 1);
    };
    int x = L, e = 0;
    while (x % 2 == 0) { x /= 2; ++e; }
    int rad[MAXSTAGES], n = 0;
    if (team && x == 1) {
        // warp teams: choose how to split 2^e into radix 2..16 stages by a
        // cost model (per group step: MB butterflies of r log2 r work plus a
        // fixed sync/index overhead); stages must fit MB <= cap(r)
        const int maxbits = dbl ? 3 : 4;
        double best = 1e300;
        int best_parts[MAXSTAGES], best_n = -1;
        int parts[MAXSTAGES];
        // iterate compositions of e into parts in [1, maxbits], larger first
        std::function<void(int, int)> rec = [&](int left, int k) {
            if (k > MAXSTAGES) return;
            if (left == 0) {
                double cost = 0;
                for (int i = 0; i < k; ++i) {
                    const int r = 1 << parts[i];
                    const long long m = L / r;
                    const long long G = std::max(1LL, std::min<long long>(nlines, cap(r) * team / m));
                    const long long mb = (G * m + team - 1) / team;
                    if (mb > cap(r)) return;
                    const long long groups = (nlines + G - 1) / G;
                    cost += groups * (mb * r * parts[i] + 24.0);
                }
                if (cost < best) {
                    best = cost;
                    best_n = k;
                    for (int i = 0; i < k; ++i) best_parts[i] = parts[i];
                }
                return;
            }
            for (int b = std::min(maxbits, left); b >= 1; --b) {
                parts[k] = b;
                rec(left - b, k + 1);
            }
        };
        rec(e, 0);
        if (best_n < 0) return -1;
        for (int i = 0; i < best_n; ++i) rad[n++] = 1 << best_parts[i];
    } else {
        const int big = (dbl || team) ? 3 : 4;
        while (e >= big) {
            if (n == MAXSTAGES) return -1;
            rad[n++] = 1 << big;
            e -= big;
        }
        if (e > 0) rad[n++] = 1 << e;
    }
    for (int p : {3, 5, 7})
        while (x % p == 0) {
            if (n == MAXSTAGES) return -1;
            rad[n++] = p;
            x /= p;
        }
    if (x != 1) {  // not 7-smooth
        n = 1;
        rad[0] = 0;
    }
    if (L == 1) n = 0;
    long long nt = team;
    if (!team) {
        nt = std::max(64, std::min(((L + 31) / 32) * 32, 1024));
        for (int i = 0; i < n; ++i) {
            const long long tot = (long long)nlines * (rad[i] ? L / rad[i] : L);
            const long long need = (tot + cap(rad[i]) - 1) / cap(rad[i]);
            nt = std::max(nt, ((need + 31) / 32) * 32);
        }
        if (nt > 1024) return -1;
    }
    g->nstages = n;
    g->plan[0] = g->plan[1] = g->plan[2] = g->plan[3] = 0;
    for (int i = 0; i < n; ++i) {
        const long long m = rad[i] ? L / rad[i] : L;  // butterflies per line
        long long G = team ? std::max(1LL, std::min<long long>(nlines, cap(rad[i]) * nt / m))
                           : nlines;
        G = std::min<long long>(G, 255);  // 8-bit field
        long long mb = (G * m + nt - 1) / nt;
        if (mb > cap(rad[i])) return -1;
        mb = mb <= 1 ? 1 : (mb <= 2 ? 2 : 4);
        const unsigned long long code =
            (unsigned long long)(rad[i] | (mb << 5) | (G << 8));
        g->plan[i >> 2] |= code << (16 * (i & 3));
    }
    g->threads = (int)nt;
    return (int)nt;
}

int block_threads(Geo &g, int nlines, int precision) {
    return plan_fft(&g, nlines, precision, 0);
}

int max_smem_optin() {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
        v = 227 * 1024;
    return v;
}

int make_knobs(const fpssft_params *p, Knobs *k) {
    if (!p) return fail(FPSSFT_EINVAL, "params is NULL");
    if (p->t_max < 1) return fail(FPSSFT_EINVAL, "max_iterations must be >= 1");
    if (p->stall_limit < 1) return fail(FPSSFT_EINVAL, "stall_limit must be >= 1");
    if (p->k_cap < 1 || (p->k_cap & (p->k_cap - 1)))
        return fail(FPSSFT_EINVAL, "k_cap must be a positive power of two");
    const double v[] = {p->mag_tol, p->verify_tol, p->round_tol, p->amp_prune_tol,
                        p->energy_floor, p->energy_floor_abs, p->residual_stop};
    const char *names[] = {"mag_tol", "verify_tol", "round_tol", "amp_prune_tol",
                           "energy_floor", "energy_floor_abs", "residual_stop"};
    for (int i = 0; i < 7; ++i)
        if (!(v[i] > 0)) return fail(FPSSFT_EINVAL, std::string(names[i]) + " must be positive");
    if (p->precision != FPSSFT_F32 && p->precision != FPSSFT_F64 &&
        p->precision != FPSSFT_F32_GUARDED)
        return fail(FPSSFT_EINVAL, "precision must be FPSSFT_F32, FPSSFT_F64 or FPSSFT_F32_GUARDED");
    if (p->mode < FPSSFT_MODE_AUTO || p->mode > FPSSFT_MODE_WARP)
        return fail(FPSSFT_EINVAL, "mode must be FPSSFT_MODE_AUTO, _CTA or _WARP");
    k->mag_tol = p->mag_tol;
    k->verify_tol = p->verify_tol;
    k->round_tol = p->round_tol;
    k->amp_prune_tol = p->amp_prune_tol;
    k->energy_floor = p->energy_floor;
    k->energy_floor_abs = p->energy_floor_abs;
    k->residual_stop = p->residual_stop;
    k->noise_coef = 0.0;
    k->guard_coef = 0.0;
    k->t_max = p->t_max;
    k->stall_limit = p->stall_limit;
    k->k_cap = p->k_cap;
    k->group = 1;
    k->staged = nullptr;
    k->staged_group_stride = 0;
    k->stage_T = 0;
    return FPSSFT_OK;
}

// Float32 rounding floor ("precision floor"): a length-L
// transform's per-bin error is ~ eps sqrt(log2 L + 1) ||x_line|| / L; bins
// below kappa times that are treated as empty.  Zero in float64 mode, where
// the reference's own floors are far above the rounding level.
// Guarded float32 (fpssft_guard.cuh): no rounding floor (the guard band
// re-evaluates what float32 cannot resolve); the transform part of the error
// bound is guard_coef * sqrt(sum |x|^2 over the D+1 lines).
void set_noise_floor(Knobs *k, const Geo &g, int precision) {
    const double kappa = 8.0, eps32 = 5.9604644775390625e-08;
    const double unit = eps32 * std::sqrt(std::log2((double)g.L) + 1.0) / (double)g.L;
    k->noise_coef = precision == FPSSFT_F32 ? kappa * unit / std::sqrt((double)g.nlines) : 0.0;
    k->guard_coef = precision == FPSSFT_F32_GUARDED ? GUARD_KF * unit : 0.0;
}

int check_launch(const char *where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, where);
    return FPSSFT_OK;
}

// The warp kernel instance for a shape: compile-time specialisations for the
// benchmark shapes, else the runtime-shape version.
template <class R>
const void *warp_kernel_for_t(const Geo &g, int k_cap) {
    if (g.off32 && g.D == 2 && g.L == 256 && k_cap == 128 && sizeof(R) == 4)  // config 2
        return (const void *)recover_warp_kernel<R, 256, 2, false, 0, 128>;
    if (g.off32 && g.D == 2 && g.L == 256) return (const void *)recover_warp_kernel<R, 256, 2>;
    if (g.off32 && g.D == 2 && g.L == 512) return (const void *)recover_warp_kernel<R, 512, 2>;
    if (g.off32 && g.D == 3 && g.L == 64) return (const void *)recover_warp_kernel<R, 64, 3>;
    return (const void *)recover_warp_kernel<R, 0, 0>;
}
// stg: the instances that read staged lines (float32 / guarded; nullptr: none)
const void *warp_kernel_for(const Geo &g, int precision, int k_cap, bool stg = false) {
    if (stg) {
        if (!g.off32 || precision == FPSSFT_F64) return nullptr;
        if (precision == FPSSFT_F32_GUARDED)
            return g.D == 3 && g.L == 64
                       ? (const void *)recover_warp_kernel<float, 64, 3, true, 0, 0, true>
                       : nullptr;
        if (g.D == 2 && g.L == 256)
            return (const void *)recover_warp_kernel<float, 256, 2, false, 0, 0, true>;
        if (g.D == 3 && g.L == 64)
            return (const void *)recover_warp_kernel<float, 64, 3, false, 0, 0, true>;
        return (const void *)recover_warp_kernel<float, 0, 0, false, 0, 0, true>;
    }
    if (precision == FPSSFT_F32_GUARDED)  // guarded float32: the noisy config-3 shape
        return g.off32 && g.D == 3 && g.L == 64
                   ? (const void *)recover_warp_kernel<float, 64, 3, true>
                   : nullptr;
    return precision == FPSSFT_F64 ? warp_kernel_for_t<double>(g, k_cap)
                                   : warp_kernel_for_t<float>(g, k_cap);
}

// The compile-time team kernel for a shape (one CTA of *nt threads per
// instance), or nullptr if the shape has none.
template <class R>
const void *team_kernel_for_t(const Geo &g, int *nt) {
    if (!g.off32) return nullptr;
    if (g.D == 3 && g.L == 64) {  // config 3: small batches leave SMs idle in warp mode
        if (*nt == 64) return (const void *)recover_team_kernel<R, 64, 3, 64>;
        *nt = 128;
        return (const void *)recover_team_kernel<R, 64, 3, 128>;
    }
    if (g.D != 2) return nullptr;
    if (g.L == 2048) {
        if (*nt == 512) return (const void *)recover_team_kernel<R, 2048, 2, 512>;
        *nt = 1024;
        return (const void *)recover_team_kernel<R, 2048, 2, 1024>;
    }
    if (g.L == 512) {
        *nt = 128;
        return (const void *)recover_team_kernel<R, 512, 2, 128>;
    }
#if FPSSFT_TEAM256
    if (g.L == 256) {  // A/B: small batches of 256-point lines, several warps per instance
        if (*nt == 64) return (const void *)recover_team_kernel<R, 256, 2, 64>;
        *nt = 128;
        return (const void *)recover_team_kernel<R, 256, 2, 128>;
    }
#endif
    return nullptr;
}
// Guarded float32 team kernels (fpssft_guard.cuh): the shapes of the noisy
// configs (3: 64^3, 5: 512 x 512).
const void *team_guard_kernel_for(const Geo &g, int *nt) {
    if (!g.off32) return nullptr;
    if (g.D == 2 && g.L == 512) {
        *nt = 128;
        return (const void *)recover_team_kernel<float, 512, 2, 128, true>;
    }
    if (g.D == 3 && g.L == 64) {
        *nt = 128;
        return (const void *)recover_team_kernel<float, 64, 3, 128, true>;
    }
    return nullptr;
}
const void *team_kernel_for(const Geo &g, int precision, int *nt, bool stg = false) {
    if (stg) {  // the float32 instances that read staged lines (configs 4 and 5's shapes)
        if (!g.off32 || precision != FPSSFT_F32 || g.D != 2) return nullptr;
        if (g.L == 2048 && (*nt == 512 || *nt == 0)) {
            *nt = 512;
            return (const void *)recover_team_kernel<float, 2048, 2, 512, false, true>;
        }
        if (g.L == 512) {
            *nt = 128;
            return (const void *)recover_team_kernel<float, 512, 2, 128, false, true>;
        }
        return nullptr;
    }
    if (precision == FPSSFT_F32_GUARDED) return team_guard_kernel_for(g, nt);
    return precision == FPSSFT_F64 ? team_kernel_for_t<double>(g, nt)
                                   : team_kernel_for_t<float>(g, nt);
}

int kernel_regs(const void *fn, int fallback) {
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, fn) == cudaSuccess && fa.numRegs > 0) return fa.numRegs;
    cudaGetLastError();  // no device: clear the error, assume the cap
    return fallback;
}

constexpr long long SMEM_PER_SM = 228 * 1024;    // B200 shared memory per SM
constexpr long long SMEM_PER_CTA = 227 * 1024;   // opt-in limit per CTA
constexpr long long SMEM_RESERVED = 1024;        // per-CTA system reservation

struct LaunchPlan {
    int mode, threads, per_cta;
    size_t smem;
    const void *kernel;  // nullptr: generic recover_kernel / recover_warp_kernel<R,0,0>
};

// Pick the kernel for a shape: warp-per-instance when the lines are short
// enough ((D+1) L <= 2048), the packed key fits 31 bits and the per-warp state
// fits; warps per CTA chosen to maximise resident instances per SM.  Else one
// CTA per instance.  `g` receives the FFT plan of the chosen mode.
// Registers per thread of the warp kernel chosen for (precision, L, D): the
// compiled value when a device is present, else the launch-bounds cap.
int warp_kernel_regs(const Geo &g, int precision, int k_cap, bool stg = false) {
    cudaFuncAttributes fa;
    const void *k = warp_kernel_for(g, precision, k_cap, stg);
    if (k && cudaFuncGetAttributes(&fa, k) == cudaSuccess &&
        fa.numRegs > 0)
        return fa.numRegs;
    cudaGetLastError();  // no device: clear the error, assume the cap
    return precision == FPSSFT_F64 ? 128 : 80;
}

// The group-gather warp kernel (GroupGather: WG warps of one CTA own WG
// consecutive members of an interleave group and gather their shared lines
// once): float32, a compile-time shape, a batch stored interleaved with
// kn.group a multiple of WG, and one schedule for the whole batch.
#ifndef FPSSFT_GROUP_WG
#define FPSSFT_GROUP_WG 8  // warps (= interleaved instances) per group-gather CTA; 0 = off
#endif
#ifndef FPSSFT_GROUP_TEAM
#define FPSSFT_GROUP_TEAM FPSSFT_GROUP_WG  // warps per gather team (a divisor of the CTA width)
#endif
#ifndef FPSSFT_GROUP_WIDE
#define FPSSFT_GROUP_WIDE 16  // a second group kernel for groups of this many (one CTA of 16
                              // warps: a 128-byte read per sample position); 0 = off
#endif
// The group kernel for an interleave group of `group` instances, and its CTA
// width in warps (*wg): 16-wide when the group is a multiple of 16 (one
// 128-byte read per position serves 16 instances: the host-memory path's
// request economy, tools/zc_group_probe.py), else 8-wide.
// (narrow: the 8-wide kernel whatever the group -- staged lines come from HBM,
// where it is the faster one.)
const void *group_kernel_for(const Geo &g, int precision, int group, int k_cap, int *wg = nullptr,
                             bool narrow = false) {
    if (!FPSSFT_GROUP_WG || precision != FPSSFT_F32 || !g.off32 || group < FPSSFT_GROUP_WG ||
        group % FPSSFT_GROUP_WG)
        return nullptr;
#if FPSSFT_GROUP_WG
    if (g.D == 2 && g.L == 256) {
#if FPSSFT_GROUP_WIDE
        if (group % FPSSFT_GROUP_WIDE == 0 && !narrow) {
            if (wg) *wg = FPSSFT_GROUP_WIDE;
            return k_cap == 128
                       ? (const void *)recover_warp_kernel<float, 256, 2, false, FPSSFT_GROUP_WIDE, 128>
                       : (const void *)recover_warp_kernel<float, 256, 2, false, FPSSFT_GROUP_WIDE>;
        }
#endif
        if (wg) *wg = FPSSFT_GROUP_WG;
        if (narrow)  // the instances that read staged lines
            return k_cap == 128
                       ? (const void *)recover_warp_kernel<float, 256, 2, false, FPSSFT_GROUP_TEAM, 128, true>
                       : (const void *)recover_warp_kernel<float, 256, 2, false, FPSSFT_GROUP_TEAM, 0, true>;
        return k_cap == 128 ? (const void *)recover_warp_kernel<float, 256, 2, false, FPSSFT_GROUP_TEAM, 128>
                            : (const void *)recover_warp_kernel<float, 256, 2, false, FPSSFT_GROUP_TEAM>;
    }
#endif
    return nullptr;
}

int make_plan(Geo &g, const Knobs &kn, int precision, int want, LaunchPlan *lp,
              bool shared_sched = false) {
    const int cs = precision == FPSSFT_F64 ? 16 : 8;
    const bool guard = precision == FPSSFT_F32_GUARDED;
    const bool stg = kn.staged != nullptr;  // the instances that read staged lines
    // candidate 1: warp per instance
    long long warp_warps = 0;
    LaunchPlan wp{};
    Geo gw = g;
    if (want != FPSSFT_MODE_CTA) {
        bool ok = g.key_bits_ <= 31 && kn.k_cap <= 32768 && (long long)g.nlines * g.L <= 2048 &&
                  (g.L & (g.L - 1)) == 0 && plan_fft(&gw, g.nlines, precision, 32) > 0 &&
                  (!(guard || stg) || warp_kernel_for(g, precision, kn.k_cap, stg) != nullptr);
        if (ok) {
            const WarpLayout wl = make_warp_layout(g.D, g.L, kn.k_cap, cs, guard);
            const int regs = (warp_kernel_regs(gw, precision, kn.k_cap, stg) + 7) / 8 * 8;
            const long long reg_warps = 65536 / (regs * 32);
            int best_w = 0;
            for (int w : {8, 7, 6, 5, 4, 3, 2, 1}) {
                if (32 * w > FPSSFT_WARP_NT) continue;
                if (FPSSFT_WARP_W && w != FPSSFT_WARP_W) continue;  // compile-time A/B
                const long long smem = (long long)wl.roots + w * (long long)wl.per_warp;
                if (smem > SMEM_PER_CTA) continue;
                const long long ctas = std::min<long long>(
                    {32, SMEM_PER_SM / (smem + SMEM_RESERVED), 64 / w, reg_warps / w});
                if (ctas * w > warp_warps) {
                    warp_warps = ctas * w;
                    best_w = w;
                }
            }
            if (best_w)
                wp = LaunchPlan{FPSSFT_MODE_WARP, 32 * best_w, best_w,
                                wl.roots + (size_t)best_w * wl.per_warp,
                                warp_kernel_for(gw, precision, kn.k_cap, stg)};
            int gwd = FPSSFT_GROUP_WG;
            const void *gk =
                shared_sched ? group_kernel_for(gw, precision, kn.group, kn.k_cap, &gwd,
                                               kn.staged != nullptr)
                             : nullptr;
            if (best_w && gk) {
                const WarpLayout gl = make_warp_layout(g.D, g.L, kn.k_cap, cs, false, true);
                const size_t smem = gl.roots + (size_t)gwd * gl.per_warp;
                if ((long long)smem <= SMEM_PER_CTA)
                    wp = LaunchPlan{FPSSFT_MODE_WARP, 32 * gwd, gwd, smem, gk};
            }
        }
        if (want == FPSSFT_MODE_WARP) {
            if (!warp_warps)
                return fail(FPSSFT_EUNSUPPORTED,
                            "shape/k_cap does not fit the warp-per-instance kernel");
            g = gw;
            *lp = wp;
            return FPSSFT_OK;
        }
    }
    // candidate 2: compile-time team kernel (one CTA per instance); among
    // its CTA sizes take the one with the most resident instances; on a tie
    // the smaller CTA (more registers per thread: measured faster on config
    // 4, 0.588 vs 0.618 ms)
    long long team_warps = 0, team_inst = 0;
    LaunchPlan tp{};
    if (g.key_bits_ <= 31 && kn.k_cap <= 32768) {
        for (int want_nt : {512, 0}) {
            if (FPSSFT_TEAM_NT && want_nt) continue;  // compile-time A/B: one pass at that size
            const int req = FPSSFT_TEAM_NT ? FPSSFT_TEAM_NT : want_nt;
            int tnt = req;
            const void *tk = team_kernel_for(g, precision, &tnt, stg);
            if (!tk || (req && tnt != req)) continue;
            const TeamLayout tl = make_team_layout(g.D, g.L, kn.k_cap, cs, tnt, guard);
            if ((long long)tl.total > SMEM_PER_CTA) continue;
            const int regs = (kernel_regs(tk, tnt >= 1024 ? 64 : 128) + 7) / 8 * 8;
            const long long ctas = std::min<long long>(
                {32, SMEM_PER_SM / ((long long)tl.total + SMEM_RESERVED), 2048 / tnt,
                 65536 / ((long long)regs * tnt)});
            if (ctas < 1) continue;
            const long long warps = ctas * tnt / 32;
            if (ctas > team_inst) {
                team_inst = ctas;
                team_warps = warps;
                tp = LaunchPlan{FPSSFT_MODE_CTA, tnt, 1, tl.total, tk};
            }
        }
    }
    // warp mode unless it keeps too few warps resident and the team kernel
    // does clearly better
    if (warp_warps && !(team_warps && warp_warps < 16 && team_warps * 2 > warp_warps * 3)) {
        g = gw;
        *lp = wp;
        return FPSSFT_OK;
    }
    if (team_warps) {
        *lp = tp;
        return FPSSFT_OK;
    }
    if (guard)  // no guarded kernel for this shape: the caller runs float64
        return fail(FPSSFT_EUNSUPPORTED, "no guarded float32 kernel for this shape");
    const int nt = plan_fft(&g, g.nlines, precision, 0);
    if (nt < 0) return fail(FPSSFT_EUNSUPPORTED, "line length too large for one CTA");
    const Layout lay = make_layout(g.D, g.L, kn.k_cap, cs);
    if ((long long)lay.total > SMEM_PER_CTA)
        return fail(FPSSFT_EUNSUPPORTED,
                    "shared memory for this (shape, k_cap, precision) is " +
                        std::to_string(lay.total) + " B, above the per-CTA limit; lower k_cap");
    *lp = LaunchPlan{FPSSFT_MODE_CTA, nt, 1, lay.total, nullptr};
    return FPSSFT_OK;
}

// Shared-memory carveout for a launch: only as much of the SM's unified
// L1/shared memory as the CTAs that will actually be co-resident need, the
// rest stays L1.  The line gathers are random 8-byte reads whose in-flight
// misses live in L1: config 3 (128 CTAs, one per SM) runs 1.30 ms with the
// driver's default 228 KB carveout (28 KB of L1) and 1.07 ms with 132 KB.
void set_carveout(const void *kernel, long long grid, int threads, size_t smem) {
    int dev = 0, sms = 0, occ = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem) != cudaSuccess ||
        sms <= 0 || occ <= 0) {
        cudaGetLastError();
        return;
    }
    const long long per_sm = std::min<long long>(occ, (grid + sms - 1) / sms);
    const long long need = per_sm * ((long long)smem + SMEM_RESERVED);
    const int pct = (int)std::min<long long>(100, (need * 100 + SMEM_PER_SM - 1) / SMEM_PER_SM);
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaGetLastError();  // a hint: never an error
}

// The arithmetic a launch really uses: FPSSFT_F32_GUARDED falls back to the
// float64 kernels (exact decisions too) for shapes without a guarded kernel.
int effective_precision(const Geo &g, const Knobs &kn, int precision, int mode) {
    if (precision != FPSSFT_F32_GUARDED) return precision;
    Geo gg = g;
    LaunchPlan lp;
    if (make_plan(gg, kn, precision, mode, &lp) == FPSSFT_OK) return precision;
    return FPSSFT_F64;
}

template <class R>
int run_batch_t(const void *cubes, int64_t batch, int64_t batch_stride, Geo g,
                const Knobs &kn, int want_mode, const int32_t *schedule,
                const int32_t *sched_index, int32_t n_sched, const OutPtrs &o, cudaStream_t st) {
    LaunchPlan lp;
    const int prec = sizeof(R) == 8 ? FPSSFT_F64
                                    : (kn.guard_coef > 0 ? FPSSFT_F32_GUARDED : FPSSFT_F32);
    int rc = make_plan(g, kn, prec, want_mode, &lp, sched_index == nullptr);
    if (rc != FPSSFT_OK) return rc;
    cudaError_t e;
    if (lp.mode == FPSSFT_MODE_CTA && lp.kernel) {  // compile-time team kernel
        auto kernel = (void (*)(const float2 *, long long, Geo, Knobs, const int *, const int *,
                                int, OutPtrs))lp.kernel;
        e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)lp.smem);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(recover_team_kernel)");
        if (batch == 0) return FPSSFT_OK;
        set_carveout((const void *)kernel, batch, lp.threads, lp.smem);
        kernel<<<(unsigned)batch, lp.threads, lp.smem, st>>>(
            (const float2 *)cubes, (long long)batch_stride, g, kn, schedule, sched_index, n_sched,
            o);
        return check_launch("recover_team_kernel");
    }
    if (lp.mode == FPSSFT_MODE_WARP) {
        // a batch smaller than one CTA per SM: fewer instances per CTA so the
        // CTAs cover every SM (config 3: 1024 instances, 7 per CTA on 147 SMs
        // instead of 8 on 128 -- 0.961 -> 0.934 ms).  The group-gather kernel
        // keeps its fixed width (its CTA is one interleave group's share).
        int sms = 0, dev = 0;
        if (lp.per_cta > 1 && lp.threads == 32 * lp.per_cta && cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess &&
            sms > 0 &&
            lp.kernel != group_kernel_for(g, prec, kn.group, kn.k_cap, nullptr,
                                          kn.staged != nullptr)) {
            const long long want = (batch + sms - 1) / sms;
            if (want < lp.per_cta) {
                const WarpLayout wl = make_warp_layout(g.D, g.L, kn.k_cap, sizeof(R) == 8 ? 16 : 8,
                                                       prec == FPSSFT_F32_GUARDED);
                lp.per_cta = (int)std::max(1LL, want);
                lp.threads = 32 * lp.per_cta;
                lp.smem = wl.roots + (size_t)lp.per_cta * wl.per_warp;
            }
        }
        cudaGetLastError();
        auto kernel = (void (*)(const float2 *, long long, long long, Geo, Knobs, const int *,
                                const int *, int, OutPtrs))lp.kernel;
        e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)lp.smem);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(recover_warp_kernel)");
        if (batch == 0) return FPSSFT_OK;
        const long long grid = (batch + lp.per_cta - 1) / lp.per_cta;
        set_carveout((const void *)kernel, grid, lp.threads, lp.smem);
        kernel<<<(unsigned)grid, lp.threads, lp.smem, st>>>(
            (const float2 *)cubes, (long long)batch, (long long)batch_stride, g, kn, schedule,
            sched_index, n_sched, o);
        return check_launch("recover_warp_kernel");
    }
    e = cudaFuncSetAttribute(recover_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)lp.smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(recover_kernel)");
    if (batch == 0) return FPSSFT_OK;
    set_carveout((const void *)recover_kernel<R>, batch, lp.threads, lp.smem);
    recover_kernel<R><<<(unsigned)batch, lp.threads, lp.smem, st>>>(
        (const float2 *)cubes, (long long)batch_stride, g, kn, schedule, sched_index, n_sched, o);
    return check_launch("recover_kernel");
}

size_t spec_smem(const Geo &g, int nlines, int cs) {
    return align16((size_t)(nlines + 1) * g.L * cs) + 64 * 8;
}

// The classifier launch shared by fpssft_decode_spectra and the device loop
// (floor_dev: the energy floor read on the device, else `floor`).
int launch_decode(const void *spectra, int64_t batch, Geo g, const Knobs &kn,
                  int precision, const int32_t *alpha_tau, int per_instance, double floor,
                  const double *floor_dev, int32_t *status, int32_t *freqs, double *amps,
                  int32_t *n_candidates, cudaStream_t st) {
    cudaError_t e;
    const int cs = precision == FPSSFT_F64 ? 16 : 8;
    const int nt = block_threads(g, g.nlines, precision);
    if (nt < 0 || (long long)spec_smem(g, g.nlines, cs) > max_smem_optin()) {
        // long lines: classify straight from global memory, roots on chip
        const size_t sm = align16((size_t)g.L * cs) + 64 * 8;
        if ((long long)sm > max_smem_optin()) return fail(FPSSFT_EUNSUPPORTED, "L too large");
        if (precision == FPSSFT_F64) {
            e = cudaFuncSetAttribute(decode_kernel<double, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
            decode_kernel<double, true><<<(unsigned)batch, 1024, sm, st>>>(
                (const cpx<double> *)spectra, g, alpha_tau, per_instance, kn, floor, status,
                freqs, amps, n_candidates, floor_dev);
        } else {
            e = cudaFuncSetAttribute(decode_kernel<float, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
            decode_kernel<float, true><<<(unsigned)batch, 1024, sm, st>>>(
                (const cpx<float> *)spectra, g, alpha_tau, per_instance, kn, floor, status,
                freqs, amps, n_candidates, floor_dev);
        }
        return check_launch("decode_kernel");
    }
    if (precision == FPSSFT_F64) {
        const size_t sm = spec_smem(g, g.nlines, 16);
        if ((long long)sm > max_smem_optin()) return fail(FPSSFT_EUNSUPPORTED, "L too large");
        e = cudaFuncSetAttribute(decode_kernel<double>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
        decode_kernel<double><<<(unsigned)batch, nt, sm, st>>>(
            (const cpx<double> *)spectra, g, alpha_tau, per_instance, kn, floor, status, freqs,
            amps, n_candidates, floor_dev);
    } else {
        const size_t sm = spec_smem(g, g.nlines, 8);
        if ((long long)sm > max_smem_optin()) return fail(FPSSFT_EUNSUPPORTED, "L too large");
        e = cudaFuncSetAttribute(decode_kernel<float>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
        decode_kernel<float><<<(unsigned)batch, nt, sm, st>>>(
            (const cpx<float> *)spectra, g, alpha_tau, per_instance, kn, floor, status, freqs,
            amps, n_candidates, floor_dev);
    }
    return check_launch("decode_kernel");
}


// The device-resident large-problem loop (fpssft_loop.cuh): the
// conditional-WHILE graph for one set of buffers is built and instantiated
// once and kept (a small cache keyed by every pointer and parameter it bakes
// in, guarded by a mutex: a repeated call -- the imaging path re-running the
// same shape through the same buffers -- only re-launches it).  Each call:
// init kernel, graph launch, compaction kernel, one wait.
struct LargeGraph {
    std::vector<unsigned char> key;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaStream_t cs = nullptr;
};
std::mutex g_large_mu;
LargeGraph g_large_cache[4];
int g_large_next = 0;

void large_graph_free(LargeGraph &c) {
    if (c.exec) cudaGraphExecDestroy(c.exec);
    if (c.graph) cudaGraphDestroy(c.graph);
    if (c.cs) cudaStreamDestroy(c.cs);
    c = LargeGraph{};
}

int build_large_graph(const void *cube, int cube_precision, const fpssft_shape *shape,
                      const Geo &g, const Knobs &kn, const int32_t *schedule, unsigned char *ws,
                      const LargeWs &w, int32_t *iter_stats, LargeGraph &out) {
    LargeState *stt = (LargeState *)(ws + w.state);
    int *at_all = (int *)(ws + w.at_all);
    cpx<double> *spec = (cpx<double> *)(ws + w.spec);
    double *proj = (double *)(ws + w.proj);
    int *status = (int *)(ws + w.status), *dfreqs = (int *)(ws + w.dfreqs);
    double *damps = (double *)(ws + w.damps);
    int *ncand = (int *)(ws + w.ncand), *slot_of = (int *)(ws + w.slot_of);
    int *sfreqs = (int *)(ws + w.sfreqs);
    double *samps = (double *)(ws + w.samps);
    const int L = g.L, nl = g.nlines;
    LargeGraph c;
    cudaError_t e;
#define LARGE_TRY(call, what)                   \
    do {                                        \
        e = (call);                             \
        if (e != cudaSuccess) {                 \
            large_graph_free(c);                \
            return cuda_fail(e, what);          \
        }                                       \
    } while (0)
    LARGE_TRY(cudaGraphCreate(&c.graph, 0), "cudaGraphCreate");
    cudaGraphConditionalHandle cond;
    LARGE_TRY(cudaGraphConditionalHandleCreate(&cond, c.graph, 1, cudaGraphCondAssignDefault),
              "cudaGraphConditionalHandleCreate");
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    LARGE_TRY(cudaGraphAddNode(&cnode, c.graph, nullptr, 0, &cp), "cudaGraphAddNode(while)");
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    LARGE_TRY(cudaStreamCreateWithFlags(&c.cs, cudaStreamNonBlocking), "cudaStreamCreate");
    LARGE_TRY(cudaStreamBeginCaptureToGraph(c.cs, body, nullptr, nullptr, 0,
                                            cudaStreamCaptureModeThreadLocal),
              "cudaStreamBeginCaptureToGraph");
    // ---- one iteration
    large_setup_kernel<<<1, 32, 0, c.cs>>>(schedule, g, kn, stt, at_all);
    int rc = fpssft_gather_lines(cube, cube_precision, 1, 0, shape, at_all, 0, spec, FPSSFT_F64,
                                 c.cs);
    if (rc == FPSSFT_OK) rc = fpssft_dft_forward(spec, nl, L, spec, FPSSFT_F64, c.cs);
    if (rc == FPSSFT_OK) {
        constexpr int PBT = 64, PCAP = 512;
        large_project_kernel<PBT, PCAP><<<(unsigned)((L + PBT - 1) / PBT), PBT, 0, c.cs>>>(
            sfreqs, samps, stt, g, at_all, proj);
        rc = check_launch("large_project_kernel");
    }
    if (rc == FPSSFT_OK) {
        large_subtract_kernel<<<(unsigned)std::min(1184, (nl * L + 255) / 256), 256, 0, c.cs>>>(
            spec, proj, nl * L, stt);
        rc = launch_decode(spec, 1, g, kn, FPSSFT_F64, at_all, 0, 0.0, &stt->floor, status,
                           dfreqs, damps, ncand, c.cs);
    }
    if (rc == FPSSFT_OK) {
        large_merge_kernel<<<1, LARGE_NT, 0, c.cs>>>(spec, status, dfreqs, damps, ncand, at_all,
                                                     g, kn, stt, slot_of, sfreqs, samps,
                                                     iter_stats, cond);
        rc = check_launch("large_merge_kernel");
    }
    cudaGraph_t captured = nullptr;
    e = cudaStreamEndCapture(c.cs, &captured);
    if (rc != FPSSFT_OK) {
        large_graph_free(c);
        return rc;
    }
    if (e != cudaSuccess) {
        large_graph_free(c);
        return cuda_fail(e, "cudaStreamEndCapture");
    }
    LARGE_TRY(cudaGraphInstantiate(&c.exec, c.graph, 0), "cudaGraphInstantiate");
#undef LARGE_TRY
    out = c;
    return FPSSFT_OK;
}

int run_large(const void *cube, int cube_precision, const fpssft_shape *shape, const Geo &g,
              const Knobs &kn, const int32_t *schedule, unsigned char *ws, const LargeWs &w,
              int32_t *freqs, double *amps, int32_t *count, int32_t *iterations,
              int64_t *samples_used, int32_t *terminated_by, int32_t *iter_stats,
              cudaStream_t st) {
    // everything the graph bakes in
    std::vector<unsigned char> key;
    auto put = [&key](const void *p, size_t n) {
        key.insert(key.end(), (const unsigned char *)p, (const unsigned char *)p + n);
    };
    int dev = 0;
    cudaGetDevice(&dev);
    put(&dev, sizeof dev);
    put(&cube, sizeof cube);
    put(&cube_precision, sizeof cube_precision);
    put(&shape->ndim, sizeof shape->ndim);
    put(shape->dims, sizeof(shape->dims[0]) * shape->ndim);
    put(shape->strides, sizeof(shape->strides[0]) * shape->ndim);
    put(&kn, sizeof kn);
    put(&schedule, sizeof schedule);
    put(&ws, sizeof ws);
    put(&iter_stats, sizeof iter_stats);
    LargeState *stt = (LargeState *)(ws + w.state);
    int *slot_of = (int *)(ws + w.slot_of);
    long long n_total = 1;
    for (int k = 0; k < g.D; ++k) n_total *= g.N[k];
    std::lock_guard<std::mutex> lock(g_large_mu);
    LargeGraph *c = nullptr;
    for (auto &e : g_large_cache)
        if (e.exec && e.key == key) c = &e;
    if (!c) {
        LargeGraph fresh;
        const int rc = build_large_graph(cube, cube_precision, shape, g, kn, schedule, ws, w,
                                         iter_stats, fresh);
        if (rc != FPSSFT_OK) return rc;
        fresh.key = key;
        LargeGraph &slot = g_large_cache[g_large_next];
        g_large_next = (g_large_next + 1) % 4;
        cudaStreamSynchronize(slot.cs ? slot.cs : st);  // (never running: launches are waited)
        large_graph_free(slot);
        slot = fresh;
        c = &slot;
    }
    large_init_kernel<<<(unsigned)std::min<long long>((n_total + 255) / 256, 1184), 256, 0, st>>>(
        stt, slot_of, n_total, kn.t_max);
    int rc = check_launch("large_init_kernel");
    if (rc != FPSSFT_OK) return rc;
    cudaError_t e = cudaGraphLaunch(c->exec, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphLaunch");
    large_final_kernel<<<1, LARGE_NT, 0, st>>>(stt, slot_of, (const int *)(ws + w.sfreqs),
                                               (const double *)(ws + w.samps), g, freqs, amps,
                                               count, iterations, (long long *)samples_used,
                                               terminated_by);
    rc = check_launch("large_final_kernel");
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize(large loop)");
    return rc;
}

}  // namespace
}  // namespace fpssft

using namespace fpssft;

extern "C" {
#if FPSSFT_PHASE_CLOCK
int fpssft_debug_phase_cycles(unsigned long long *out, int reset) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(g_phase_cycles));
    if (reset) {
        static const unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
    }
    return 0;
}
#endif

const char *fpssft_last_error(void) { return g_err.c_str(); }
int fpssft_abi_version(void) { return 1; }
int fpssft_launches_per_batch(void) { return 1; }

#if FPSSFT_GUARD_CALIB
// Calibration builds only: the largest float32 bin-value error seen against
// the exact values, in units of the kappa = 1 guard bound, and how many bins
// were measured; resets both.
int fpssft_guard_calib(float *max_ratio, unsigned long long *count) {
    unsigned int m = 0;
    unsigned long long c = 0;
    cudaMemcpyFromSymbol(&m, g_guard_calib_max, sizeof m);
    cudaMemcpyFromSymbol(&c, g_guard_calib_count, sizeof c);
    unsigned int z = 0;
    unsigned long long zc = 0;
    cudaMemcpyToSymbol(g_guard_calib_max, &z, sizeof z);
    cudaMemcpyToSymbol(g_guard_calib_count, &zc, sizeof zc);
    std::memcpy(max_ratio, &m, sizeof m);
    *count = c;
    return FPSSFT_OK;
}
#if FPSSFT_GUARD_CALIB == 2
int fpssft_guard_reasons(unsigned long long *out) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_guard_reason, sizeof(g_guard_reason));
    static const unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_guard_reason, z, sizeof(z));
    return 0;
}
#endif
#endif

/* Device-resident loop for one large problem: see include/fpssft.h. */
int64_t fpssft_recover_large_workspace(const fpssft_shape *shape, int32_t k_cap) {
    Geo g;
    if (make_geo(shape, &g) != FPSSFT_OK) return -1;
    if (k_cap < 1) return -1;
    return (int64_t)large_ws(g, k_cap).total;
}

int fpssft_recover_large(const void *cube, int32_t cube_precision, const fpssft_shape *shape,
                         const fpssft_params *params, const int32_t *schedule, void *workspace,
                         int64_t workspace_bytes, int32_t *freqs, double *amps, int32_t *count,
                         int32_t *iterations, int64_t *samples_used, int32_t *terminated_by,
                         int32_t *iter_stats, void *stream) {
    Geo g;
    Knobs kn;
    int rc;
    if ((rc = make_geo(shape, &g)) != FPSSFT_OK) return rc;
    if ((rc = make_knobs(params, &kn)) != FPSSFT_OK) return rc;
    if (params->precision != FPSSFT_F64)
        return fail(FPSSFT_EUNSUPPORTED, "the device-resident large loop runs in float64");
    if (cube_precision != FPSSFT_F32 && cube_precision != FPSSFT_F64)
        return fail(FPSSFT_EINVAL, "cube_precision must be FPSSFT_F32 or FPSSFT_F64");
    if (!cube || !schedule || !workspace || !freqs || !amps || !count || !iterations ||
        !samples_used || !terminated_by)
        return fail(FPSSFT_EINVAL, "NULL buffer");
    const LargeWs w = large_ws(g, kn.k_cap);
    if (workspace_bytes < (int64_t)w.total)
        return fail(FPSSFT_EINVAL, "workspace smaller than fpssft_recover_large_workspace()");
    return run_large(cube, cube_precision, shape, g, kn, schedule, (unsigned char *)workspace, w,
                     freqs, amps, count, iterations, samples_used, terminated_by, iter_stats,
                     (cudaStream_t)stream);
}

int fpssft_set_l2_fetch_granularity(int32_t bytes) {
    if (bytes < 0 || bytes > 128 || (bytes & (bytes - 1)))
        return fail(FPSSFT_EINVAL, "L2 fetch granularity must be 0 or a power of two <= 128");
    cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceSetLimit(MaxL2FetchGranularity)");
    return FPSSFT_OK;
}

int fpssft_get_l2_fetch_granularity(void) {
    size_t v = 0;
    if (cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity) != cudaSuccess) return -1;
    return (int)v;
}

int fpssft_block_threads(const fpssft_shape *shape, int32_t precision) {
    (void)precision;
    Geo g;
    if (make_geo(shape, &g) != FPSSFT_OK) return -1;
    return block_threads(g, g.nlines, precision);
}

size_t fpssft_smem_bytes(const fpssft_shape *shape, const fpssft_params *params) {
    size_t smem = 0;
    if (fpssft_plan(shape, params, nullptr, nullptr, nullptr, &smem) != FPSSFT_OK) return 0;
    return smem;
}

int fpssft_run_batch(const void *cubes, int64_t batch, int64_t batch_stride,
                     const fpssft_shape *shape, const fpssft_params *params,
                     const int32_t *schedule, const int32_t *sched_index, int32_t n_sched,
                     const fpssft_out *out, void *stream) {
    return fpssft_run_batch_grouped(cubes, batch, 1, batch_stride, shape, params, schedule,
                                    sched_index, n_sched, out, stream);
}

int fpssft_run_batch_grouped(const void *cubes, int64_t batch, int32_t group,
                             int64_t group_stride, const fpssft_shape *shape,
                             const fpssft_params *params, const int32_t *schedule,
                             const int32_t *sched_index, int32_t n_sched, const fpssft_out *out,
                             void *stream) {
    Geo g;
    Knobs kn;
    int rc;
    const int64_t batch_stride = group_stride;
    if ((rc = make_geo(shape, &g)) != FPSSFT_OK) return rc;
    if ((rc = make_knobs(params, &kn)) != FPSSFT_OK) return rc;
    if (group < 1 || group > 64) return fail(FPSSFT_EINVAL, "group must be in [1, 64]");
    kn.group = group;
    const int prec = effective_precision(g, kn, params->precision, params->mode);
    set_noise_floor(&kn, g, prec);
    if (batch < 0) return fail(FPSSFT_EINVAL, "batch must be >= 0");
    if (batch > INT_MAX) return fail(FPSSFT_EINVAL, "batch exceeds the grid limit");
    if (batch > 0 && (!cubes || !schedule || !out || !out->freqs || !out->amps || !out->count ||
                      !out->iterations || !out->samples_used || !out->terminated_by))
        return fail(FPSSFT_EINVAL, "NULL buffer");
    if (n_sched < 1) return fail(FPSSFT_EINVAL, "n_sched must be >= 1");
    OutPtrs o{out ? out->freqs : nullptr,
              out ? out->amps : nullptr,
              out ? out->count : nullptr,
              out ? out->iterations : nullptr,
              out ? (long long *)out->samples_used : nullptr,
              out ? out->terminated_by : nullptr,
              out ? out->iter_stats : nullptr};
    cudaStream_t st = (cudaStream_t)stream;
    if (prec == FPSSFT_F64)
        return run_batch_t<double>(cubes, batch, batch_stride, g, kn, params->mode, schedule,
                                   sched_index, n_sched, o, st);
    return run_batch_t<float>(cubes, batch, batch_stride, g, kn, params->mode, schedule,
                              sched_index, n_sched, o, st);
}

int64_t fpssft_stage_bytes(const fpssft_shape *shape, int32_t group, int64_t batch,
                           int32_t stage_iterations) {
    Geo g;
    if (make_geo(shape, &g) != FPSSFT_OK) return -1;
    if (group < 2 || group > 64 || (group & 1) || batch < 0 || stage_iterations < 1) return -1;
    const int64_t groups = (batch + group - 1) / group;
    return groups * stage_iterations * (int64_t)g.nlines * g.L * group * 8;
}

namespace {
// Argument checks shared by fpssft_stage_lines and fpssft_run_batch_staged;
// *t0 = the iterations really staged.
int staged_args(const void *cubes, int64_t batch, int32_t group, int64_t group_stride,
                const fpssft_shape *shape, const fpssft_params *params, const int32_t *schedule,
                const void *staging, int64_t staging_bytes, int32_t stage_iterations, Geo *g,
                Knobs *kn, int *t0) {
    int rc;
    if ((rc = make_geo(shape, g)) != FPSSFT_OK) return rc;
    if ((rc = make_knobs(params, kn)) != FPSSFT_OK) return rc;
    if (group < 2 || group > 64 || (group & 1))
        return fail(FPSSFT_EINVAL, "staged lines: group must be even, in [2, 64]");
    if (stage_iterations < 1) return fail(FPSSFT_EINVAL, "stage_iterations must be >= 1");
    {   // the warp-per-instance kernels read staged lines (the group-gather
        // one for the team, the others per instance), in float32 / guarded
        const int prec = effective_precision(*g, *kn, params->precision, params->mode);
        Geo gp = *g;
        LaunchPlan lp;
        Knobs ks = *kn;
        ks.group = group;
        ks.staged = (const float2 *)staging;
        if (prec == FPSSFT_F64 || !g->off32 ||
            make_plan(gp, ks, prec, params->mode, &lp, true) != FPSSFT_OK ||
            !(lp.mode == FPSSFT_MODE_WARP ||
              (lp.mode == FPSSFT_MODE_CTA && lp.kernel && prec == FPSSFT_F32)))
            return fail(FPSSFT_EUNSUPPORTED,
                        "staged lines need a warp-per-instance kernel (float32 or guarded) or a "
                        "compile-time float32 team kernel, 32-bit offsets");
    }
    if (batch < 0 || batch > INT_MAX) return fail(FPSSFT_EINVAL, "bad batch");
    *t0 = std::min<int>(stage_iterations, kn->t_max);
    if (batch == 0) return FPSSFT_OK;
    if (!cubes || !schedule || !staging) return fail(FPSSFT_EINVAL, "NULL buffer");
    if (staging_bytes < fpssft_stage_bytes(shape, group, batch, *t0))
        return fail(FPSSFT_EINVAL, "staging buffer smaller than fpssft_stage_bytes()");
    for (int k = 0; k < g->D; ++k)
        if (shape->strides[k] % group)
            return fail(FPSSFT_EINVAL, "staged lines: strides must be multiples of group");
    if (((uintptr_t)cubes | (uintptr_t)staging) & 15 || (group_stride * 8) % 16)
        return fail(FPSSFT_EINVAL, "staged lines: 16-byte aligned cubes and staging buffer");
    if ((batch + group - 1) / group > 65535 || *t0 > 65535)
        return fail(FPSSFT_EINVAL, "staged lines: too many groups");
    return FPSSFT_OK;
}

int launch_stage(const void *cubes, int64_t batch, int32_t group, int64_t group_stride,
                 const Geo &g, const int32_t *schedule, void *staging, int t0, cudaStream_t st) {
    const int64_t groups = (batch + group - 1) / group;
    const int NLL = g.nlines * g.L;
    // one CTA per SM (a second one does not fit beside it): 256 bulk copies in
    // flight per SM keep the host link full, and a recovery CTA of another
    // stream still finds room (pipelined chunks, hostpath.py)
    const size_t smem = std::max<size_t>((size_t)stage::POS * 8 * group, 120 * 1024);
    cudaError_t e = cudaFuncSetAttribute(stage::stage_lines_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(stage_lines_kernel)");
    dim3 grid((unsigned)((NLL + stage::POS - 1) / stage::POS), (unsigned)t0, (unsigned)groups);
    stage::stage_lines_kernel<<<grid, stage::POS, smem, st>>>(
        (const float2 *)cubes, (long long)group_stride, g, group, schedule, t0,
        (float2 *)staging, (long long)t0 * NLL * group);
    return check_launch("stage_lines_kernel");
}
}  // namespace

int fpssft_stage_lines(const void *cubes, int64_t batch, int32_t group, int64_t group_stride,
                       const fpssft_shape *shape, const fpssft_params *params,
                       const int32_t *schedule, void *staging, int64_t staging_bytes,
                       int32_t stage_iterations, void *stream) {
    Geo g;
    Knobs kn;
    int t0 = 0;
    int rc = staged_args(cubes, batch, group, group_stride, shape, params, schedule, staging,
                         staging_bytes, stage_iterations, &g, &kn, &t0);
    if (rc != FPSSFT_OK || batch == 0) return rc;
    return launch_stage(cubes, batch, group, group_stride, g, schedule, staging, t0,
                        (cudaStream_t)stream);
}

int fpssft_run_batch_staged(const void *cubes, int64_t batch, int32_t group,
                            int64_t group_stride, const fpssft_shape *shape,
                            const fpssft_params *params, const int32_t *schedule,
                            const fpssft_out *out, void *staging, int64_t staging_bytes,
                            int32_t stage_iterations, int32_t already_staged, void *stream) {
    Geo g;
    Knobs kn;
    int t0 = 0;
    int rc = staged_args(cubes, batch, group, group_stride, shape, params, schedule, staging,
                         staging_bytes, stage_iterations, &g, &kn, &t0);
    if (rc != FPSSFT_OK || batch == 0) return rc;
    if (!out || !out->freqs || !out->amps || !out->count || !out->iterations ||
        !out->samples_used || !out->terminated_by)
        return fail(FPSSFT_EINVAL, "NULL buffer");
    cudaStream_t st = (cudaStream_t)stream;
    if (!already_staged &&
        (rc = launch_stage(cubes, batch, group, group_stride, g, schedule, staging, t0, st)) !=
            FPSSFT_OK)
        return rc;
    kn.group = group;
    kn.staged = (const float2 *)staging;
    kn.staged_group_stride = (long long)t0 * g.nlines * g.L * group;
    kn.stage_T = t0;
    set_noise_floor(&kn, g, effective_precision(g, kn, params->precision, params->mode));
    OutPtrs o{out->freqs, out->amps, out->count, out->iterations,
              (long long *)out->samples_used, out->terminated_by, out->iter_stats};
    return run_batch_t<float>(cubes, batch, group_stride, g, kn, params->mode, schedule, nullptr,
                              1, o, st);
}

int fpssft_synthesize(const int32_t *freqs, const double *amps, const int32_t *counts,
                      int64_t batch, int32_t k_cap, const fpssft_shape *shape, void *cubes,
                      int64_t batch_stride, int32_t precision, void *stream) {
    Geo gc, gr;
    int rc;
    if ((rc = make_geo(shape, &gc)) != FPSSFT_OK) return rc;
    if (batch < 0 || batch > INT_MAX) return fail(FPSSFT_EINVAL, "bad batch");
    if (k_cap < 1) return fail(FPSSFT_EINVAL, "k_cap must be >= 1");
    for (int k = 0; k < gc.D; ++k)
        if (shape->strides[k] != (k == gc.D - 1 ? 1 : shape->strides[k + 1] * shape->dims[k + 1]))
            return fail(FPSSFT_EINVAL, "synthesize writes row-major contiguous cubes");
    if (batch == 0) return FPSSFT_OK;
    if (!freqs || !amps || !counts || !cubes) return fail(FPSSFT_EINVAL, "NULL buffer");
    fpssft_shape row;
    std::memset(&row, 0, sizeof(row));
    row.ndim = 1;
    row.dims[0] = shape->dims[gc.D - 1];
    row.strides[0] = 1;
    if ((rc = make_geo(&row, &gr)) != FPSSFT_OK) return rc;
    const int NT = 256, NL = gr.L;
    const int cs = precision == FPSSFT_F64 ? 16 : 8;
    if (FPSSFT_SYNTH_REG && precision != FPSSFT_F64 && gc.D == 2 && NL == 512 &&
        gc.N[0] % FPSSFT_SYNTH_RC == 0 && (long long)gc.L * gc.N[0] < (1LL << 32)) {
        // config 5's 512 x 512 images in float32: register row FFTs (fpssft_synth.cuh)
        const size_t smr = align16((size_t)(FPSSFT_SYNTH_DB ? 2 : 1) * FPSSFT_SYNTH_RC * synth::VS * 8) +
                           align16((size_t)gc.L * 8) +
                           align16((size_t)k_cap * 8) + align16((size_t)k_cap * 4) +
                           align16((size_t)513 * 4) + align16((size_t)512 * 4) + 64 * 8;
        if ((long long)smr <= SMEM_PER_CTA &&
            (size_t)k_cap * 4 <= (size_t)FPSSFT_SYNTH_RC * synth::VS * 8) {
            auto k = synth::synth512_kernel<FPSSFT_SYNTH_RC, FPSSFT_SYNTH_NT, (bool)FPSSFT_SYNTH_DB>;
            cudaError_t e =
                cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smr);
            if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(synth512)");
            k<<<(unsigned)batch, FPSSFT_SYNTH_NT, smr, (cudaStream_t)stream>>>(
                freqs, amps, counts, k_cap, gc, (float2 *)cubes, batch_stride);
            return check_launch("synth512_kernel");
        }
    }
    if (gc.D == 2 && NL == 512 && gc.N[0] % SYNTH_RC == 0 &&
        (long long)gc.L * gc.N[0] < (1LL << 32)) {
        // compile-time variant: config 5's 512 x 512 images, SYNTH_RC rows per
        // chunk, SYNTH_NT threads
        const size_t sm2 = align16((size_t)SYNTH_RC * (512 + 512 / 16 + 1) * cs) +  // V (padded)
                           align16((size_t)gc.L * cs) + align16((size_t)512 * cs) +
                           align16((size_t)k_cap * cs) + align16((size_t)k_cap * 4) +
                           align16((size_t)513 * 4) + align16((size_t)512 * 4) +
                           align16((size_t)k_cap * 4) + align16((size_t)512 * 4) + 64 * 8;
        if ((long long)sm2 <= SMEM_PER_CTA) {
            cudaStream_t st = (cudaStream_t)stream;
            cudaError_t e;
            if (precision == FPSSFT_F64) {
                auto k = synth_static_kernel<double, 512, SYNTH_RC, SYNTH_NT>;
                e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
                if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(synth)");
                k<<<(unsigned)batch, SYNTH_NT, sm2, st>>>(freqs, amps, counts, k_cap, gc,
                                                          (float2 *)cubes, batch_stride);
            } else {
                auto k = synth_static_kernel<float, 512, SYNTH_RC, SYNTH_NT>;
                e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
                if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(synth)");
                k<<<(unsigned)batch, SYNTH_NT, sm2, st>>>(freqs, amps, counts, k_cap, gc,
                                                          (float2 *)cubes, batch_stride);
            }
            return check_launch("synth_static_kernel");
        }
    }
    int rcnt = std::max(1, std::min(16, 65536 / (NL * cs)));  // rows per chunk
    while (rcnt > 1 && plan_fft(&gr, rcnt, precision, NT) < 0) rcnt /= 2;
    if (plan_fft(&gr, rcnt, precision, NT) < 0)
        return fail(FPSSFT_EUNSUPPORTED, "row length too large for the synthesis kernel");
    size_t sm = align16((size_t)rcnt * NL * cs) + align16((size_t)gc.L * cs) +
                align16((size_t)NL * cs) + align16((size_t)k_cap * cs) +
                align16((size_t)k_cap * 4 * MAXD) + align16((size_t)(NL + 1) * 4) +
                align16((size_t)NL * 4) + align16((size_t)k_cap * 4) + 64 * 8;
    if ((long long)sm > SMEM_PER_CTA) return fail(FPSSFT_EUNSUPPORTED, "k_cap/row too large");
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e;
    if (precision == FPSSFT_F64) {
        e = cudaFuncSetAttribute(synth_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(synth_kernel)");
        synth_kernel<double><<<(unsigned)batch, NT, sm, st>>>(freqs, amps, counts, k_cap, gc, gr,
                                                             rcnt, (float2 *)cubes, batch_stride);
    } else {
        e = cudaFuncSetAttribute(synth_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(synth_kernel)");
        synth_kernel<float><<<(unsigned)batch, NT, sm, st>>>(freqs, amps, counts, k_cap, gc, gr,
                                                            rcnt, (float2 *)cubes, batch_stride);
    }
    return check_launch("synth_kernel");
}

int fpssft_plan(const fpssft_shape *shape, const fpssft_params *params, int32_t *mode,
                int32_t *threads_per_cta, int32_t *instances_per_cta, size_t *smem_bytes) {
    return fpssft_plan_batch(shape, params, 1, 0, mode, threads_per_cta, instances_per_cta,
                             smem_bytes);
}

int fpssft_plan_batch(const fpssft_shape *shape, const fpssft_params *params, int32_t group,
                      int32_t per_instance_schedules, int32_t *mode, int32_t *threads_per_cta,
                      int32_t *instances_per_cta, size_t *smem_bytes) {
    Geo g;
    Knobs kn;
    int rc;
    if ((rc = make_geo(shape, &g)) != FPSSFT_OK) return rc;
    if ((rc = make_knobs(params, &kn)) != FPSSFT_OK) return rc;
    if (group < 1 || group > 64) return fail(FPSSFT_EINVAL, "group must be in [1, 64]");
    kn.group = group;
    LaunchPlan lp;
    const int prec = effective_precision(g, kn, params->precision, params->mode);
    if ((rc = make_plan(g, kn, prec, params->mode, &lp, !per_instance_schedules)) != FPSSFT_OK)
        return rc;
    if (mode) *mode = lp.mode;
    if (threads_per_cta) *threads_per_cta = lp.threads;
    if (instances_per_cta) *instances_per_cta = lp.per_cta;
    if (smem_bytes) *smem_bytes = lp.smem;
    return FPSSFT_OK;
}

int fpssft_line_spectra(const void *cubes, int64_t batch, int64_t batch_stride,
                        const fpssft_shape *shape, const int32_t *alpha_tau,
                        int32_t per_instance, void *spectra, int32_t precision, void *stream) {
    Geo g;
    int rc;
    if ((rc = make_geo(shape, &g)) != FPSSFT_OK) return rc;
    if (batch < 0 || batch > INT_MAX) return fail(FPSSFT_EINVAL, "bad batch");
    if (batch == 0) return FPSSFT_OK;
    if (!cubes || !alpha_tau || !spectra) return fail(FPSSFT_EINVAL, "NULL buffer");
    const int nt = block_threads(g, g.nlines, precision);
    if (nt < 0) return fail(FPSSFT_EUNSUPPORTED, "line length too large for one CTA");
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e;
    if (precision == FPSSFT_F64) {
        const size_t sm = spec_smem(g, g.nlines, 16);
        if ((long long)sm > max_smem_optin()) return fail(FPSSFT_EUNSUPPORTED, "L too large");
        e = cudaFuncSetAttribute(line_spectra_kernel<double>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
        line_spectra_kernel<double><<<(unsigned)batch, nt, sm, st>>>(
            (const float2 *)cubes, batch_stride, g, alpha_tau, per_instance, (cpx<double> *)spectra);
    } else {
        const size_t sm = spec_smem(g, g.nlines, 8);
        if ((long long)sm > max_smem_optin()) return fail(FPSSFT_EUNSUPPORTED, "L too large");
        e = cudaFuncSetAttribute(line_spectra_kernel<float>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
        line_spectra_kernel<float><<<(unsigned)batch, nt, sm, st>>>(
            (const float2 *)cubes, batch_stride, g, alpha_tau, per_instance, (cpx<float> *)spectra);
    }
    return check_launch("line_spectra_kernel");
}

int fpssft_gather_lines(const void *cubes, int32_t cube_precision, int64_t batch,
                        int64_t batch_stride, const fpssft_shape *shape, const int32_t *alpha_tau,
                        int32_t per_instance, void *lines, int32_t precision, void *stream) {
    Geo g;
    int rc;
    if ((rc = make_geo(shape, &g)) != FPSSFT_OK) return rc;
    if (batch < 0 || batch > 65535) return fail(FPSSFT_EINVAL, "bad batch (0..65535)");
    if (batch == 0) return FPSSFT_OK;
    if (!cubes || !alpha_tau || !lines) return fail(FPSSFT_EINVAL, "NULL buffer");
    if (cube_precision != FPSSFT_F32 && cube_precision != FPSSFT_F64)
        return fail(FPSSFT_EINVAL, "cube_precision must be FPSSFT_F32 or FPSSFT_F64");
    cudaStream_t st = (cudaStream_t)stream;
    const long long n = (long long)g.nlines * g.L;
    const dim3 grid((unsigned)std::min<long long>((n + 255) / 256, 4096), (unsigned)batch);
    const bool c128 = cube_precision == FPSSFT_F64;
    if (precision == FPSSFT_F64) {
        if (c128)
            gather_lines_kernel<double2, double><<<grid, 256, 0, st>>>(
                (const double2 *)cubes, batch_stride, g, alpha_tau, per_instance,
                (cpx<double> *)lines);
        else
            gather_lines_kernel<float2, double><<<grid, 256, 0, st>>>(
                (const float2 *)cubes, batch_stride, g, alpha_tau, per_instance,
                (cpx<double> *)lines);
    } else {
        if (c128)
            gather_lines_kernel<double2, float><<<grid, 256, 0, st>>>(
                (const double2 *)cubes, batch_stride, g, alpha_tau, per_instance,
                (cpx<float> *)lines);
        else
            gather_lines_kernel<float2, float><<<grid, 256, 0, st>>>(
                (const float2 *)cubes, batch_stride, g, alpha_tau, per_instance,
                (cpx<float> *)lines);
    }
    return check_launch("gather_lines_kernel");
}

int fpssft_dft_forward(const void *lines, int64_t batch, int32_t L, void *out, int32_t precision,
                       void *stream) {
    if (L < 1) return fail(FPSSFT_EINVAL, "expected a nonempty 1-D array");
    fpssft_shape sh;
    std::memset(&sh, 0, sizeof(sh));
    sh.ndim = 1;
    sh.dims[0] = L;
    sh.strides[0] = 1;
    Geo g;
    int rc;
    if ((rc = make_geo(&sh, &g)) != FPSSFT_OK) return rc;
    if (batch < 0 || batch > INT_MAX) return fail(FPSSFT_EINVAL, "bad batch");
    if (batch == 0) return FPSSFT_OK;
    if (!lines || !out) return fail(FPSSFT_EINVAL, "NULL buffer");
    const int nt = block_threads(g, 1, precision);
    if (nt < 0) return fail(FPSSFT_EUNSUPPORTED, "line length too large for one CTA");
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e;
    if (precision == FPSSFT_F64) {
        const size_t sm = spec_smem(g, 1, 16);
        if ((long long)sm > max_smem_optin()) return fail(FPSSFT_EUNSUPPORTED, "L too large");
        e = cudaFuncSetAttribute(dft_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
        dft_kernel<double><<<(unsigned)batch, nt, sm, st>>>((const cpx<double> *)lines, g,
                                                           (cpx<double> *)out);
    } else {
        const size_t sm = spec_smem(g, 1, 8);
        if ((long long)sm > max_smem_optin()) return fail(FPSSFT_EUNSUPPORTED, "L too large");
        e = cudaFuncSetAttribute(dft_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
        dft_kernel<float><<<(unsigned)batch, nt, sm, st>>>((const cpx<float> *)lines, g,
                                                          (cpx<float> *)out);
    }
    return check_launch("dft_kernel");
}

int fpssft_decode_spectra(const void *spectra, int64_t batch, const fpssft_shape *shape,
                          const int32_t *alpha_tau, int32_t per_instance,
                          const fpssft_params *params, double floor, int32_t *status,
                          int32_t *freqs, double *amps, int32_t *n_candidates, void *stream) {
    Geo g;
    Knobs kn;
    int rc;
    if ((rc = make_geo(shape, &g)) != FPSSFT_OK) return rc;
    if ((rc = make_knobs(params, &kn)) != FPSSFT_OK) return rc;
    set_noise_floor(&kn, g, params->precision);
    if (batch < 0 || batch > INT_MAX) return fail(FPSSFT_EINVAL, "bad batch");
    if (batch == 0) return FPSSFT_OK;
    if (!spectra || !alpha_tau || !status || !freqs || !amps || !n_candidates)
        return fail(FPSSFT_EINVAL, "NULL buffer");
    return launch_decode(spectra, batch, g, kn, params->precision, alpha_tau, per_instance, floor,
                         nullptr, status, freqs, amps, n_candidates, (cudaStream_t)stream);
}

int fpssft_project_onto_bins(const int32_t *freqs, const double *amps, const int32_t *counts,
                             int64_t batch, int32_t k_max, const fpssft_shape *shape,
                             const int32_t *alpha_tau, int32_t per_instance, double *out,
                             int32_t precision, void *stream) {
    Geo g;
    int rc;
    if ((rc = make_geo(shape, &g)) != FPSSFT_OK) return rc;
    if (batch < 0 || batch > INT_MAX) return fail(FPSSFT_EINVAL, "bad batch");
    if (k_max < 1) return fail(FPSSFT_EINVAL, "k_max must be >= 1");
    if (batch == 0) return FPSSFT_OK;
    if (!freqs || !amps || !counts || !alpha_tau || !out) return fail(FPSSFT_EINVAL, "NULL buffer");
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e;
    const int cs = precision == FPSSFT_F64 ? 16 : 8;
    const int nt = block_threads(g, 1, precision);
    const size_t sm = make_layout(g.D, g.L, k_max, cs).total;
    if (nt < 0 || (long long)sm > max_smem_optin()) {
        // large sets / long lines: one thread per bin scanning the entries
        constexpr int BT = 64, CAP = 1536;
        const dim3 grid((unsigned)((g.L + BT - 1) / BT), (unsigned)batch);
        if (precision == FPSSFT_F64)
            project_global_kernel<double, BT, CAP><<<grid, BT, 0, st>>>(
                freqs, amps, counts, k_max, g, alpha_tau, per_instance, out);
        else
            project_global_kernel<float, BT, CAP><<<grid, BT, 0, st>>>(
                freqs, amps, counts, k_max, g, alpha_tau, per_instance, out);
        return check_launch("project_global_kernel");
    }
    if (precision == FPSSFT_F64) {
        e = cudaFuncSetAttribute(project_kernel<double>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
        project_kernel<double><<<(unsigned)batch, nt, sm, st>>>(freqs, amps, counts, k_max, g,
                                                               alpha_tau, per_instance, out);
    } else {
        e = cudaFuncSetAttribute(project_kernel<float>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
        project_kernel<float><<<(unsigned)batch, nt, sm, st>>>(freqs, amps, counts, k_max, g,
                                                              alpha_tau, per_instance, out);
    }
    return check_launch("project_kernel");
}

}  // extern "C"
