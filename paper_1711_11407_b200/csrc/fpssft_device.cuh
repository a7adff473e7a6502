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
template <class R>
__device__ __forceinline__ R cabs(cpx<R> a) { return hypot(a.re, a.im); }
__device__ __forceinline__ float cabs(cpx<float> a) { return hypotf(a.re, a.im); }

// ---------------------------------------------------------------- geometry
// CubeShape (core.py:26-73) as the kernels see it.
struct Geo {
    int D, L, nlines;               // nlines = D + 1
    int N[MAXD];                    // extents
    int cof[MAXD];                  // c_k = L / N_k
    long long stride[MAXD];         // element strides of one cube
    unsigned long long magic[MAXD]; // fastmod multipliers for N_k
    int nstages;                    // FFT plan, 8 bits per stage s in plan[s/8] >> 8(s%8):
    unsigned long long plan[2];     //   low 5 bits radix {2,3,4,5,7,8,16} (0 = direct O(L^2)),
                                    //   high 3 bits butterflies per thread {1,2,4}
    int threads;                    // CTA size the plan was made for
};
__host__ __device__ __forceinline__ int stage_code(const Geo &g, int s) {
    const unsigned long long w = s < 8 ? g.plan[0] : g.plan[1];  // no dynamic indexing
    return (int)((w >> (8 * (s & 7))) & 255ULL);
}

// Tolerances / knobs (FpsSftConfig, driver.py:29-63).
struct Knobs {
    double mag_tol, verify_tol, round_tol, amp_prune_tol;
    double energy_floor, energy_floor_abs, residual_stop;
    double noise_coef;  // float32 rounding floor: coef * sqrt(sum |x|^2 over the D+1 lines)
    int t_max, stall_limit, k_cap;
};

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

// ------------------------------------------------------------------ gather
// Line samples x[(alpha*l + tau) mod N] for the D+1 offsets tau, tau+e_k
// (lines.py:36-64).  Row l of offset k+1 differs from offset 0 only in
// coordinate k, advanced by one with wrap, so each thread issues its D+1
// loads from one base address.  Index math is fastmod, no division.
// Returns this thread's share of sum |x|^2 over the gathered samples.
template <class R>
__device__ __forceinline__ R gather_lines(cpx<R> *spec, const float2 *__restrict__ cube,
                                          const Geo &g, const int *al, const int *ta) {
    const int L = g.L, D = g.D;
    R energy = (R)0;
    for (int l = threadIdx.x; l < L; l += blockDim.x) {
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
        spec[l] = {(R)v[0].x, (R)v[0].y};
        energy += (R)v[0].x * (R)v[0].x + (R)v[0].y * (R)v[0].y;
#pragma unroll
        for (int k = 0; k < MAXD; ++k)
            if (k < D) {
                spec[(k + 1) * L + l] = {(R)v[k + 1].x, (R)v[k + 1].y};
                energy += (R)v[k + 1].x * (R)v[k + 1].x + (R)v[k + 1].y * (R)v[k + 1].y;
            }
    }
    return energy;
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

// One Stockham stage: butterfly q (of nlines*L/RAD) reads x[line][j + k L/RAD],
// twiddles by W_{Ns RAD}^{(j mod Ns) k}, and writes y[line][(j - j mod Ns) RAD
// + j mod Ns + k Ns].  Each thread owns MB butterflies (q = tid + i*NT); the
// host sizes NT so MB*NT covers the stage.
template <class R, int RAD, int MB>
__device__ __forceinline__ void fft_stage(cpx<R> *x, int nlines, int L, int Ns,
                                          const cpx<R> *roots, bool last) {
    const int m = L / RAD, total = nlines * m, NT = blockDim.x;
    const int step = L / (Ns * RAD);
    cpx<R> v[MB][RAD];
    int ob[MB];
#pragma unroll
    for (int j = 0; j < MB; ++j) {
        const int q = threadIdx.x + j * NT;
        ob[j] = -1;
        if (q < total) {
            const int line = q / m, jj = q - line * m;
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
    __syncthreads();
    const R fl = (R)L;
#pragma unroll
    for (int j = 0; j < MB; ++j) {
        if (ob[j] >= 0) {
#pragma unroll
            for (int k = 0; k < RAD; ++k) {
                cpx<R> o = v[j][k];
                if (last) o = {o.re / fl, o.im / fl};
                x[ob[j] + k * Ns] = o;
            }
        }
    }
    __syncthreads();
}

// Direct O(L^2) pass for lengths with a prime factor > 7 (test-size L only).
template <class R, int MB>
__device__ __forceinline__ void dft_direct(cpx<R> *x, int nlines, int L, const cpx<R> *roots) {
    const int total = nlines * L, NT = blockDim.x;
    cpx<R> acc[MB];
#pragma unroll
    for (int j = 0; j < MB; ++j) {
        const int q = threadIdx.x + j * NT;
        if (q < total) {
            const int line = q / L, k = q - line * L;
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
    __syncthreads();
    const R fl = (R)L;
#pragma unroll
    for (int j = 0; j < MB; ++j) {
        const int q = threadIdx.x + j * NT;
        if (q < total) x[q] = {acc[j].re / fl, acc[j].im / fl};
    }
    __syncthreads();
}

template <class R, int RAD>
__device__ __forceinline__ void fft_stage_mb(cpx<R> *x, int nlines, int L, int Ns, int mb,
                                             const cpx<R> *roots, bool last) {
    // register budget (matches plan_fft's caps): complex values per thread
    // <= 16 (float) / 8 (double)
    constexpr int R4 = sizeof(R) == 4 ? (RAD <= 4 ? 4 : (RAD <= 8 ? 2 : 1))
                                      : (RAD <= 2 ? 4 : (RAD <= 4 ? 2 : 1));
    if (mb <= 1) fft_stage<R, RAD, 1>(x, nlines, L, Ns, roots, last);
    else if (mb <= 2 || R4 < 4) fft_stage<R, RAD, (R4 < 2 ? 1 : 2)>(x, nlines, L, Ns, roots, last);
    else fft_stage<R, RAD, R4>(x, nlines, L, Ns, roots, last);
}

template <class R>
__device__ __forceinline__ void fft_lines(cpx<R> *x, int nlines, const Geo &g,
                                          const cpx<R> *roots) {
    int Ns = 1;
    for (int s = 0; s < g.nstages; ++s) {
        const int code = stage_code(g, s);
        const int r = code & 31, mb = code >> 5;
        const bool last = (s == g.nstages - 1);
        switch (r) {
            case 16: fft_stage_mb<R, 16>(x, nlines, g.L, Ns, mb, roots, last); break;
            case 8: fft_stage_mb<R, 8>(x, nlines, g.L, Ns, mb, roots, last); break;
            case 4: fft_stage_mb<R, 4>(x, nlines, g.L, Ns, mb, roots, last); break;
            case 2: fft_stage_mb<R, 2>(x, nlines, g.L, Ns, mb, roots, last); break;
            case 3: fft_stage_mb<R, 3>(x, nlines, g.L, Ns, mb, roots, last); break;
            case 5: fft_stage_mb<R, 5>(x, nlines, g.L, Ns, mb, roots, last); break;
            case 7: fft_stage_mb<R, 7>(x, nlines, g.L, Ns, mb, roots, last); break;
            default:
                if (mb <= 1) dft_direct<R, 1>(x, nlines, g.L, roots);
                else if (mb <= 2) dft_direct<R, 2>(x, nlines, g.L, roots);
                else dft_direct<R, 4>(x, nlines, g.L, roots);
                break;
        }
        Ns *= (r > 0 ? r : g.L);
    }
    if (g.nstages == 0) {  // L == 1: the DFT of one sample is itself
        __syncthreads();
    }
}

// ------------------------------------------------------------- bin map
// bin(m) = sum_k (c_k alpha_k mod L) m_k mod L (numtheory.py:139-153);
// u_tau(m) = sum_k c_k tau_k m_k mod L (decoder.py:41-46).  The host guards
// D * L * max N_k < 2^31 so int32 products are exact.
__device__ __forceinline__ int bin_of(const int *m, const Geo &g, const int *al) {
    int acc = 0;
#pragma unroll
    for (int k = 0; k < MAXD; ++k)
        if (k < g.D) acc += ((g.cof[k] * al[k]) % g.L) * m[k];
    return acc % g.L;
}
__device__ __forceinline__ int phase_of(const int *m, const Geo &g, const int *ta) {
    int acc = 0;
#pragma unroll
    for (int k = 0; k < MAXD; ++k)
        if (k < g.D) acc += ((g.cof[k] * ta[k]) % g.L) * m[k];
    return acc % g.L;
}
// Phase of offset i (0 = tau, i = tau + e_{i-1}) from u_0: the step adds
// c_{i-1} m_{i-1} (a wrap of tau adds L m, which vanishes mod L).
// (Selects instead of indexing with i keeps m and g in registers.)
__device__ __forceinline__ int phase_step(int u0, int i, const int *m, const Geo &g) {
    int add = 0;
#pragma unroll
    for (int k = 0; k < MAXD; ++k)
        if (k == i - 1) add = g.cof[k] * m[k];
    return (int)(((long long)u0 + add) % g.L);
}

// ---------------------------------------------------------- classifier
// decode_spectra for one bin b (decoder.py:127-169) with the driver's guard
// (driver.py:166-176).  Returns 0 (not a candidate), 1 (candidate,
// rejected), 2 (accepted), 3 (decoded and verified but guard failed).
template <class R>
__device__ __forceinline__ int classify_bin(const cpx<R> *spec, const Geo &g, int b,
                                            const int *al, const int *ta, const cpx<R> *roots,
                                            R mag_tol, R round_tol, R verify_tol, R floor,
                                            int *m, cpx<R> *amp_out) {
    const int L = g.L, D = g.D;
    cpx<R> s[MAXD + 1];
    R mag[MAXD + 1];
    R top, low;
#pragma unroll
    for (int i = 0; i < MAXD + 1; ++i) {
        if (i <= D) {
            s[i] = spec[i * L + b];
            mag[i] = cabs(s[i]);
        }
    }
    top = mag[0];
    low = mag[0];
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
            int mk = ((int)near) % g.N[k];
            m[k] = mk < 0 ? mk + g.N[k] : mk;
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

}  // namespace fpssft
