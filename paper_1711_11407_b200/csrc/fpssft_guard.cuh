// Guarded float32 decisions (precision FPSSFT_F32_GUARDED).
//
// The loop runs in float32, but every decision is the one the float64
// reference makes on the same inputs:
//   * each float32 decision statistic -- the floor test and the magnitude
//     spread test (decoder.py:146-148), the rounding test (:153-156) and the
//     re-prediction test (:160-163) -- is compared with its threshold together
//     with a bound on its float32 error; a bin whose statistic lies inside
//     that guard band is re-evaluated exactly: its D+1 values in float64 (line
//     0 from the float64 spectrum below, lines 1..D as single-bin DFTs of the
//     complex64 samples minus the float64 projection of the recovered set)
//     and the reference's decision on them (classify_values<double>);
//   * the recovered amplitudes are float64: every accepted amplitude is
//     S_0[b] conj(root[u_0]) with S_0 from a float64 transform of line 0 minus
//     the float64 projection (decoder.py:160), and the merge-by-sum, prune and
//     amp_sum run in float64 (driver.py:103-108) -- so the float64 values the
//     guard falls back to are the reference's own, not a drifting copy.
// Error bound of a float32 bin value (absolute, any line):
//   E_b = guard_coef * sqrt(sum |x|^2 over the D+1 lines) + KP * pabs[b]
//         (transform rounding, kappa_f u sqrt(log2 L + 1) ||x|| / L, and the
//          projection's: kappa_p u times the sum of |a| of the slots in bin b)
// plus the rounding of each statistic's own float32 evaluation.
#pragma once
// (included inside namespace fpssft)

constexpr float U32 = 5.9604644775390625e-08f;  // float32 unit roundoff, 2^-24
#ifndef FPSSFT_GUARD_KF
#define FPSSFT_GUARD_KF 6.0  // transform: kappa_f, in units of u sqrt(log2 L + 1) ||x|| / L
#endif
#ifndef FPSSFT_GUARD_KP
#define FPSSFT_GUARD_KP 6.0f  // projection: kappa_p, in units of u sum |a|
#endif
#ifndef FPSSFT_GUARD_CALIB
#define FPSSFT_GUARD_CALIB 0  // calibration builds: every candidate re-evaluated, errors recorded
#endif
constexpr float GUARD_KP = FPSSFT_GUARD_KP * U32;
constexpr double GUARD_KF = FPSSFT_GUARD_KF;     // Knobs::guard_coef = GUARD_KF * unit
constexpr int ST_FLAG = 4;                       // decision inside the guard band
constexpr unsigned short CAND_FLAG = 0x8000;     // candidate-list entry flagged at the magnitude test
#if FPSSFT_GUARD_CALIB == 2
// why decisions were flagged: [0] magnitude test, [1] phase too uncertain,
// [2] rint may round either way, [3] verify band, [4] round_tol band,
// [5] decodes attempted, [6] certain rejections by the bin map
__device__ unsigned long long g_guard_reason[8];
#define GUARD_REASON(i) atomicAdd(&g_guard_reason[i], 1ull)
#else
#define GUARD_REASON(i) do {} while (0)
#endif
#if FPSSFT_GUARD_CALIB
// largest |S_float32 - S_exact| / (unit bound) seen (float bits, positive)
__device__ unsigned int g_guard_calib_max;
__device__ unsigned long long g_guard_calib_count;
#endif

// Magnitude half of the 1-sparse test (bin_is_candidate, float32) plus the
// guard: *flag when |S_0| is within the error bound of the floor or the
// spread low - (1 - mag_tol) top is within (2 - mag_tol) bounds of 0.
template <bool PAD>
__device__ __forceinline__ bool bin_is_candidate_guarded(const cpx<float> *spec, const Geo &g,
                                                         int b, float mag_tol, float floor,
                                                         float Eb0, float *res, bool *flag) {
    const float q0 = cabs2(spec[padi<PAD>(b)]);
    float top = q0, low = q0;
#pragma unroll
    for (int i = 1; i < MAXD + 1; ++i) {
        if (i <= g.D) {
            const float qi = cabs2(spec[padi<PAD>(i * g.L + b)]);
            top = fmaxf(top, qi);
            low = fminf(low, qi);
        }
    }
    *res = top;
    const float c = 1.f - mag_tol;
    const bool ok = q0 > floor * floor && (mag_tol >= 1.f || low >= c * c * top);
    const float t = sqrtf(top), lo = sqrtf(low), s0 = sqrtf(q0);
    const float Eb = Eb0 + 2.f * U32 * t;
    *flag = fabsf(s0 - floor) <= Eb || (mag_tol < 1.f && fabsf(lo - c * t) <= (1.f + c) * Eb);
    if (*flag) GUARD_REASON(0);
    return ok;
}

// decode_candidate (float32) plus the guard: 1 rejected, 2 accepted, 3 guard
// (bin map) failed, ST_FLAG when float32 cannot tell.  A bin counts as
// accepted iff every rounding test and every re-prediction test passes
// (decoder.py:153-163) and its frequency maps back onto it (driver.py:
// 166-176); "rejected" and "guard failed" are the same outcome for the log
// and the recovered set.  So a test that fails beyond its error bound, or a
// certain m whose bin is not b, decides "rejected" whatever the uncertain
// statistics say -- noise bins decode to random m and are dismissed by the
// exact integer bin map -- and only a bin whose outcome hinges on a
// statistic inside its guard band is flagged.
template <bool PAD>
__device__ __forceinline__ int decode_candidate_guarded(const cpx<float> *spec, const Geo &g,
                                                        int b, const int *al, const int *ta,
                                                        const cpx<float> *roots, float round_tol,
                                                        float verify_tol, float Eb0, int *m) {
    const int L = g.L, D = g.D;
    cpx<float> s[MAXD + 1];
    float mg[MAXD + 1];
    float top = 0.f;
#pragma unroll
    for (int i = 0; i < MAXD + 1; ++i)
        if (i <= D) {
            s[i] = spec[padi<PAD>(i * L + b)];
            mg[i] = cabs(s[i]);
            top = fmaxf(top, mg[i]);
        }
    const float Eb = Eb0 + 2.f * U32 * top;
    const float inv2pi = 0.15915494309189533577f;
    bool fail_sure = false, round_unsure = false;
    int m_alt[MAXD];
    unsigned m_unsure = 0;  // coordinates whose rint may round the other way
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
        if (k < D) {
            const cpx<float> z = mulc(s[k + 1], s[0]);
            const float theta = atan2f(z.im, z.re);
            const float raw = (float)g.N[k] * theta * inv2pi;
            const float near = rintf(raw);
            const float d = fabsf(raw - near);
            m[k] = wrap_index((int)near, g.N[k]);
            // angle error <= asin(E/|S_k+1|) + asin(E/|S_0|) (+ atan2f's own);
            // asin(x) <= 1.02 x for x <= 1/4, else no useful bound
            const float dth = (mg[k + 1] > 4.f * Eb && mg[0] > 4.f * Eb)
                                  ? 1.02f * (Eb / mg[k + 1] + Eb / mg[0]) + 8.f * U32
                                  : 4.f;
            const float draw = (float)g.N[k] * (dth * inv2pi + 4.f * U32);
            // (d near 1/2 fails for either rounding when round_tol + draw < d)
            if (d > round_tol + draw) fail_sure = true;          // fails whatever the error
            else if (d >= round_tol - draw) round_unsure = true; // inside the band
            if (draw >= 0.5f) {
                m_unsure |= 0x80u;  // phase too uncertain to bound m
            } else if (d >= 0.5f - draw) {
                m_unsure |= 1u << k;
                m_alt[k] = wrap_index((int)near + (raw > near ? 1 : -1), g.N[k]);
            }
        }
    }
    GUARD_REASON(5);
    if (fail_sure) return 1;
    if (m_unsure & 0x80u) {
        GUARD_REASON(1);
        return ST_FLAG;
    }
    // the exact bin map: a frequency that does not map back onto b is
    // rejected (driver.py:166-176) -- for every m the rounding may give
    {
        bool maps = false;
        for (unsigned c = 0; c < (1u << D); ++c) {
            if (c & ~m_unsure) continue;
            int mc[MAXD];
#pragma unroll
            for (int k = 0; k < MAXD; ++k) mc[k] = (c >> k & 1u) ? m_alt[k] : m[k];
            maps = maps || bin_of(mc, g, al) == b;
        }
        if (!maps) {
            GUARD_REASON(6);
            return 3;
        }
    }
    if (m_unsure) {
        GUARD_REASON(2);
        return ST_FLAG;
    }
    const int u0 = phase_of(m, g, ta);
    const cpx<float> amp = mulc(s[0], roots[u0]);
    const float lim = verify_tol * mg[0];
    const float marg = 2.f * Eb + verify_tol * (Eb + 2.f * U32 * mg[0]) + 8.f * U32 * mg[0];
    bool verify_unsure = false;
#pragma unroll
    for (int i = 0; i < MAXD + 1; ++i) {
        if (i <= D) {
            const cpx<float> dv = amp * roots[phase_step(u0, i, m, g)] - s[i];
            const float r = cabs(dv);
            if (r > lim + marg) fail_sure = true;
            else if (r >= lim - marg) verify_unsure = true;
        }
    }
    if (fail_sure) return 1;
    if (verify_unsure) GUARD_REASON(3);
    else if (round_unsure) GUARD_REASON(4);
    if (verify_unsure || round_unsure) return ST_FLAG;
    return 2;
}

#ifndef FPSSFT_REEVAL_UNROLL
#define FPSSFT_REEVAL_UNROLL 2  // sample-loop unrolling of the exact re-evaluation (1: -0 %, 2: -1.7 %, 4: -0.4 %, 8: +7 %)
#endif
// Exact (float64) values of bin b on lines 1..D, as the team's partial sums:
// single-bin DFTs of the complex64 line samples (the reference's
// dft_forward(line)[b] = fft(line)[b] / L, transform.py:17-22) and the
// projection of the live slots that fall in bin b (project_onto_bins,
// decoder.py:172-191).  Every thread of the team (tid of nth) adds its share;
// dft[i-1] / prj[i-1] are this thread's partial sums for line i.
template <class AmpT, class RT>
__device__ __forceinline__ void exact_bin_partials(int b, const float2 *__restrict__ cube,
                                                   const Geo &g, const int *al, const int *ta,
                                                   RT roots64, int n_slots,
                                                   const int *slot_key,
                                                   const unsigned char *slot_live,
                                                   const cpx<AmpT> *amp64, int tid, int nth,
                                                   cpx<double> *dft, cpx<double> *prj,
                                                   const float2 *__restrict__ sline = nullptr,
                                                   int sG = 1) {
    const int L = g.L, D = g.D;
    const bool pow2 = (L & (L - 1)) == 0;
#pragma unroll
    for (int i = 0; i < MAXD; ++i) dft[i] = prj[i] = {0.0, 0.0};
    // n_k(l) = (alpha_k l + tau_k) mod N_k and l b mod L, advanced by nth per
    // step without division (every term < 2^31: the make_geo guard)
    int n[MAXD], step[MAXD];
#pragma unroll
    for (int k = 0; k < MAXD; ++k)
        if (k < D) {
            n[k] = (int)fastmod((unsigned)al[k] * (unsigned)tid + (unsigned)ta[k], g.magic[k],
                                (unsigned)g.N[k]);
            step[k] = (int)fastmod((unsigned)al[k] * (unsigned)nth, g.magic[k], (unsigned)g.N[k]);
        }
    const int wstep = (int)(((long long)nth * b) % L);
    int w = (int)(((long long)tid * b) % L);
    constexpr int kUnroll = FPSSFT_REEVAL_UNROLL;
#pragma unroll kUnroll
    for (int l = tid; l < L; l += nth) {
        const cpx<double> r = roots64[w];
        long long base = 0;
#pragma unroll
        for (int k = 0; k < MAXD; ++k)
            if (k < D) base += (long long)n[k] * g.stride[k];
#pragma unroll
        for (int i = 1; i < MAXD + 1; ++i) {
            if (i <= D) {
                const int k = i - 1;  // tau + e_k: coordinate k one further, wrapping
                const long long off = base + (n[k] + 1 == g.N[k] ? -(long long)n[k] * g.stride[k]
                                                                 : g.stride[k]);
                // sline (the STG kernels): the same sample from the staged lines
                const float2 x = sline != nullptr ? __ldg(sline + ((long long)i * L + l) * sG)
                                                  : __ldg(cube + off);
                const cpx<double> xv = {(double)x.x, (double)x.y};
                dft[k] = dft[k] + mulc(xv, r);
            }
        }
#pragma unroll
        for (int k = 0; k < MAXD; ++k)
            if (k < D) {
                n[k] += step[k];
                if (n[k] >= g.N[k]) n[k] -= g.N[k];
            }
        w += wstep;
        if (pow2) w &= L - 1;
        else if (w >= L) w -= L;
    }
    for (int s = tid; s < n_slots; s += nth) {
        if (!slot_live[s]) continue;
        int m[MAXD];
#pragma unroll
        for (int k = 0; k < MAXD; ++k)
            m[k] = k < D ? (slot_key[s] >> g.key_shift[k]) & g.key_mask[k] : 0;
        if (bin_of(m, g, al) != b) continue;
        const int u0 = phase_of(m, g, ta);
        const cpx<double> a = {(double)amp64[s].re, (double)amp64[s].im};
#pragma unroll
        for (int i = 1; i < MAXD + 1; ++i)
            if (i <= D) prj[i - 1] = prj[i - 1] + a * roots64[phase_step(u0, i, m, g)];
    }
}

// The exact re-evaluation of one flagged bin bf by a whole warp: the float64
// values of its D+1 lines (line 0 given, s0; lines 1..D from the samples and
// the float64 projection) and the reference's decision on them.  Out of line
// (FPSSFT_GUARD_NOINLINE): a rare path whose float64 atan2 / hypot code would
// otherwise sit inside the hot loop and crowd the instruction cache.  Every
// lane returns the same decision; *m gets the decoded frequency.
#ifndef FPSSFT_GUARD_NOINLINE
#define FPSSFT_GUARD_NOINLINE 0  // A/B: 1 measured slower (stack frame, spills)
#endif
#if FPSSFT_GUARD_NOINLINE
#define GUARD_REEVAL_INLINE __noinline__
#else
#define GUARD_REEVAL_INLINE __forceinline__
#endif
template <class AmpT, class RT, int LC, int DC>
__device__ GUARD_REEVAL_INLINE int exact_reeval_warp(int bf, const float2 *__restrict__ cube,
                                                     const Geo &g, const int *al, const int *ta,
                                                     RT roots64, int n_slots, const int *slot_key,
                                                     const unsigned char *slot_live,
                                                     const cpx<AmpT> *amp64, cpx<double> s0,
                                                     const Knobs &kn, double floor, int lane,
                                                     int *m, cpx<double> *S_out = nullptr,
                                                     const float2 *__restrict__ sline = nullptr) {
    Geo gc = g;  // the compile-time shape, for the callee's loops
    gc.L = LC;
    gc.D = DC;
    gc.nlines = DC + 1;
    cpx<double> dft[MAXD], prj[MAXD];
    exact_bin_partials<AmpT>(bf, cube, gc, al, ta, roots64, n_slots, slot_key, slot_live, amp64,
                             lane, 32, dft, prj, sline, kn.group);
    cpx<double> S[MAXD + 1];
    S[0] = s0;
#pragma unroll
    for (int i = 0; i < MAXD; ++i)
        if (i < DC)
            S[i + 1] = {warp_sum(dft[i].re) / (double)LC - warp_sum(prj[i].re),
                        warp_sum(dft[i].im) / (double)LC - warp_sum(prj[i].im)};
    if (S_out != nullptr)  // calibration builds: the exact values
        for (int i = 0; i <= DC; ++i) S_out[i] = S[i];
    cpx<double> ax;
    return classify_values<double, RT>(S, gc, bf, al, ta, roots64, kn.mag_tol, kn.round_tol,
                                       kn.verify_tol, floor, m, &ax);
}
