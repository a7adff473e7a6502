// 512-point DFTs held in the registers of one warp (float32), shared by the
// re-synthesis kernel (inverse row transforms, fpssft_synth.cuh) and the team
// recovery kernel (forward line transforms of config 5, fpssft_team.cuh).
// 512 = 16 x 32: lane b holds x[32 a + b] (a = 0..15), a 16-point DFT over a in
// registers, twiddle e^{2 pi i b c / 512}, one shared-memory exchange (row
// stride 34, conflict-free both ways), a 16-point DFT over beta (b = 2 beta +
// h) and a radix-2 combine with the partner lane; lane (c, h) ends with
// X[c + 16 d + 256 h], d = 0..15.
#pragma once
// (included inside namespace fpssft)
#ifndef FPSSFT_FFT256_LEAN
#define FPSSFT_FFT256_LEAN 0  // A/B: 256-point lines, scale folded into twiddles, fma signs, static
                              // offsets (group +1.2 % from a spill, batch-major -0.8 %: off)
#endif
#ifndef FPSSFT_FFT256_TW_HOIST
#define FPSSFT_FFT256_TW_HOIST 0  // A/B: 256-point lines, first-stage twiddles held across lines
#endif
namespace regfft {

// constexpr e^{+2 pi i j / 16} and e^{+2 pi i j / 32}
__device__ __forceinline__ float2 w16(int j) {
    constexpr float C[16] = {1.0f, 0.92387953251128674f, 0.70710678118654752f, 0.38268343236508977f,
                             0.0f, -0.38268343236508977f, -0.70710678118654752f, -0.92387953251128674f,
                             -1.0f, -0.92387953251128674f, -0.70710678118654752f, -0.38268343236508977f,
                             0.0f, 0.38268343236508977f, 0.70710678118654752f, 0.92387953251128674f};
    return make_float2(C[j & 15], C[(j + 12) & 15]);  // (cos, sin): sin x = cos(x - pi/2)
}
__device__ __forceinline__ float2 w32(int j) {
    constexpr float C[32] = {
        1.0f, 0.98078528040323044f, 0.92387953251128674f, 0.83146961230254524f,
        0.70710678118654752f, 0.55557023301960218f, 0.38268343236508977f, 0.19509032201612826f,
        0.0f, -0.19509032201612826f, -0.38268343236508977f, -0.55557023301960218f,
        -0.70710678118654752f, -0.83146961230254524f, -0.92387953251128674f, -0.98078528040323044f,
        -1.0f, -0.98078528040323044f, -0.92387953251128674f, -0.83146961230254524f,
        -0.70710678118654752f, -0.55557023301960218f, -0.38268343236508977f, -0.19509032201612826f,
        0.0f, 0.19509032201612826f, 0.38268343236508977f, 0.55557023301960218f,
        0.70710678118654752f, 0.83146961230254524f, 0.92387953251128674f, 0.98078528040323044f};
    return make_float2(C[j & 31], C[(j + 24) & 31]);
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 mul_i(float2 a) { return make_float2(-a.y, a.x); }  // * (+i)

// X[k] = sum_n x[n] e^{+2 pi i n k / 4}
__device__ __forceinline__ void dft4(float2 &x0, float2 &x1, float2 &x2, float2 &x3) {
    const float2 t0 = cadd(x0, x2), t1 = csub(x0, x2), t2 = cadd(x1, x3), t3 = mul_i(csub(x1, x3));
    x0 = cadd(t0, t2);
    x2 = csub(t0, t2);
    x1 = cadd(t1, t3);
    x3 = csub(t1, t3);
}

// In place, natural order in and out: v[k] <- sum_n v[n] e^{+2 pi i n k / 16}
// (n = 4 n1 + n2, k = k1 + 4 k2: DFT-4 over n1, twiddle, DFT-4 over n2).
__device__ __forceinline__ void dft16(float2 *v) {
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) dft4(v[n2], v[4 + n2], v[8 + n2], v[12 + n2]);
    // v[4 k1 + n2] now holds Y[n2][k1]; twiddle by e^{2 pi i n2 k1 / 16}
#pragma unroll
    for (int n2 = 1; n2 < 4; ++n2)
#pragma unroll
        for (int k1 = 1; k1 < 4; ++k1) v[4 * k1 + n2] = cmul(v[4 * k1 + n2], w16(n2 * k1));
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
    // v[4 k1 + k2] holds X[k1 + 4 k2]: transpose the 4 x 4 index (registers only)
    float2 t[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) t[i] = v[i];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = t[4 * k1 + k2];
}

// Packed float32 pairs (sm_100 FADD2 / FMUL2 / FFMA2: one instruction per
// complex add, two per complex multiply; the (-y, x) swap of a multiply by i
// and the scalar broadcast fold into SASS operand modifiers).
typedef unsigned long long f32x2_t;
__device__ __forceinline__ f32x2_t pk2(float x, float y) {
    f32x2_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
    return r;
}
__device__ __forceinline__ float2 upk2(f32x2_t a) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(a));
    return r;
}
__device__ __forceinline__ float2 cadd_p(float2 a, float2 b) {
    f32x2_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
    return upk2(r);
}
__device__ __forceinline__ float2 csub_p(float2 a, float2 b) {
    f32x2_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
    return upk2(r);
}
// a * b = b.x (a.x, a.y) + b.y (-a.y, a.x): the data operand first, the
// broadcast factor second (the order ptxas folds into modifiers)
__device__ __forceinline__ float2 cmul_p(float2 a, float2 b) {
    f32x2_t t, r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.x)));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(-a.y, a.x)), "l"(pk2(b.y, b.y)), "l"(t));
    return upk2(r);
}
__device__ __forceinline__ void dft4_p(float2 &x0, float2 &x1, float2 &x2, float2 &x3) {
    const float2 t0 = cadd_p(x0, x2), t1 = csub_p(x0, x2), t2 = cadd_p(x1, x3),
                 t3 = mul_i(csub_p(x1, x3));
    x0 = cadd_p(t0, t2);
    x2 = csub_p(t0, t2);
    x1 = cadd_p(t1, t3);
    x3 = csub_p(t1, t3);
}
// dft16 with packed arithmetic (same index maps)
__device__ __forceinline__ void dft16_p(float2 *v) {
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) dft4_p(v[n2], v[4 + n2], v[8 + n2], v[12 + n2]);
#pragma unroll
    for (int n2 = 1; n2 < 4; ++n2)
#pragma unroll
        for (int k1 = 1; k1 < 4; ++k1) {
            if (n2 * k1 == 4)
                v[4 * k1 + n2] = mul_i(v[4 * k1 + n2]);
            else
                v[4 * k1 + n2] = cmul_p(v[4 * k1 + n2], w16(n2 * k1));
        }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4_p(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
    float2 t[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) t[i] = v[i];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = t[4 * k1 + k2];
}

// X[k] = sum_n v[n] e^{+2 pi i n k / 8}, in place, natural order (radix 2 x 4).
__device__ __forceinline__ void dft8(float2 *v) {
    float2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
    float2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    dft4(e0, e1, e2, e3);
    dft4(o0, o1, o2, o3);
    const float h = 0.70710678118654752f;
    const float2 t1 = make_float2(h * (o1.x - o1.y), h * (o1.x + o1.y));    // e^{i pi/4} o1
    const float2 t2 = make_float2(-o2.y, o2.x);                            // i o2
    const float2 t3 = make_float2(-h * (o3.x + o3.y), h * (o3.x - o3.y));  // e^{3 i pi/4} o3
    v[0] = cadd(e0, o0);
    v[4] = csub(e0, o0);
    v[1] = cadd(e1, t1);
    v[5] = csub(e1, t1);
    v[2] = cadd(e2, t2);
    v[6] = csub(e2, t2);
    v[3] = cadd(e3, t3);
    v[7] = csub(e3, t3);
}

// Forward 1/L-normalised DFTs of `nlines` 256-point lines (padded layout),
// one warp doing the lines one after another, in registers: 256 = 8 x 32.
// Lane b holds x[32 a + b] (a = 0..7): 8-point DFT over a, twiddle
// e^{2 pi i b k1 / 256}, one shared-memory exchange (rows of 33) inside the
// line's own padded region, then lane (k1, h) = (lane / 4, lane % 4) holds
// y[4 beta + h] (beta = 0..7) of row k1: 8-point DFT over beta, twiddle
// e^{2 pi i h k2a / 32}, and a 4-point DFT across the 4 lanes h by shuffles
// (lane h ends with k2b = h / 2 + 2 (h % 2)): X[k1 + 8 (k2a + 8 k2b)].
// Forward = conjugate of the inverse of the conjugate.  Returns this lane's
// share of sum |x|^2 over the input samples, like fft_static.
__device__ __forceinline__ float fft256_lines_warp(cpx<float> *spec, int nlines,
                                                   const cpx<float> *roots, int lane) {
    constexpr int PADL = 256 + 16, S = 33;
    float energy = 0.f;
    const int k1 = lane >> 2, h = lane & 3, k2b = (h >> 1) + 2 * (h & 1);
#if FPSSFT_FFT256_TW_HOIST
    float2 tw1[8];  // first-stage twiddles, loaded once for every line
#pragma unroll
    for (int c = 1; c < 8; ++c) {
        const cpx<float> r = roots[lane * c];
        tw1[c] = make_float2(r.re, r.im);
    }
#endif
#pragma unroll 1
    for (int line = 0; line < nlines; ++line) {
        float2 *base = (float2 *)(spec + line * PADL);
        float2 v[8];
        float el = 0.f;  // this line's share, then added (the assisted path's order)
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const int i = 32 * a + lane;
            const float2 x = base[i + (i >> 4)];
            el += x.x * x.x + x.y * x.y;
            v[a] = make_float2(x.x, -x.y);  // conjugate in
        }
        energy = line == 0 ? el : energy + el;
        dft8(v);
#pragma unroll
        for (int c = 1; c < 8; ++c) {
#if FPSSFT_FFT256_TW_HOIST
            v[c] = cmul(v[c], tw1[c]);
#else
            const cpx<float> r = roots[lane * c];
            v[c] = cmul(v[c], make_float2(r.re, r.im));
#endif
        }
        __syncwarp();  // the line's inputs are read before the exchange overwrites them
#pragma unroll
        for (int c = 0; c < 8; ++c) base[c * S + lane] = v[c];
        __syncwarp();
#pragma unroll
        for (int be = 0; be < 8; ++be) v[be] = base[k1 * S + 4 * be + h];
        dft8(v);
#if FPSSFT_FFT256_LEAN
        // the 1/256 (a power of two: exact) folded into the twiddles and v[0]
        const float inv = 1.f / 256.f;
        v[0] = make_float2(v[0].x * inv, v[0].y * inv);
#pragma unroll
        for (int d = 1; d < 8; ++d) {  // e^{2 pi i h d / 32} = roots[8 h d] (a runtime h)
            const cpx<float> r = roots[8 * h * d];
            v[d] = cmul(v[d], make_float2(r.re * inv, r.im * inv));
        }
        // 4-point DFT across lanes h (xor 2, then xor 1); x + p or p - x as
        // one fma with the lane's sign (exactly the same roundings)
        const float s2 = (h & 2) ? -1.f : 1.f, s1 = (h & 1) ? -1.f : 1.f;
#pragma unroll
        for (int d = 0; d < 8; ++d) {
            float2 x = v[d];
            float2 p = make_float2(__shfl_xor_sync(FULL, x.x, 2), __shfl_xor_sync(FULL, x.y, 2));
            x = make_float2(fmaf(s2, x.x, p.x), fmaf(s2, x.y, p.y));
            if (h == 3) x = mul_i(x);
            p = make_float2(__shfl_xor_sync(FULL, x.x, 1), __shfl_xor_sync(FULL, x.y, 1));
            v[d] = make_float2(fmaf(s1, x.x, p.x), fmaf(s1, x.y, p.y));
        }
        __syncwarp();  // every lane has read the exchange before outputs land in it
        // X[k], k = k1 + 8 (d + 8 k2b), at k + (k >> 4) = k1 + 68 k2b + 8 d + (d >> 1)
        float2 *ob = base + k1 + 68 * k2b;
#pragma unroll
        for (int d = 0; d < 8; ++d) ob[8 * d + (d >> 1)] = make_float2(v[d].x, -v[d].y);  // conj out
#else
#pragma unroll
        for (int d = 1; d < 8; ++d) {  // e^{2 pi i h d / 32} = roots[8 h d] (a runtime h)
            const cpx<float> r = roots[8 * h * d];
            v[d] = cmul(v[d], make_float2(r.re, r.im));
        }
#pragma unroll
        for (int d = 0; d < 8; ++d) {  // 4-point DFT across lanes h (xor 2, then xor 1)
            float2 x = v[d];
            float2 p = make_float2(__shfl_xor_sync(FULL, x.x, 2), __shfl_xor_sync(FULL, x.y, 2));
            x = (h & 2) ? csub(p, x) : cadd(x, p);
            if (h == 3) x = mul_i(x);
            p = make_float2(__shfl_xor_sync(FULL, x.x, 1), __shfl_xor_sync(FULL, x.y, 1));
            v[d] = (h & 1) ? csub(p, x) : cadd(x, p);
        }
        __syncwarp();  // every lane has read the exchange before outputs land in it
        const float inv = 1.f / 256.f;
#pragma unroll
        for (int d = 0; d < 8; ++d) {
            const int k = k1 + 8 * (d + 8 * k2b);
            base[k + (k >> 4)] = make_float2(v[d].x * inv, -v[d].y * inv);  // conjugate out
        }
#endif
        __syncwarp();
    }
    return energy;
}

// Forward 1/64-normalised DFT of one 64-point float64 line (padded layout,
// in place) by one warp, in registers: lane l holds x[l] and x[l + 32]; one
// radix-2 step in the lane (a = x[l] + x[l+32], b = (x[l] - x[l+32]) w^l,
// w = e^{-2 pi i / 64}), then the two 32-point DFTs (A -> X[2k], B -> X[2k+1])
// across the lanes by five decimation-in-frequency shuffle stages; lane p
// ends with A[bitrev5(p)], B[bitrev5(p)].  `roots` is any float64-exact
// table e^{+2 pi i j / 64}.
template <class RT>
__device__ __forceinline__ void fft64_line_f64(cpx<double> *x, RT roots, int lane) {
    const cpx<double> u = x[lane + (lane >> 4)], v = x[lane + 32 + ((lane + 32) >> 4)];
    const cpx<double> r0 = roots[lane];
    cpx<double> a = {u.re + v.re, u.im + v.im};
    const cpx<double> d = {u.re - v.re, u.im - v.im};
    cpx<double> b = mulc(d, r0);  // d e^{-2 pi i l / 64}
    // stage twiddles (loaded up front): the lower half of each 2h block
    // takes (x[p-h] - x[p]) W_{2h}^{p mod h}, the upper half x[p] + x[p+h];
    // branch-free: t = x[partner] + sgn x[p], times w (1 in the upper half)
    cpx<double> w[5];
#pragma unroll
    for (int st = 0; st < 5; ++st) {
        const int h = 16 >> st;
        w[st] = (lane & h) ? roots[(lane & (h - 1)) * (32 / h)] : cpx<double>{1.0, 0.0};
    }
#pragma unroll
    for (int st = 0; st < 5; ++st) {
        const int h = 16 >> st;
        const double sg = (lane & h) ? -1.0 : 1.0;
        const cpx<double> pa = {__shfl_xor_sync(FULL, a.re, h), __shfl_xor_sync(FULL, a.im, h)};
        const cpx<double> pb = {__shfl_xor_sync(FULL, b.re, h), __shfl_xor_sync(FULL, b.im, h)};
        a = mulc(cpx<double>{fma(sg, a.re, pa.re), fma(sg, a.im, pa.im)}, w[st]);
        b = mulc(cpx<double>{fma(sg, b.re, pb.re), fma(sg, b.im, pb.im)}, w[st]);
    }
    const int k = (int)(__brev((unsigned)lane) >> 27);  // bitrev5
    __syncwarp();  // every lane read its inputs before outputs land
    const double inv = 1.0 / 64.0;
    const int e0 = 2 * k, e1 = 2 * k + 1;
    x[e0 + (e0 >> 4)] = {a.re * inv, a.im * inv};
    x[e1 + (e1 >> 4)] = {b.re * inv, b.im * inv};
    __syncwarp();
}

// As fft256_lines_warp for a compile-time number of lines NL, all lines
// transformed together phase by phase: NL independent chains per phase for
// the scheduler to interleave, and each twiddle loaded once for every line.
template <int NL>
__device__ __forceinline__ float fft256_lines_joint(cpx<float> *spec, const cpx<float> *roots,
                                                    int lane) {
    constexpr int PADL = 256 + 16, S = 33;
    float energy = 0.f;
    const int k1 = lane >> 2, h = lane & 3, k2b = (h >> 1) + 2 * (h & 1);
    float2 *base = (float2 *)spec;
    float2 v[NL][8];
#pragma unroll
    for (int l = 0; l < NL; ++l)
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const int i = 32 * a + lane;
            const float2 x = base[l * PADL + i + (i >> 4)];
            energy += x.x * x.x + x.y * x.y;
            v[l][a] = make_float2(x.x, -x.y);  // conjugate in
        }
    float2 tw[8];
#pragma unroll
    for (int c = 1; c < 8; ++c) {
        const cpx<float> r = roots[lane * c];
        tw[c] = make_float2(r.re, r.im);
    }
#pragma unroll
    for (int l = 0; l < NL; ++l) {
        dft8(v[l]);
#pragma unroll
        for (int c = 1; c < 8; ++c) v[l][c] = cmul(v[l][c], tw[c]);
    }
    __syncwarp();  // the lines' inputs are read before the exchange overwrites them
#pragma unroll
    for (int l = 0; l < NL; ++l)
#pragma unroll
        for (int c = 0; c < 8; ++c) base[l * PADL + c * S + lane] = v[l][c];
    __syncwarp();
#pragma unroll
    for (int l = 0; l < NL; ++l)
#pragma unroll
        for (int be = 0; be < 8; ++be) v[l][be] = base[l * PADL + k1 * S + 4 * be + h];
#pragma unroll
    for (int d = 1; d < 8; ++d) {  // e^{2 pi i h d / 32} = roots[8 h d] (a runtime h)
        const cpx<float> r = roots[8 * h * d];
        tw[d] = make_float2(r.re, r.im);
    }
#pragma unroll
    for (int l = 0; l < NL; ++l) {
        dft8(v[l]);
#pragma unroll
        for (int d = 1; d < 8; ++d) v[l][d] = cmul(v[l][d], tw[d]);
    }
#pragma unroll
    for (int d = 0; d < 8; ++d) {  // 4-point DFTs across lanes h (xor 2, then xor 1)
        float2 x[NL], p[NL];
#pragma unroll
        for (int l = 0; l < NL; ++l) {
            x[l] = v[l][d];
            p[l] = make_float2(__shfl_xor_sync(FULL, x[l].x, 2), __shfl_xor_sync(FULL, x[l].y, 2));
        }
#pragma unroll
        for (int l = 0; l < NL; ++l) {
            x[l] = (h & 2) ? csub(p[l], x[l]) : cadd(x[l], p[l]);
            if (h == 3) x[l] = mul_i(x[l]);
            p[l] = make_float2(__shfl_xor_sync(FULL, x[l].x, 1), __shfl_xor_sync(FULL, x[l].y, 1));
        }
#pragma unroll
        for (int l = 0; l < NL; ++l) v[l][d] = (h & 1) ? csub(p[l], x[l]) : cadd(x[l], p[l]);
    }
    __syncwarp();  // every lane has read the exchange before outputs land in it
    const float inv = 1.f / 256.f;
#pragma unroll
    for (int l = 0; l < NL; ++l)
#pragma unroll
        for (int d = 0; d < 8; ++d) {
            const int k = k1 + 8 * (d + 8 * k2b);
            base[l * PADL + k + (k >> 4)] = make_float2(v[l][d].x * inv, -v[l][d].y * inv);
        }
    __syncwarp();
    return energy;
}

// Forward 1/L-normalised DFTs of `nlines` 512-point lines in the padded
// spectra layout (padi), one warp per line (warps >= nlines idle): the
// conjugate of the inverse transform of the conjugated line.  `roots` is the
// L = 512 table e^{2 pi i j / 512}.  Returns this thread's share of sum |x|^2
// over the input samples (each read once), like fft_static.  No block
// barrier inside: the caller synchronises before (inputs) and after (outputs).
template <int NT>
__device__ __forceinline__ float fft512_lines_warp(cpx<float> *spec, int nlines,
                                                   const cpx<float> *roots, int tid) {
    const int warp = tid >> 5, lane = tid & 31;
    const int cc = lane >> 1, h = lane & 1;
    float energy = 0.f;
    for (int line = warp; line < nlines; line += NT / 32) {
        float2 *base = (float2 *)(spec + line * (512 + 32));  // padi(line * 512)
        float2 v[16];
#pragma unroll
        for (int a = 0; a < 16; ++a) {
            const int i = 32 * a + lane;
            const float2 x = base[i + (i >> 4)];
            energy += x.x * x.x + x.y * x.y;
            v[a] = make_float2(x.x, -x.y);  // conjugate in
        }
        dft16(v);
#pragma unroll
        for (int c = 1; c < 16; ++c) {
            const cpx<float> r = roots[lane * c];
            v[c] = cmul(v[c], make_float2(r.re, r.im));
        }
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 16; ++c) base[34 * c + lane] = v[c];
        __syncwarp();
#pragma unroll
        for (int b = 0; b < 16; ++b) v[b] = base[34 * cc + 2 * b + h];
        dft16(v);
        __syncwarp();  // every lane has read the exchange before it is overwritten
        const float sg = h ? -1.f : 1.f, inv = 1.f / 512.f;
#pragma unroll
        for (int d = 0; d < 16; ++d) {
            const float2 tv = cmul(w32(d), v[d]);
            const float2 y = h ? tv : v[d];
            const float2 p = make_float2(__shfl_xor_sync(FULL, y.x, 1),
                                         __shfl_xor_sync(FULL, y.y, 1));
            const int k = cc + 16 * d + 256 * h;
            // conjugate out, 1/L (exact: a power of two)
            base[k + (k >> 4)] = make_float2(fmaf(sg, y.x, p.x) * inv, -fmaf(sg, y.y, p.y) * inv);
        }
    }
    return energy;
}

// Forward 1/L-normalised DFTs of `nlines` 2048-point lines (padded layout),
// 128 threads (4 warps) per line, in registers: 2048 = 16 x 128.  Thread t
// holds x[128 a + t] (a = 0..15): 16-point DFT over a, twiddle
// e^{2 pi i t c / 2048}, one shared-memory exchange (row stride 136) inside
// the line's own padded region, then 16 DFTs of 128 points: thread (c, q) =
// (t / 8, t % 8) holds z[8 mu + q] (mu = 0..15) of DFT c: 16-point DFT over mu,
// twiddle e^{2 pi i q d / 128}, and an 8-point DFT across the 8 lanes q by
// shuffles (decimation in frequency: lane q ends with output 16 bitrev3(q)
// + d).  Forward = conjugate of the inverse of the conjugate.  The 4 warps of
// a line meet at named barriers (ids 1..nlines); no block barrier inside.
__device__ __forceinline__ void bar_line(int id) {
    asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory");
}
template <int NT>
__device__ __forceinline__ float fft2048_lines_team(cpx<float> *spec, int nlines,
                                                    const cpx<float> *roots, int tid) {
    constexpr int PADL = 2048 + 128, S = 136;
    const int line = tid >> 7, t = tid & 127;
    float energy = 0.f;
    if (line >= nlines) return energy;
    float2 *base = (float2 *)(spec + line * PADL);
    float2 v[16];
#pragma unroll
    for (int a = 0; a < 16; ++a) {
        const int i = 128 * a + t;
        const float2 x = base[i + (i >> 4)];
        energy += x.x * x.x + x.y * x.y;
        v[a] = make_float2(x.x, -x.y);
    }
    dft16(v);
#pragma unroll
    for (int c = 1; c < 16; ++c) {
        const cpx<float> r = roots[t * c];
        v[c] = cmul(v[c], make_float2(r.re, r.im));
    }
    bar_line(1 + line);  // the line's inputs are read before the exchange overwrites them
#pragma unroll
    for (int c = 0; c < 16; ++c) base[c * S + t] = v[c];
    bar_line(1 + line);
    const int cq = t >> 3, q = t & 7;
#pragma unroll
    for (int mu = 0; mu < 16; ++mu) v[mu] = base[cq * S + 8 * mu + q];
    dft16(v);
#pragma unroll
    for (int d = 1; d < 16; ++d) {
        const cpx<float> r = roots[16 * q * d];
        v[d] = cmul(v[d], make_float2(r.re, r.im));
    }
    // 8-point DFT across lanes q (partners xor 4, 2, 1), positive exponent
    const cpx<float> r4 = roots[256 * (q & 3)], r2 = roots[512 * (q & 1)];
    const float2 w4 = make_float2(r4.re, r4.im), w2 = make_float2(r2.re, r2.im);
#pragma unroll
    for (int d = 0; d < 16; ++d) {
        float2 x = v[d];
        float2 p = make_float2(__shfl_xor_sync(FULL, x.x, 4), __shfl_xor_sync(FULL, x.y, 4));
        x = (q & 4) ? cmul(csub(p, x), w4) : cadd(x, p);
        p = make_float2(__shfl_xor_sync(FULL, x.x, 2), __shfl_xor_sync(FULL, x.y, 2));
        x = (q & 2) ? cmul(csub(p, x), w2) : cadd(x, p);
        p = make_float2(__shfl_xor_sync(FULL, x.x, 1), __shfl_xor_sync(FULL, x.y, 1));
        v[d] = (q & 1) ? csub(p, x) : cadd(x, p);
    }
    const int s = ((q & 1) << 2) | (q & 2) | ((q >> 2) & 1);  // bitrev3(q)
    bar_line(1 + line);  // every thread has read the exchange before outputs land in it
    const float inv = 1.f / 2048.f;
#pragma unroll
    for (int d = 0; d < 16; ++d) {
        const int k = cq + 16 * (d + 16 * s);
        base[k + (k >> 4)] = make_float2(v[d].x * inv, -v[d].y * inv);
    }
    return energy;
}

}  // namespace regfft
