// Re-synthesis of 2-D grids with 512-point rows (config 5: 512 x 512 images),
// float32: x(n0, n1) = sum_i a_i root_L[(c0 n0 m0_i + c1 n1 m1_i) mod L], the
// dense form of SyntheticSource.sample_many (reference core.py:176-217).
//
// One CTA per image, RC rows per chunk:
//   sparse part  V[r][m1] = sum over entries of column m1 (entry order) of
//                a * root_L[c0 n0 m0 mod L]  -- one thread per column, every
//                column written (zeros included), so V needs no clearing;
//   dense part   x[r][n1] = sum_m1 V[r][m1] e^{+2 pi i n1 m1 / 512} -- one
//                warp per row, in registers: m1 = 32a + b, n1 = c + 16d.
//                Lane b: 16-point DFT over a (in registers), twiddle
//                e^{2 pi i b c / 512} (per-lane constants), one shared-memory
//                exchange (stride 34: both sides conflict-free) to lanes
//                (c, h) = (lane/2, lane%2) holding b = 2 beta + h, 16-point
//                DFT over beta, radix-2 combine with the partner lane (shfl)
//                gives n1 = c + 16 d' + 256 h: every warp store writes two
//                full 128-byte lines, straight from registers.
// Shared-memory traffic per row: 3 x 4 KB (V read, exchange write + read),
// against 6 x 4 KB + twiddle loads for three radix-8 passes in shared memory.
// Bound: the HBM write of the grid (2 MiB per 512 x 512 frame).

// (included inside namespace fpssft)
namespace synth {

// helpers: regfft:: in fpssft_regfft.cuh
using namespace regfft;

#if FPSSFT_SYNTH_QUAD && !(FPSSFT_SYNTH_PAIR && FPSSFT_SYNTH_RC == 16 && FPSSFT_SYNTH_SPARSE == 0)
#error "FPSSFT_SYNTH_QUAD needs the row-pair dense part, 16-row chunks and the default sparse part"
#endif
#if FPSSFT_SYNTH_PACKED
#define SY_CMUL cmul_p
#define SY_CADD cadd_p
#define SY_CSUB csub_p
#define SY_DFT16 dft16_p
#else
#define SY_CMUL cmul
#define SY_CADD cadd
#define SY_CSUB csub
#define SY_DFT16 dft16
#endif

constexpr int VS = 544;  // row stride of V (cpx): holds the 16 x 34 exchange tile

template <int RC, int NT, bool DB>
__global__ void __launch_bounds__(NT, 512 / NT) synth512_kernel(const int *__restrict__ freqs,
                                                         const double *__restrict__ amps,
                                                         const int *__restrict__ counts, int k_cap,
                                                         Geo gc, float2 *out, long long out_stride) {
    constexpr int NL = 512, NW = NT / 32, RW = RC / NW;
    static_assert(RC % NW == 0 && NL % NT == 0, "whole rows per warp, whole column passes");
    extern __shared__ __align__(16) unsigned char sm[];
    const int L = gc.L, N0 = gc.N[0], c0 = gc.cof[0];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long inst = blockIdx.x;
    const int n = min(counts[inst], k_cap);
    size_t o = 0;
    float2 *V = (float2 *)(sm + o);      o = align16(o + (size_t)(DB ? 2 : 1) * RC * VS * 8);
    float2 *rootsL = (float2 *)(sm + o); o = align16(o + (size_t)L * 8);
    float2 *samp = (float2 *)(sm + o);   o = align16(o + (size_t)k_cap * 8);  // column-sorted
    int *sm0 = (int *)V;  // entry ids, set-up only: V is first written after the set-up
    int *ecol = (int *)(sm + o);         o = align16(o + (size_t)k_cap * 4);
    int *col_start = (int *)(sm + o);    o = align16(o + (size_t)(NL + 1) * 4);
    int *col_fill = (int *)(sm + o);     o = align16(o + (size_t)NL * 4);
    int *ired = (int *)(sm + o);

    for (int j = tid; j < L; j += NT) {
        double s, c;
        sincospi(2.0 * (double)j / (double)L, &s, &c);
        rootsL[j] = make_float2((float)c, (float)s);
    }
    for (int c = tid; c < NL; c += NT) col_fill[c] = 0;
    __syncthreads();
    for (int e = tid; e < n; e += NT) {
        const int c = freqs[(inst * k_cap + e) * 2 + 1];
        ecol[e] = c;
        atomicAdd(&col_fill[c], 1);
    }
    __syncthreads();
    int carry = 0;
    for (int j0 = 0; j0 < NL; j0 += NT) {  // column -> range of the column-sorted entries
        const int c = j0 + tid;
        const int cnt = c < NL ? col_fill[c] : 0;
        int tot;
        const int pre = block_exscan(cnt, ired, &tot);
        if (c < NL) {
            col_start[c] = carry + pre;
            col_fill[c] = carry + pre;
        }
        carry += tot;
    }
    if (tid == 0) col_start[NL] = carry;
    __syncthreads();
    // entry order inside a column is the input order (deterministic sums):
    // scatter by column, insertion-sort each (short) column, then gather the
    // entries' m0 and amplitude into column-sorted arrays
    for (int e = tid; e < n; e += NT) {
        const int c = ecol[e];
        const int pos = atomicAdd(&col_fill[c], 1);
        FPSSFT_CHECK(c >= 0 && c < NL && pos < n);
        sm0[pos] = e;  // sm0 holds entry ids for now
    }
    __syncthreads();
    for (int c = tid; c < NL; c += NT) {
        const int st = col_start[c], en = col_start[c + 1];
        for (int i = st + 1; i < en; ++i) {
            const int v = sm0[i];
            int j = i - 1;
            while (j >= st && sm0[j] > v) {
                sm0[j + 1] = sm0[j];
                --j;
            }
            sm0[j + 1] = v;
        }
    }
    __syncthreads();
    for (int p = tid; p < n; p += NT) {
        const long long src = inst * k_cap + sm0[p];
        samp[p] = make_float2((float)amps[src * 2], (float)amps[src * 2 + 1]);
        ecol[p] = freqs[src * 2];  // m0, column-sorted
    }
    __syncthreads();
#if FPSSFT_SYNTH_PAIR
    // column order: the 32 columns of each residue class c mod 16 ranked by
    // descending entry count (ties by column); position = rank * 16 + residue.
    // A half-warp then holds 16 distinct residues (its 64-bit stores into a
    // row of V hit 16 distinct bank pairs: conflict-free) of the same rank
    // (near-equal loop lengths).
    int *corder = col_fill;  // col_fill is free now
    for (int c = tid; c < NL; c += NT) {
        const int cnt = col_start[c + 1] - col_start[c];
        int rank = 0;
#pragma unroll 4
        for (int j = 0; j < NL / 16; ++j) {
            const int c2 = (c & 15) + 16 * j;
            const int cnt2 = col_start[c2 + 1] - col_start[c2];
            rank += (cnt2 > cnt) || (cnt2 == cnt && c2 < c);
        }
        corder[rank * 16 + (c & 15)] = c;
    }
    __syncthreads();
#else
    // columns by descending entry count (bucket min(count, 31)); the order
    // inside a bucket does not matter: one thread sums one column
    int *corder = col_fill;  // col_fill is free now
    if (tid < 32) ired[tid] = 0;
    __syncthreads();
    for (int c = tid; c < NL; c += NT)
        atomicAdd(&ired[31 - min(col_start[c + 1] - col_start[c], 31)], 1);
    __syncthreads();
    if (tid < 32) {  // exclusive scan of the 32 bucket sizes -> cursors
        const int v = ired[tid];
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, x, o);
            if (tid >= o) x += y;
        }
        ired[tid] = x - v;
    }
    __syncthreads();
    for (int c = tid; c < NL; c += NT)
        corder[atomicAdd(&ired[31 - min(col_start[c + 1] - col_start[c], 31)], 1)] = c;
    __syncthreads();
#endif
    // per-lane twiddles e^{2 pi i lane c / 512}, c = 0..15 (exact table phases)
    float2 tw[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) tw[c] = rootsL[lane * c * (L / NL)];
    const unsigned long long magicL = ~0ULL / (unsigned)L + 1ULL;
    float2 *img = out + inst * out_stride;
    // sparse part of chunk r0 into buffer Vb (every column, zeros included),
    // columns in descending entry count so the lanes of a warp run equally
    // long loops; each entry's RC row phasors a w^{u0 + r step} by recurrence
    // from the exact table value at the chunk's first row (|error| ~ RC ulp)
    auto sparse = [&](int r0, float2 *Vb) {
        // QUAD: chunk r0 holds rows (r0 / 4) + j + (N0 / 4) q
        const unsigned r0L = fastmod((unsigned)c0 * (unsigned)(FPSSFT_SYNTH_QUAD ? r0 >> 2 : r0),
                                     magicL, (unsigned)L);
        for (int i = 0; i < NL / NT; ++i) {
            // snake over the count-sorted columns: warp w takes group w of even
            // passes and group NW-1-w of odd ones, evening out the warps' loads
            const int g = (i & 1) ? NW - 1 - warp : warp;
            const int c = corder[i * NT + g * 32 + lane];
            float2 acc[RC];
#pragma unroll
            for (int r = 0; r < RC; ++r) acc[r] = make_float2(0.f, 0.f);
            const int en = col_start[c + 1];
            for (int p = col_start[c]; p < en; ++p) {
                const unsigned m0 = (unsigned)ecol[p];
                const unsigned step = fastmod((unsigned)c0 * m0, magicL, (unsigned)L);
                const unsigned u = fastmod(r0L * m0, magicL, (unsigned)L);
#if FPSSFT_SYNTH_SPARSE == 1  // A/B: packed pairs in the sparse part only
                float2 z = cmul_p(samp[p], rootsL[u]);
                const float2 ws = rootsL[step];
#pragma unroll
                for (int r = 0; r < RC; ++r) {
                    acc[r] = cadd_p(acc[r], z);
                    if (r + 1 < RC) z = cmul_p(z, ws);
                }
#elif FPSSFT_SYNTH_SPARSE == 2  // A/B: two interleaved phasor chains (rows r, r + 1 step by ws^2)
                float2 z = cmul(samp[p], rootsL[u]);
                const float2 ws = rootsL[step];
                float2 z1 = cmul(z, ws);
                const float2 ws2 = cmul(ws, ws);
#pragma unroll
                for (int r = 0; r < RC; r += 2) {
                    acc[r] = cadd(acc[r], z);
                    acc[r + 1] = cadd(acc[r + 1], z1);
                    if (r + 2 < RC) {
                        z = cmul(z, ws2);
                        z1 = cmul(z1, ws2);
                    }
                }
#elif FPSSFT_SYNTH_QUAD
                // rows n0 + j + (N0/4) q, j, q = 0..3: the quarter-period shift
                // multiplies an entry's phasor by i^(m0 q), a swap and signs
                // (per-entry constants), so one recurrence step serves 4 rows
                float2 z = cmul(samp[p], rootsL[u]);
                const float2 ws = rootsL[step];
                const bool sw = (m0 & 1u) != 0;
                const float sx = ((m0 + 1u) & 2u) ? -1.f : 1.f, sy = (m0 & 2u) ? -1.f : 1.f;
                const float s2 = sw ? -1.f : 1.f, sx3 = s2 * sx, sy3 = s2 * sy;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float tx = sw ? z.y : z.x, ty = sw ? z.x : z.y;
                    acc[j] = cadd(acc[j], z);
                    acc[4 + j] = make_float2(fmaf(sx, tx, acc[4 + j].x), fmaf(sy, ty, acc[4 + j].y));
                    acc[8 + j] = make_float2(fmaf(s2, z.x, acc[8 + j].x), fmaf(s2, z.y, acc[8 + j].y));
                    acc[12 + j] = make_float2(fmaf(sx3, tx, acc[12 + j].x), fmaf(sy3, ty, acc[12 + j].y));
                    if (j + 1 < 4) z = cmul(z, ws);
                }
#else
                float2 z = SY_CMUL(samp[p], rootsL[u]);
                const float2 ws = rootsL[step];
#pragma unroll
                for (int r = 0; r < RC; ++r) {
                    acc[r] = SY_CADD(acc[r], z);
                    if (r + 1 < RC) z = SY_CMUL(z, ws);
                }
#endif
            }
#pragma unroll
            for (int r = 0; r < RC; ++r) Vb[r * VS + c] = acc[r];
        }
    };
#if FPSSFT_SYNTH_PAIR
    // dense part of chunk r0 from buffer Vb: one warp per pair of rows.  First
    // stage (lane b, one row at a time) as above; second stage: lane (c, q) =
    // (lane % 16, lane / 16) holds all 32 values b of row q's column c (eight
    // 16-byte loads per 16 values, conflict-free per quarter warp), two
    // 16-point DFTs over the even and odd b and the radix-2 combine in its
    // own registers: no shuffles, and every warp store writes one whole
    // 128-byte line of each of the two rows.
    auto dense = [&](int r0, float2 *Vb) {
        static_assert(RW % 2 == 0, "row pairs");
#pragma unroll 1
        for (int rr = 0; rr < RW; rr += 2) {
            const int r = warp * RW + rr;
#pragma unroll 1
            for (int q = 0; q < 2; ++q) {
                float2 *Vr = Vb + (r + q) * VS;
                float2 v[16];
#pragma unroll
                for (int a = 0; a < 16; ++a) v[a] = Vr[32 * a + lane];
                SY_DFT16(v);
#pragma unroll
                for (int c = 1; c < 16; ++c) v[c] = SY_CMUL(v[c], tw[c]);
                __syncwarp();
#pragma unroll
                for (int c = 0; c < 16; ++c) Vr[34 * c + lane] = v[c];
            }
            __syncwarp();
            const int cc = lane & 15, q = lane >> 4;
            const float4 *X = (const float4 *)(Vb + (r + q) * VS + 34 * cc);
            float2 e[16], o[16];
#pragma unroll
            for (int b = 0; b < 16; ++b) {
                const float4 x = X[b];
                e[b] = make_float2(x.x, x.y);
                o[b] = make_float2(x.z, x.w);
            }
            SY_DFT16(e);
            SY_DFT16(o);
#if FPSSFT_SYNTH_QUAD
            const int rq = r + q;  // chunk row -> image row (r0 / 4) + rq % 4 + (N0 / 4) (rq / 4)
            float2 *row = img + (long long)((r0 >> 2) + (rq & 3) + (N0 >> 2) * (rq >> 2)) * NL + cc;
#else
            float2 *row = img + (long long)(r0 + r + q) * NL + cc;
#endif
#pragma unroll
            for (int d = 0; d < 16; ++d) {
                const float2 t = SY_CMUL(o[d], w32(d));
                __stcs(row + 16 * d, SY_CADD(e[d], t));
                __stcs(row + 16 * d + 256, SY_CSUB(e[d], t));
            }
        }
    };
#else
    // dense part of chunk r0 from buffer Vb: one warp per row
    auto dense = [&](int r0, float2 *Vb) {
#pragma unroll 1
        for (int rr = 0; rr < RW; ++rr) {
            const int r = warp * RW + rr;
            float2 *Vr = Vb + r * VS;
            float2 v[16];
#pragma unroll
            for (int a = 0; a < 16; ++a) v[a] = Vr[32 * a + lane];
            dft16(v);
#pragma unroll
            for (int c = 1; c < 16; ++c) v[c] = cmul(v[c], tw[c]);
            __syncwarp();
#pragma unroll
            for (int c = 0; c < 16; ++c) Vr[34 * c + lane] = v[c];
            __syncwarp();
            const int cc = lane >> 1, h = lane & 1;
#pragma unroll
            for (int b = 0; b < 16; ++b) v[b] = Vr[34 * cc + 2 * b + h];
            dft16(v);
            float2 *row = img + (long long)(r0 + r) * NL + cc + 256 * h;
            const float sg = h ? -1.f : 1.f;
#pragma unroll
            for (int d = 0; d < 16; ++d) {
                // lane h=1 holds E1 and sends t E1; lane h=0 holds E0 and sends E0:
                // out = E0 + t E1 (h=0) = p + y;  E0 - t E1 (h=1) = p - y
                const float2 tv = cmul(w32(d), v[d]);
                const float2 y = h ? tv : v[d];
                const float2 p = make_float2(__shfl_xor_sync(FULL, y.x, 1),
                                             __shfl_xor_sync(FULL, y.y, 1));
                __stcs(row + 16 * d, make_float2(fmaf(sg, y.x, p.x), fmaf(sg, y.y, p.y)));
            }
        }
    };
#endif
    // two V buffers: chunk k+1's sparse part and chunk k's dense part run in
    // the same phase, so one barrier per chunk and the sparse part's uneven
    // per-warp work is absorbed by the (even) dense work
    if constexpr (DB) {
        sparse(0, V);
        __syncthreads();
        for (int k = 0, r0 = 0; r0 < N0; ++k, r0 += RC) {
            if (r0 + RC < N0) sparse(r0 + RC, V + ((k + 1) & 1) * RC * VS);
            dense(r0, V + (k & 1) * RC * VS);
            __syncthreads();
        }
    } else {
        for (int r0 = 0; r0 < N0; r0 += RC) {
            sparse(r0, V);
            __syncthreads();
            dense(r0, V);
            __syncthreads();
        }
    }
}

}  // namespace synth
