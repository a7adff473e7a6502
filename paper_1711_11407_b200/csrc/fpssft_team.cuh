// CTA-per-instance kernel with a compile-time shape (team of NT threads).
//
// The same loop as recover_warp_kernel for lines too long for one warp
// (config 4: L = 2048) or instances whose on-chip state is too large to keep
// many warps resident (config 5: L = 512, k_cap = 1024): NT threads own one
// instance and synchronise with block barriers.  Per iteration:
//   cp.async gather -> compile-time FFT (padded layout) -> projection of the
//   recovered set (warp match_any groups, warps applied in order) -> magnitude
//   test on every bin with block-scan compaction of candidates -> dense decode
//   of the candidates -> merge in candidate (= ascending bin) order -> residual
//   and amp_sum reductions -> termination.
// GUARD (float32 only): the decisions of the float64 reference on the same
// inputs (fpssft_guard.cuh) -- float64 slot amplitudes, a float64 transform
// of line 0 (by the warp the register FFTs leave idle), guard-band flags on
// every float32 decision statistic and exact re-evaluation of flagged bins.
// Included by fpssft.cu after the warp kernel (shares its helpers).
#pragma once
// (included inside namespace fpssft)
#ifndef TEAM_SORT_BITS
#define TEAM_SORT_BITS 11  // output counting-sort buckets (2048)
#endif
#ifndef FPSSFT_TEAM_REGFFT
#define FPSSFT_TEAM_REGFFT 1  // 512-point lines: per-warp register FFTs (regfft::)
#endif
#ifndef FPSSFT_TEAM_GUARD_THREADS
#define FPSSFT_TEAM_GUARD_THREADS 384  // guarded team kernel: threads per SM its registers allow
#endif
#ifndef FPSSFT_TEAM_PROJ_Q
#define FPSSFT_TEAM_PROJ_Q 2  // projection sub-rounds per ordered apply
#endif

struct TeamLayout {
    size_t spec, roots, slot_amp, slot_key, hash, slot_live;
    size_t x0d, roots64, pabs;                 // GUARD only
    size_t proj, cand;  // union: projection / classifier scratch
    size_t red, total;
    int H;
};

__host__ __device__ inline TeamLayout make_team_layout(int D, int L, int k_cap, int cs, int nt,
                                                       bool guard = false) {
    TeamLayout y;
    const int acs = guard ? 16 : cs;  // slot amplitude bytes (complex128 when guarded)
    size_t spec_bytes = (size_t)(D + 1) * (L + L / 16 + 1) * cs;  // padi() layout
    if (stage16_ok(D, L, cs, nt) && spec_bytes < (size_t)(D + 1) * L * 16)
        spec_bytes = (size_t)(D + 1) * L * 16;  // 16-byte staging slots (gather_lines_cg16)
    const size_t sort_bytes = ((size_t)1 << TEAM_SORT_BITS) * 4 + (size_t)k_cap * 4;
    size_t o = 0;
    y.H = 2 * k_cap;
    y.spec = o;      o = align16(o + (spec_bytes > sort_bytes ? spec_bytes : sort_bytes));
    y.roots = o;     o = align16(o + (size_t)L * cs);
    y.slot_amp = o;  o = align16(o + (size_t)k_cap * acs);
    y.slot_key = o;  o = align16(o + (size_t)k_cap * 4);
    y.hash = o;      o = align16(o + (size_t)y.H * 2);
    y.slot_live = o; o = align16(o + (size_t)k_cap);
    y.x0d = y.roots64 = y.pabs = o;
    if (guard) {
        y.x0d = o;     o = align16(o + (size_t)(L + L / 16 + 1) * 16);
        y.roots64 = o; o = align16(o + (size_t)L * 8);  // lo half of Roots64Split
        y.pabs = o;    o = align16(o + (size_t)L * 4);
    }
    // union: the projection's per-warp scratch (phases + amplitudes of 32
    // slots) / the classifier's candidate list
    const size_t u = o;
    y.proj = u;
    // (float32: per lane its contributions on the D+1 lines, guarded also a
    // float64 line-0 one and |a|)
    const size_t per_lane = cs == 16 ? (MAXD + 1) * 4 + acs
                                     : (size_t)(D + 1) * cs + (guard ? 16 + 4 : 0);
    const size_t a = align16(u + (size_t)(nt / 32) * 32 * per_lane);
    y.cand = u;      const size_t b = align16(u + (size_t)L * 2);
    o = a > b ? a : b;
    y.red = o;       o = align16(o + 64 * 8);  // 256 B of ints, then NW floats/doubles
    y.total = o;
    return y;
}

constexpr unsigned short U16_NONE = 0xFFFF;

template <class R, int LC, int DC, int NT, bool GUARD = false, bool STG = false>
__global__ void __launch_bounds__(NT, GUARD ? (FPSSFT_TEAM_GUARD_THREADS / NT > 1
                                                     ? FPSSFT_TEAM_GUARD_THREADS / NT : 1)
                                            : (512 / NT > 1 ? 512 / NT : 1))
    recover_team_kernel(const float2 *__restrict__ cubes, long long batch_stride, Geo g_in,
                        Knobs kn, const int *__restrict__ schedule,
                        const int *__restrict__ sched_index, int n_sched, OutPtrs out) {
    static_assert(!GUARD || (sizeof(R) == 4 && NT <= 512), "guarded mode: float32, NT <= 512");
    extern __shared__ __align__(16) unsigned char sm[];
    constexpr bool PAD = true;
    using A = typename std::conditional<GUARD, double, R>::type;  // slot amplitude type
    Geo g = g_in;
    g.L = LC;
    g.D = DC;
    g.nlines = DC + 1;
    constexpr int L = LC, D = DC, nl = DC + 1, NW = NT / 32;
    const TeamLayout lay = make_team_layout(D, L, kn.k_cap, (int)sizeof(cpx<R>), NT, GUARD);
    cpx<R> *spec = (cpx<R> *)(sm + lay.spec);
    cpx<R> *roots = (cpx<R> *)(sm + lay.roots);
    cpx<A> *slot_amp = (cpx<A> *)(sm + lay.slot_amp);
    int *slot_key = (int *)(sm + lay.slot_key);
    unsigned short *hash = (unsigned short *)(sm + lay.hash);
    unsigned char *slot_live = sm + lay.slot_live;
    [[maybe_unused]] cpx<double> *x0d = (cpx<double> *)(sm + lay.x0d);
    [[maybe_unused]] cpx<float> *roots_lo = (cpx<float> *)(sm + lay.roots64);
    [[maybe_unused]] const Roots64Split roots64{(const cpx<float> *)roots, roots_lo};
    [[maybe_unused]] float *pabs = (float *)(sm + lay.pabs);
    unsigned short *cand = (unsigned short *)(sm + lay.cand);
    int *ired = (int *)(sm + lay.red);
    R *rred = (R *)(sm + lay.red + 256);
    [[maybe_unused]] double *dred = (double *)(sm + lay.red + 256);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, H = lay.H;
    const long long inst = blockIdx.x;
    const float2 *cube = cube_base(cubes, (long long)inst, batch_stride, kn.group);
    int sidx = sched_index ? sched_index[inst] : 0;
    const bool sched_ok = sidx >= 0 && sidx < n_sched;
    if (!sched_ok) sidx = 0;
    const int *sched = schedule + (long long)sidx * kn.t_max * 2 * D;
    const R mag_tol = (R)kn.mag_tol, round_tol = (R)kn.round_tol, verify_tol = (R)kn.verify_tol;

    build_roots(roots, L);
    if constexpr (GUARD) build_roots_lo(roots_lo, L);
    for (int h = tid; h < H; h += NT) hash[h] = U16_NONE;
    __syncthreads();

    [[maybe_unused]] const float2 *sbase =
        (STG && !GUARD && kn.staged != nullptr)
            ? kn.staged + (long long)((int)inst / kn.group) * kn.staged_group_stride +
                  ((int)inst % kn.group)
            : nullptr;
    int n_slots = 0, stall = 0, it_run = 0;
    int term = sched_ok ? FPSSFT_TERM_MAX_ITERATIONS : -1;
    A amp_sum = (A)0;
    int nal[MAXD], nta[MAXD];
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
        nal[k] = k < D ? sched[k] : 0;
        nta[k] = k < D ? sched[D + k] : 0;
    }

    PCLK_DECL();
    for (int it = 0; it < kn.t_max && term != -1; ++it) {
        int al[MAXD], ta[MAXD];
#pragma unroll
        for (int k = 0; k < MAXD; ++k) {
            al[k] = nal[k];
            ta[k] = nta[k];
        }
        if (!line_params_ok(g, al, ta)) {
            term = -1;
            break;
        }
        it_run = it + 1;
        // staged lines: this iteration's samples of this instance (else nullptr)
        [[maybe_unused]] const float2 *sline =
            (STG && sizeof(R) == 4 && !GUARD && sbase != nullptr && it < kn.stage_T)
                ? sbase + (long long)it * (nl * L) * kn.group
                : nullptr;

        PCLK(0);
        // (1) gather + (2) DFT                                 driver.py:146-154
        bool staged = false;
        unsigned par = 0, dup = 0;
        if constexpr (sizeof(R) == 4) {
            bool reg_gather = false;
            // staged lines (fpssft_stage.cuh): this iteration's samples sit in
            // line order in HBM, kn.group instances per position
            const bool from_hbm = sline != nullptr;
            if (from_hbm) {
                for (int q = tid; q < nl * L; q += NT)
                    cp_async8((cpx<float> *)spec + padi<PAD>(q), sline + (long long)q * kn.group);
            } else if constexpr (stage16_ok(DC, LC, 8, NT)) {
                staged = g.off32;
                if (staged)
                    par = gather_lines_cg16<LC, DC, NT>((float4 *)spec, cube, g, al, ta, tid, &dup);
            } else if constexpr (FPSSFT_TEAM_GATHER_NC && DC != 0) {
                reg_gather = g.off32;
                if (reg_gather) gather_lines_nc<LC, DC, NT>(spec, cube, g, al, ta, tid);
            }
            if (!reg_gather && !staged && !from_hbm)
                gather_lines_async<LC, NT>(spec, cube, g, al, ta, tid, NT);
        } else {
            gather_lines<R, PAD>(spec, cube, g, al, ta, tid, NT);
        }
        if (it + 1 < kn.t_max) {
#pragma unroll
            for (int k = 0; k < MAXD; ++k) {
                nal[k] = k < D ? sched[(long long)(it + 1) * 2 * D + k] : 0;
                nta[k] = k < D ? sched[(long long)(it + 1) * 2 * D + D + k] : 0;
            }
            // (no L2 prefetch here: measured slower on config 5, 42.3 vs 38.2 ms)
        }
        if constexpr (GUARD)
            for (int b = tid; b < L; b += NT) pabs[b] = 0.f;
        if constexpr (sizeof(R) == 4) cp_async_wait_all();
        if constexpr (stage16_ok(DC, LC, (int)sizeof(cpx<R>), NT)) {
            if (staged)
                compact_stage16<LC, nl, NT, BlockTeam>((cpx<float> *)spec, par, dup, tid,
                                                       GUARD ? x0d : nullptr);
        }
        __syncthreads();
        if constexpr (GUARD) {
            if (!staged) {  // line 0's samples into the float64 buffer
                for (int l = tid; l < L; l += NT) {
                    const cpx<R> v = spec[padi<PAD>(l)];
                    x0d[padi<PAD>(l)] = {(double)v.re, (double)v.im};
                }
                __syncthreads();
            }
        }
        R my_energy;
        PCLK(2);
        constexpr bool REG512 = FPSSFT_TEAM_REGFFT && LC == 512 && sizeof(R) == 4 && NW >= nl;
        if constexpr (REG512) {
            // one warp per line, in registers (regfft::): no block barrier inside
            my_energy = regfft::fft512_lines_warp<NT>((cpx<float> *)spec, nl,
                                                      (const cpx<float> *)roots, tid);
            if constexpr (GUARD) {  // line 0 in float64 by the warp left idle, else after
                if (NW > nl && warp == NW - 1)
                    fft_static<double, LC, 1, 32, WarpTeam, Roots64Split>(x0d, roots64, lane);
            }
            __syncthreads();
            if constexpr (GUARD) {
                if (NW == nl) fft_static<double, LC, 1, NT, BlockTeam, Roots64Split>(x0d, roots64, tid);
            }
        } else if constexpr (FPSSFT_TEAM_REGFFT && LC == 2048 && sizeof(R) == 4 &&
                             NT >= 128 * nl && nl < 16) {
            // four warps per line, in registers, named barriers per line
            my_energy = regfft::fft2048_lines_team<NT>((cpx<float> *)spec, nl,
                                                       (const cpx<float> *)roots, tid);
            __syncthreads();
            if constexpr (GUARD) fft_static<double, LC, 1, NT, BlockTeam, Roots64Split>(x0d, roots64, tid);
        } else {
            my_energy = fft_static<R, LC, nl, NT, BlockTeam>(spec, roots, tid);
            if constexpr (GUARD) fft_static<double, LC, 1, NT, BlockTeam, Roots64Split>(x0d, roots64, tid);
        }
        PCLK(3);
        R noise_floor = (R)0;
        [[maybe_unused]] float Ef = 0.f;  // GUARD: transform part of the error bound
        if constexpr (GUARD) {
            Ef = (float)(kn.guard_coef * sqrt((double)block_sum(my_energy, rred)));
        } else if (sizeof(R) == 4 && kn.noise_coef > 0) {
            noise_floor = (R)kn.noise_coef * sqrt(block_sum(my_energy, rred));
        }

        // (3) construction-subtraction: NT slots per round, 32 per warp;
        //     slots sharing a bin inside a warp are summed by their lowest
        //     lane (match_any), and the warps apply their partial sums one
        //     after another -- a fixed order, so the result is deterministic
        //     without a sort.  GUARD: also the float64 line-0 projection and
        //     the bins' sum |a| (the projection's share of the error bound).
        if (n_slots > 0) {
            int *scr_u = (int *)(sm + lay.proj) + warp * 32 * (MAXD + 1);
            cpx<A> *scr_amp = (cpx<A> *)((int *)(sm + lay.proj) + NW * 32 * (MAXD + 1)) +
                              warp * 32;
            // Q sub-rounds of NT slots per round: the warps' ordered apply (NW-1
            // barriers) is paid once per Q * NT slots
            constexpr int Q = FPSSFT_TEAM_PROJ_Q;
#pragma unroll 1
            for (int c0 = 0; c0 < n_slots; c0 += Q * NT) {
                cpx<R> P[Q][MAXD + 1];
                [[maybe_unused]] cpx<double> P0[Q];
                [[maybe_unused]] float pa[Q];
                int bq[Q];
                bool leader[Q];
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    const int s = c0 + q * NT + tid;
                    const bool valid = s < n_slots && slot_live[s];
                    int b = -1 - lane;
                    if (q) __syncwarp();  // the previous sub-round's scratch is read
                    if constexpr (sizeof(R) == 4) {
                        // float32: every lane its slot's contribution on each
                        // line; shared memory only for bins hit twice
                        cpx<R> *scr_c = (cpx<R> *)(sm + lay.proj) + warp * 32 * nl;
                        [[maybe_unused]] cpx<double> *scr_c0 =
                            (cpx<double> *)(sm + lay.proj + (size_t)NW * 32 * nl * 8) + warp * 32;
                        [[maybe_unused]] float *scr_ca =
                            (float *)(sm + lay.proj + (size_t)NW * 32 * (nl * 8 + 16)) + warp * 32;
#pragma unroll
                        for (int i = 0; i < MAXD + 1; ++i) P[q][i] = {(R)0, (R)0};
                        if constexpr (GUARD) {
                            P0[q] = {0.0, 0.0};
                            pa[q] = 0.f;
                        }
                        if (valid) {
                            int m[MAXD];
                            unpack_key(slot_key[s], g, m);
                            b = bin_of(m, g, al);
                            const int u0 = phase_of(m, g, ta);
                            const cpx<A> aj = slot_amp[s];
                            const cpx<R> ar = {(R)aj.re, (R)aj.im};
#pragma unroll
                            for (int i = 0; i < MAXD + 1; ++i)
                                if (i < nl) P[q][i] = ar * roots[phase_step(u0, i, m, g)];
                            if constexpr (GUARD) {
                                P0[q] = cpx<double>{(double)aj.re, (double)aj.im} * roots64[u0];
                                pa[q] = cabs(ar);
                            }
                        }
                        const unsigned grp = __match_any_sync(FULL, b);
                        const bool multi = (grp & (grp - 1)) != 0;
                        leader[q] = valid && lane == __ffs(grp) - 1;
                        bq[q] = b;
                        if (__any_sync(FULL, valid && multi)) {
                            if (valid && multi && !leader[q]) {
#pragma unroll
                                for (int i = 0; i < MAXD + 1; ++i)
                                    if (i < nl) scr_c[i * 32 + lane] = P[q][i];
                                if constexpr (GUARD) {
                                    scr_c0[lane] = P0[q];
                                    scr_ca[lane] = pa[q];
                                }
                            }
                            __syncwarp();
                            if (leader[q] && multi)
                                for (unsigned rest = grp & (grp - 1); rest; rest &= rest - 1) {
                                    const int j = __ffs(rest) - 1;
#pragma unroll
                                    for (int i = 0; i < MAXD + 1; ++i)
                                        if (i < nl) P[q][i] = P[q][i] + scr_c[i * 32 + j];
                                    if constexpr (GUARD) {
                                        P0[q] = P0[q] + scr_c0[j];
                                        pa[q] += scr_ca[j];
                                    }
                                }
                        }
                        continue;
                    }
                    if (valid) {
                        int m[MAXD];
                        unpack_key(slot_key[s], g, m);
                        b = bin_of(m, g, al);
                        const int u0 = phase_of(m, g, ta);
#pragma unroll
                        for (int i = 0; i < MAXD + 1; ++i)
                            if (i < nl) scr_u[i * 32 + lane] = phase_step(u0, i, m, g);
                        scr_amp[lane] = slot_amp[s];
                    }
                    __syncwarp();
                    const unsigned grp = __match_any_sync(FULL, b);
                    leader[q] = valid && lane == __ffs(grp) - 1;
                    bq[q] = b;
#pragma unroll
                    for (int i = 0; i < MAXD + 1; ++i) P[q][i] = {(R)0, (R)0};
                    if constexpr (GUARD) {
                        P0[q] = {0.0, 0.0};
                        pa[q] = 0.f;
                    }
                    if (leader[q]) {
                        for (unsigned rest = grp; rest; rest &= rest - 1) {
                            const int j = __ffs(rest) - 1;
                            const cpx<A> aj = scr_amp[j];
                            const cpx<R> ar = {(R)aj.re, (R)aj.im};
#pragma unroll
                            for (int i = 0; i < MAXD + 1; ++i)
                                if (i < nl) P[q][i] = P[q][i] + ar * roots[scr_u[i * 32 + j]];
                            if constexpr (GUARD) {
                                const cpx<double> ad = {(double)aj.re, (double)aj.im};
                                P0[q] = P0[q] + ad * roots64[scr_u[j]];
                                pa[q] += cabs(ar);
                            }
                        }
                    }
                }
                const int nw_live = min(NW, (n_slots - c0 + 31) / 32);
                for (int w2 = 0; w2 < nw_live; ++w2) {
                    if (w2) __syncthreads();
                    if (warp == w2) {
#pragma unroll
                        for (int q = 0; q < Q; ++q)
                            if (leader[q]) {
#pragma unroll
                                for (int i = 0; i < MAXD + 1; ++i)
                                    if (i < nl)
                                        spec[padi<PAD>(i * L + bq[q])] =
                                            spec[padi<PAD>(i * L + bq[q])] - P[q][i];
                                if constexpr (GUARD) {
                                    x0d[padi<PAD>(bq[q])] = x0d[padi<PAD>(bq[q])] - P0[q];
                                    pabs[bq[q]] += pa[q];
                                }
                            }
                    }
                }
                __syncthreads();
            }
        }

        PCLK(4);
        // (4) magnitude test on every bin, candidates compacted in ascending
        //     order; the residual of non-candidate bins is folded in.  GUARD:
        //     bins inside the guard band join the list, flagged
        const A floor_a = max(max((A)kn.energy_floor_abs, (A)kn.energy_floor * amp_sum),
                              (A)noise_floor);
        const R floor = (R)floor_a;
        R resid = (R)0;
        int n_cand = 0;
        {
            // thread t tests the BPT consecutive bins [t BPT, (t+1) BPT): one
            // block scan of the per-thread counts keeps ascending order
            constexpr int BPT = (LC + NT - 1) / NT;
            unsigned okm = 0, flm = 0;
#pragma unroll
            for (int j = 0; j < BPT; ++j) {
                const int b = tid * BPT + j;
                R top = (R)0;
                bool ok = false, fl = false;
                if (b < L) {
                    if constexpr (GUARD)
                        ok = bin_is_candidate_guarded<PAD>((const cpx<float> *)spec, g, b,
                                                           (float)mag_tol, (float)floor,
                                                           Ef + GUARD_KP * pabs[b], (float *)&top,
                                                           &fl);
                    else
                        ok = bin_is_candidate<R, PAD>(spec, g, b, mag_tol, floor, &top);
                }
                if (!ok && !fl) resid = max(resid, top);
                okm |= (unsigned)(ok || fl) << j;
                flm |= (unsigned)fl << j;
            }
            int pos = block_exscan(__popc(okm), ired, &n_cand);
#pragma unroll
            for (int j = 0; j < BPT; ++j)
                if (okm >> j & 1)
                    cand[pos++] = (unsigned short)(tid * BPT + j) |
                                  (unsigned short)((flm >> j & 1) ? CAND_FLAG : 0);
        }
        __syncthreads();

        PCLK(5);
        // (5) decode + merge-by-sum, NT candidates per round in ascending bin
        //     order (driver.py:103-108); decode results stay in registers
        int n_acc = 0, n_cand_x = 0;
        [[maybe_unused]] A d_amp = (A)0;  // GUARD: this thread's change of amp_sum
        bool overflow = false;
#pragma unroll 1
        for (int c0 = 0; c0 < n_cand; c0 += NT) {
            PCLK(5);
            const int idx = c0 + tid;
            const int ce = idx < n_cand ? cand[idx] : -1;
            const int b = ce >= 0 ? (ce & ~(int)CAND_FLAG) : -1;
            int m[MAXD];
            cpx<R> a;
            int st = 0;
            if constexpr (GUARD) {
                const bool mflag = ce >= 0 && ((ce & CAND_FLAG) || FPSSFT_GUARD_CALIB == 1);
                if (b >= 0 && !mflag)
                    st = decode_candidate_guarded<PAD>((const cpx<float> *)spec, g, b, al, ta,
                                                       (const cpx<float> *)roots,
                                                       (float)round_tol, (float)verify_tol,
                                                       Ef + GUARD_KP * pabs[b], m);
                PCLK(9);
                const unsigned need = __ballot_sync(FULL, b >= 0 && (mflag || st == ST_FLAG));
#if FPSSFT_GUARD_CALIB == 2
                if (lane == 0 && need) atomicAdd(&g_guard_calib_count, (unsigned long long)__popc(need));
#endif
                // exact float64 re-evaluation of this warp's flagged bins, one
                // at a time by the whole warp (no block barrier)
                for (unsigned rest = need; rest; rest &= rest - 1) {
                    const int owner = __ffs(rest) - 1;
                    const int bf = __shfl_sync(FULL, b, owner);
                    int mx[MAXD];
                    [[maybe_unused]] cpx<double> S[MAXD + 1];
                    // every lane gets the same decision, the owner keeps it
                    const int sx = exact_reeval_warp<A, Roots64Split, LC, DC>(
                        bf, cube, g, al, ta, roots64, n_slots, slot_key, slot_live, slot_amp,
                        x0d[padi<PAD>(bf)], kn, (double)floor_a, lane, mx,
                        FPSSFT_GUARD_CALIB == 1 ? S : nullptr);
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
                                                  verify_tol, m, &a);
            }
            PCLK(10);
            int found = -1, key = 0;
            if (st == 2) {
                key = pack_key(m, g);
                found = hash16_find(hash, slot_key, H, key);
            }
            const int fresh = st == 2 && found < 0;
            int tot;  // packed counts: new slots, accepted (, candidates when guarded)
            int pre, tot_new, tot_acc;
            if constexpr (GUARD) {
                pre = block_exscan(fresh | ((st == 2) << 10) | ((st >= 1) << 20), ired, &tot);
                tot_new = tot & 0x3FF;
                tot_acc = (tot >> 10) & 0x3FF;
                n_cand_x += (tot >> 20) & 0x3FF;
                pre &= 0x3FF;
            } else {
                pre = block_exscan(fresh | ((st == 2) << 16), ired, &tot);
                tot_new = tot & 0xFFFF;
                tot_acc = tot >> 16;
                pre &= 0xFFFF;
            }
            if (n_slots + tot_new > kn.k_cap) {
                overflow = true;
                break;
            }
            if (st == 2) {
                cpx<A> av;
                if constexpr (GUARD) {  // the float64 amplitude (decoder.py:160)
                    const int u0 = phase_of(m, g, ta);
                    av = mulc(x0d[padi<PAD>(b)], roots64[u0]);
                    a = {(R)av.re, (R)av.im};
                } else {
                    av = a;
                }
                cpx<A> v = av;
                int s;
                if (fresh) {
                    s = n_slots + pre;
                    FPSSFT_CHECK(s < kn.k_cap);
                    slot_key[s] = key;
                    hash16_insert(hash, H, key, s);
                } else {
                    s = found;
                    v = slot_amp[s] + av;  // a pruned slot holds 0: entries.get(f, 0) + a
                }
                const A av_new = cabs(v);
                const bool keep = !(av_new <= (A)kn.amp_prune_tol);
                if constexpr (GUARD)  // amp_sum kept incrementally (float64)
                    d_amp += (keep ? av_new : (A)0) - (fresh ? (A)0 : cabs(slot_amp[s]));
                slot_amp[s] = keep ? v : cpx<A>{(A)0, (A)0};
                slot_live[s] = keep;
                const int u0 = phase_of(m, g, ta);  // driver.py:189-194
#pragma unroll
                for (int i = 0; i < MAXD + 1; ++i)
                    if (i < nl)
                        spec[padi<PAD>(i * L + b)] =
                            spec[padi<PAD>(i * L + b)] - a * roots[phase_step(u0, i, m, g)];
            }
            if (b >= 0) resid = max(resid, bin_residual<R, PAD>(spec, g, b));
            n_slots += tot_new;
            n_acc += tot_acc;
            __syncthreads();  // inserts visible to the next round's lookups
        }
        if constexpr (GUARD) n_cand = n_cand_x;
        if (overflow) {
            term = FPSSFT_TERM_K_CAP_OVERFLOW;
            if (tid == 0 && out.iter_stats) {
                int *st = out.iter_stats + (inst * kn.t_max + it) * 3;
                st[0] = n_cand;
                st[1] = 0;
                st[2] = n_cand;
            }
            break;
        }

        PCLK(6);
        // (6) amp_sum and (7) termination                   driver.py:108,196-204
        if constexpr (GUARD) {
            amp_sum += block_sum(d_amp, dred);
        } else {
            A my = (A)0;
            for (int s = tid; s < n_slots; s += NT)
                if (slot_live[s]) my += cabs(slot_amp[s]);
            amp_sum = block_sum(my, rred);
        }
        const R worst = block_max(resid, rred);  // |S|^2 (float) or |S| (double)
        stall = n_acc > 0 ? 0 : stall + 1;
        const R clean = (R)max((A)kn.energy_floor_abs, (A)kn.residual_stop * amp_sum);
        const bool is_clean = sizeof(R) == 8 ? worst <= clean : worst <= clean * clean;
        if (tid == 0 && out.iter_stats) {
            int *st = out.iter_stats + (inst * kn.t_max + it) * 3;
            st[0] = n_cand;
            st[1] = n_acc;
            st[2] = n_cand - n_acc;
        }
        __syncthreads();
        if (is_clean) {
            term = FPSSFT_TERM_RESIDUAL_CLEAN;
            break;
        }
        if (stall >= kn.stall_limit) {
            term = FPSSFT_TERM_STALL;
            break;
        }
    }

    PCLK(7);
    // ---- RecoveryReport: counting sort of the live keys on their top
    //      TEAM_SORT_BITS bits, then insertion sort inside the (short)
    //      buckets.  Fine buckets matter: clustered spectra (config 4's blobs)
    //      put dozens of entries in one 8-bit bucket, and a single thread's
    //      quadratic sort then held the whole CTA at the barrier.
    __syncthreads();
    constexpr int SB = TEAM_SORT_BITS, NB = 1 << SB;
    int *hist = (int *)spec;
    int *sslot = hist + NB;
    const int kb = g.key_bits_;
    const int shift = kb > SB ? kb - SB : 0;
    for (int i = tid; i < NB; i += NT) hist[i] = 0;
    __syncthreads();
    int my_live = 0;
    for (int s = tid; s < n_slots; s += NT)
        if (slot_live[s]) {
            ++my_live;
            atomicAdd(&hist[slot_key[s] >> shift], 1);
        }
    const int count = block_sum(my_live, ired);
    {   // exclusive scan of the bucket counts, NT at a time
        int carry = 0;
#pragma unroll 1
        for (int j0 = 0; j0 < NB; j0 += NT) {
            const int c = j0 + tid < NB ? hist[j0 + tid] : 0;
            int tot;
            const int pre = block_exscan(c, ired, &tot);
            if (j0 + tid < NB) hist[j0 + tid] = carry + pre;  // the bucket's fill cursor
            carry += tot;
            __syncthreads();
        }
    }
    for (int s = tid; s < n_slots; s += NT)
        if (slot_live[s]) {
            const int pos = atomicAdd(&hist[slot_key[s] >> shift], 1);
            FPSSFT_CHECK(pos >= 0 && pos < count);
            sslot[pos] = s;
        }
    __syncthreads();
    for (int bkt = tid; bkt < NB; bkt += NT) {
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
    __syncthreads();
    for (int r = tid; r < count; r += NT) {
        const int s = sslot[r];
        int m[MAXD];
        unpack_key(slot_key[s], g, m);
        int *fo = out.freqs + (inst * kn.k_cap + r) * D;
#pragma unroll
        for (int k = 0; k < MAXD; ++k)
            if (k < D) fo[k] = m[k];
        double *ao = out.amps + (inst * kn.k_cap + r) * 2;
        ao[0] = (double)slot_amp[s].re;
        ao[1] = (double)slot_amp[s].im;
    }
    if (tid == 0) {
        out.count[inst] = count;
        out.iterations[inst] = it_run;
        out.samples_used[inst] = (long long)it_run * nl * L;
        out.terminated_by[inst] = term;
    }
    PCLK(8);
    PCLK_FLUSH();
}
