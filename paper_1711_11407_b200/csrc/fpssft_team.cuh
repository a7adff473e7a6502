// CTA-per-instance kernel with a compile-time shape (team of NT threads).
//
// The same loop as recover_warp_kernel for lines too long for one warp
// (config 4: L = 2048) or instances whose on-chip state is too large to keep
// many warps resident (config 5: L = 512, k_cap = 1024): NT threads own one
// instance and synchronise with block barriers.  Per iteration:
//   cp.async gather -> compile-time FFT (padded layout) -> projection of the
//   recovered set (counting sort by bin, 16-bit scratch) -> magnitude test on
//   every bin with block-scan compaction of candidates -> dense decode of the
//   candidates -> merge in candidate (= ascending bin) order -> residual and
//   amp_sum reductions -> termination.
// Included by fpssft.cu after the warp kernel (shares its helpers).
#pragma once
// (included inside namespace fpssft)
#ifndef TEAM_SORT_BITS
#define TEAM_SORT_BITS 11  // output counting-sort buckets (2048)
#endif
#ifndef FPSSFT_TEAM_REGFFT
#define FPSSFT_TEAM_REGFFT 1  // 512-point lines: per-warp register FFTs (regfft::)
#endif
#ifndef FPSSFT_TEAM_PROJ_Q
#define FPSSFT_TEAM_PROJ_Q 2  // projection sub-rounds per ordered apply (match_any path)
#endif
#ifndef FPSSFT_TEAM_PROJ
#define FPSSFT_TEAM_PROJ 1  // projection: 1 = warp match_any + ordered apply, 0 = counting sort
#endif

struct TeamLayout {
    size_t spec, roots, slot_amp, slot_key, hash, slot_live;
    size_t bin_start, bin_fill, seg, slot_bin, slot_u0;  // projection scratch (union A)
    size_t cand;                                         // classifier scratch (union B)
    size_t red, total;
    int H;
};

__host__ __device__ inline TeamLayout make_team_layout(int D, int L, int k_cap, int cs, int nt) {
    TeamLayout y;
    size_t spec_bytes = (size_t)(D + 1) * (L + L / 16 + 1) * cs;  // padi() layout
    if (stage16_ok(D, L, cs, nt) && spec_bytes < (size_t)(D + 1) * L * 16)
        spec_bytes = (size_t)(D + 1) * L * 16;  // 16-byte staging slots (gather_lines_cg16)
    const size_t sort_bytes = ((size_t)1 << TEAM_SORT_BITS) * 4 + (size_t)k_cap * 4;
    size_t o = 0;
    y.H = 2 * k_cap;
    y.spec = o;      o = align16(o + (spec_bytes > sort_bytes ? spec_bytes : sort_bytes));
    y.roots = o;     o = align16(o + (size_t)L * cs);
    y.slot_amp = o;  o = align16(o + (size_t)k_cap * cs);
    y.slot_key = o;  o = align16(o + (size_t)k_cap * 4);
    y.hash = o;      o = align16(o + (size_t)y.H * 2);
    y.slot_live = o; o = align16(o + (size_t)k_cap);
    const size_t u = o;
    y.bin_start = u; size_t a = align16(u + (size_t)(L + 1) * 2);
    y.bin_fill = a;  a = align16(a + (size_t)L * 4);
    y.seg = a;       a = align16(a + (size_t)k_cap * 2);
    y.slot_bin = a;  a = align16(a + (size_t)k_cap * 2);
    y.slot_u0 = a;   a = align16(a + (size_t)k_cap * 2);
    y.cand = u;      size_t b = align16(u + (size_t)L * 2);
    // the match_any projection's per-warp scratch also lives in this union
    const size_t c = align16(u + (size_t)(nt / 32) * 32 * ((MAXD + 1) * 4 + cs));
    o = b > c ? b : c;
    if (!FPSSFT_TEAM_PROJ) o = o > a ? o : a;  // the counting-sort projection's scratch
    y.red = o;       o = align16(o + 64 * 8);
    y.total = o;
    return y;
}

constexpr unsigned short U16_NONE = 0xFFFF;

template <class R, int LC, int DC, int NT>
__global__ void __launch_bounds__(NT, (512 / NT > 1 ? 512 / NT : 1)) recover_team_kernel(const float2 *__restrict__ cubes,
                                                             long long batch_stride, Geo g_in,
                                                             Knobs kn,
                                                             const int *__restrict__ schedule,
                                                             const int *__restrict__ sched_index,
                                                             int n_sched, OutPtrs out) {
    extern __shared__ __align__(16) unsigned char sm[];
    constexpr bool PAD = true;
    Geo g = g_in;
    g.L = LC;
    g.D = DC;
    g.nlines = DC + 1;
    constexpr int L = LC, D = DC, nl = DC + 1;
    const TeamLayout lay = make_team_layout(D, L, kn.k_cap, (int)sizeof(cpx<R>), NT);
    cpx<R> *spec = (cpx<R> *)(sm + lay.spec);
    cpx<R> *roots = (cpx<R> *)(sm + lay.roots);
    cpx<R> *slot_amp = (cpx<R> *)(sm + lay.slot_amp);
    int *slot_key = (int *)(sm + lay.slot_key);
    unsigned short *hash = (unsigned short *)(sm + lay.hash);
    unsigned char *slot_live = sm + lay.slot_live;
    [[maybe_unused]] unsigned short *bin_start = (unsigned short *)(sm + lay.bin_start);
    [[maybe_unused]] unsigned short *bin_fill = (unsigned short *)(sm + lay.bin_fill);
    [[maybe_unused]] unsigned short *seg = (unsigned short *)(sm + lay.seg);
    [[maybe_unused]] unsigned short *slot_bin = (unsigned short *)(sm + lay.slot_bin);
    [[maybe_unused]] unsigned short *slot_u0 = (unsigned short *)(sm + lay.slot_u0);
    unsigned short *cand = (unsigned short *)(sm + lay.cand);
    int *ired = (int *)(sm + lay.red);
    R *rred = (R *)(sm + lay.red + 256);

    const int tid = threadIdx.x, H = lay.H;
    const long long inst = blockIdx.x;
    const float2 *cube = cube_base(cubes, (long long)inst, batch_stride, kn.group);
    int sidx = sched_index ? sched_index[inst] : 0;
    const bool sched_ok = sidx >= 0 && sidx < n_sched;
    if (!sched_ok) sidx = 0;
    const int *sched = schedule + (long long)sidx * kn.t_max * 2 * D;
    const R mag_tol = (R)kn.mag_tol, round_tol = (R)kn.round_tol, verify_tol = (R)kn.verify_tol;
    const R prune = (R)kn.amp_prune_tol;

    build_roots(roots, L);
    for (int h = tid; h < H; h += NT) hash[h] = U16_NONE;
    __syncthreads();

    int n_slots = 0, stall = 0, it_run = 0;
    int term = sched_ok ? FPSSFT_TERM_MAX_ITERATIONS : -1;
    R amp_sum = (R)0;
    int nal[MAXD], nta[MAXD];
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
        nal[k] = k < D ? sched[k] : 0;
        nta[k] = k < D ? sched[D + k] : 0;
    }

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

        // (1) gather + (2) DFT                                 driver.py:146-154
        bool staged = false;
        unsigned par = 0, dup = 0;
        if constexpr (sizeof(R) == 4) {
            bool reg_gather = false;
            if constexpr (stage16_ok(DC, LC, 8, NT)) {
                staged = g.off32;
                if (staged)
                    par = gather_lines_cg16<LC, DC, NT>((float4 *)spec, cube, g, al, ta, tid, &dup);
            } else if constexpr (FPSSFT_TEAM_GATHER_NC && DC != 0) {
                reg_gather = g.off32;
                if (reg_gather) gather_lines_nc<LC, DC, NT>(spec, cube, g, al, ta, tid);
            }
            if (!reg_gather && !staged) gather_lines_async<LC, NT>(spec, cube, g, al, ta, tid, NT);
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
        if constexpr (sizeof(R) == 4) cp_async_wait_all();
        if constexpr (stage16_ok(DC, LC, (int)sizeof(cpx<R>), NT)) {
            if (staged) compact_stage16<LC, nl, NT, BlockTeam>((cpx<float> *)spec, par, dup, tid);
        }
        __syncthreads();
        R my_energy;
        if constexpr (FPSSFT_TEAM_REGFFT && LC == 512 && sizeof(R) == 4 && NT / 32 >= nl) {
            // one warp per line, in registers (regfft::): no block barrier inside
            my_energy = regfft::fft512_lines_warp<NT>((cpx<float> *)spec, nl,
                                                      (const cpx<float> *)roots, tid);
            __syncthreads();
        } else if constexpr (FPSSFT_TEAM_REGFFT && LC == 2048 && sizeof(R) == 4 &&
                             NT >= 128 * nl && nl < 16) {
            // four warps per line, in registers, named barriers per line
            my_energy = regfft::fft2048_lines_team<NT>((cpx<float> *)spec, nl,
                                                       (const cpx<float> *)roots, tid);
            __syncthreads();
        } else {
            my_energy = fft_static<R, LC, nl, NT, BlockTeam>(spec, roots, tid);
        }
        R noise_floor = (R)0;
        if (sizeof(R) == 4 && kn.noise_coef > 0)
            noise_floor = (R)kn.noise_coef * sqrt(block_sum(my_energy, rred));

        // (3) construction-subtraction
#if FPSSFT_TEAM_PROJ == 1
        //     NT slots per round, 32 per warp; slots sharing a bin inside a
        //     warp are summed by their lowest lane (match_any), and the warps
        //     apply their partial sums one after another -- a fixed order, so
        //     the result is deterministic without a sort
        if (n_slots > 0) {
            constexpr int NW = NT / 32;
            const int warp = tid >> 5, lane = tid & 31;
            int *scr_u = (int *)(sm + lay.bin_start) + warp * 32 * (MAXD + 1);
            cpx<R> *scr_amp = (cpx<R> *)((int *)(sm + lay.bin_start) + NW * 32 * (MAXD + 1)) +
                              warp * 32;
            // Q sub-rounds of NT slots per round: the warps' ordered apply (NW-1
            // barriers) is paid once per Q * NT slots
            constexpr int Q = FPSSFT_TEAM_PROJ_Q;
#pragma unroll 1
            for (int c0 = 0; c0 < n_slots; c0 += Q * NT) {
                cpx<R> P[Q][MAXD + 1];
                int bq[Q];
                bool leader[Q];
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    const int s = c0 + q * NT + tid;
                    const bool valid = s < n_slots && slot_live[s];
                    int b = -1 - lane;
                    if (q) __syncwarp();  // the previous sub-round's scratch is read
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
                    if (leader[q]) {
                        for (unsigned rest = grp; rest; rest &= rest - 1) {
                            const int j = __ffs(rest) - 1;
                            const cpx<R> aj = scr_amp[j];
#pragma unroll
                            for (int i = 0; i < MAXD + 1; ++i)
                                if (i < nl) P[q][i] = P[q][i] + aj * roots[scr_u[i * 32 + j]];
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
                            }
                    }
                }
                __syncthreads();
            }
        }
#else
        //     counting sort of the live slots by
        //     bin, per-bin sums in slot order (deterministic, no float atomics)
        if (n_slots > 0) {
            int *fill = (int *)bin_fill;
            for (int b = tid; b < L; b += NT) fill[b] = 0;
            __syncthreads();
            for (int s = tid; s < n_slots; s += NT) {
                unsigned short bb = U16_NONE;
                if (slot_live[s]) {
                    int m[MAXD];
                    unpack_key(slot_key[s], g, m);
                    const int b = bin_of(m, g, al);
                    bb = (unsigned short)b;
                    slot_u0[s] = (unsigned short)phase_of(m, g, ta);
                    atomicAdd(&fill[b], 1);
                }
                slot_bin[s] = bb;
            }
            __syncthreads();
            int carry = 0;
#pragma unroll 1
            for (int j0 = 0; j0 < L; j0 += NT) {
                const int b = j0 + tid;
                const int c = b < L ? fill[b] : 0;
                int tot;
                const int pre = block_exscan(c, ired, &tot);
                if (b < L) {
                    bin_start[b] = (unsigned short)(carry + pre);
                    fill[b] = 0;
                }
                carry += tot;
            }
            if (tid == 0) bin_start[L] = (unsigned short)carry;
            __syncthreads();
            for (int s = tid; s < n_slots; s += NT) {
                const unsigned short bb = slot_bin[s];
                if (bb != U16_NONE) seg[bin_start[bb] + atomicAdd(&fill[bb], 1)] = (unsigned short)s;
            }
            __syncthreads();
            for (int b = tid; b < L; b += NT) {
                const int st = bin_start[b], en = bin_start[b + 1];
                if (en == st) continue;
                for (int i = st + 1; i < en; ++i) {  // short segments: insertion sort
                    const unsigned short v = seg[i];
                    int j = i - 1;
                    while (j >= st && seg[j] > v) {
                        seg[j + 1] = seg[j];
                        --j;
                    }
                    seg[j + 1] = v;
                }
                cpx<R> P[MAXD + 1];
#pragma unroll
                for (int i = 0; i < MAXD + 1; ++i) P[i] = {(R)0, (R)0};
                for (int p = st; p < en; ++p) {
                    const int s = seg[p];
                    int m[MAXD];
                    unpack_key(slot_key[s], g, m);
                    const cpx<R> as = slot_amp[s];
                    const int u0 = slot_u0[s];
#pragma unroll
                    for (int i = 0; i < MAXD + 1; ++i)
                        if (i < nl) P[i] = P[i] + as * roots[phase_step(u0, i, m, g)];
                }
#pragma unroll
                for (int i = 0; i < MAXD + 1; ++i)
                    if (i < nl) spec[padi<PAD>(i * L + b)] = spec[padi<PAD>(i * L + b)] - P[i];
            }
            __syncthreads();
        }

#endif

        // (4) magnitude test on every bin, candidates compacted in ascending
        //     order; the residual of non-candidate bins is folded in
        const R floor =
            max(max((R)kn.energy_floor_abs, (R)kn.energy_floor * amp_sum), noise_floor);
        R resid = (R)0;
        int n_cand = 0;
        {
            // thread t tests the BPT consecutive bins [t BPT, (t+1) BPT): one
            // block scan of the per-thread counts keeps ascending order
            constexpr int BPT = (LC + NT - 1) / NT;
            unsigned okm = 0;
#pragma unroll
            for (int j = 0; j < BPT; ++j) {
                const int b = tid * BPT + j;
                R top = (R)0;
                const bool ok = b < L && bin_is_candidate<R, PAD>(spec, g, b, mag_tol, floor, &top);
                if (!ok) resid = max(resid, top);
                okm |= (unsigned)ok << j;
            }
            int pos = block_exscan(__popc(okm), ired, &n_cand);
#pragma unroll
            for (int j = 0; j < BPT; ++j)
                if (okm >> j & 1) cand[pos++] = (unsigned short)(tid * BPT + j);
        }
        __syncthreads();

        // (5) decode + merge-by-sum, NT candidates per round in ascending bin
        //     order (driver.py:103-108); decode results stay in registers
        int n_acc = 0;
        bool overflow = false;
#pragma unroll 1
        for (int c0 = 0; c0 < n_cand; c0 += NT) {
            const int idx = c0 + tid;
            const int b = idx < n_cand ? cand[idx] : -1;
            int m[MAXD];
            cpx<R> a;
            int st = 0;
            if (b >= 0)
                st = decode_candidate<R, PAD>(spec, g, b, al, ta, roots, round_tol, verify_tol, m, &a);
            int found = -1, key = 0;
            if (st == 2) {
                key = pack_key(m, g);
                found = hash16_find(hash, slot_key, H, key);
            }
            const int fresh = st == 2 && found < 0;
            int tot;  // low 16 bits: new slots, high: accepted
            const int pre = block_exscan(fresh | ((st == 2) << 16), ired, &tot);
            const int tot_new = tot & 0xFFFF;
            if (n_slots + tot_new > kn.k_cap) {
                overflow = true;
                break;
            }
            if (st == 2) {
                cpx<R> v = a;
                int s;
                if (fresh) {
                    s = n_slots + (pre & 0xFFFF);
                    slot_key[s] = key;
                    hash16_insert(hash, H, key, s);
                } else {
                    s = found;
                    v = slot_amp[s] + a;  // a pruned slot holds 0: entries.get(f, 0) + a
                }
                const bool keep = !(cabs(v) <= prune);
                slot_amp[s] = keep ? v : cpx<R>{(R)0, (R)0};
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
            n_acc += tot >> 16;
            __syncthreads();  // inserts visible to the next round's lookups
        }
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

        // (6) amp_sum and (7) termination                   driver.py:108,196-204
        R my = (R)0;
        for (int s = tid; s < n_slots; s += NT)
            if (slot_live[s]) my += cabs(slot_amp[s]);
        amp_sum = block_sum(my, rred);
        const R worst = block_max(resid, rred);  // |S|^2 (float) or |S| (double)
        stall = n_acc > 0 ? 0 : stall + 1;
        const R clean = max((R)kn.energy_floor_abs, (R)kn.residual_stop * amp_sum);
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
        if (slot_live[s]) sslot[atomicAdd(&hist[slot_key[s] >> shift], 1)] = s;
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
}

