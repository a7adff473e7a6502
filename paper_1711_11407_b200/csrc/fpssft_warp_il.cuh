// Interleaved warp-per-instance kernel: each warp owns NI instances at once
// and software-pipelines them.  While one instance's line gather for its next
// iteration is in flight (cp.async group), the warp runs the FFT / classify /
// merge of another instance.  Without this, all resident warps of a launch
// gather at the same time (DRAM busy, SMs idle) and then compute at the same
// time (SMs busy, DRAM idle); here the DRAM queue stays busy while the SMs
// compute.  Same per-instance arithmetic and decisions as recover_warp_kernel
// (compile-time shapes, float32).
// Included by fpssft.cu inside namespace fpssft, after the warp kernel.
#pragma once

template <class R>
struct IlInst {  // one in-flight instance
    cpx<R> *spec, *slot_amp, *scr_amp;
    int *slot_key, *scr_u;
    unsigned short *hash, *cand;
    unsigned char *slot_live;
    const float2 *cube;
    const int *sched;
    long long inst;
    int it, n_slots, stall, term, it_run, seq;
    R amp_sum;
    int al[MAXD], ta[MAXD];  // line parameters of the gather in flight
    bool active;
};

// Issue the gather of iteration st.it (parameters already in st.al / st.ta).
template <int LC, class R>
__device__ __forceinline__ void il_issue(IlInst<R> &st, const Geo &g, int lane, int &seq) {
    gather_lines_async<LC>(st.spec, st.cube, g, st.al, st.ta, lane, 32);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    st.seq = seq++;
}

template <class R>
__device__ __forceinline__ bool il_load_params(IlInst<R> &st, const Geo &g, int it) {
    const int D = g.D;
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
        st.al[k] = k < D ? st.sched[(long long)it * 2 * D + k] : 0;
        st.ta[k] = k < D ? st.sched[(long long)it * 2 * D + D + k] : 0;
    }
    return line_params_ok(g, st.al, st.ta);
}

// Output of a finished instance: live entries sorted by packed key.
template <class R>
__device__ __forceinline__ void il_finish(IlInst<R> &st, const Geo &g, const Knobs &kn,
                                          const OutPtrs &out, int lane) {
    const int D = g.D;
    __syncwarp();
    int *hist = (int *)st.spec;  // the spectra are free now
    int *sslot = hist + 256;
    const int kb = g.key_bits_;
    const int shift = kb > 8 ? kb - 8 : 0;
    for (int i = lane; i < 256; i += 32) hist[i] = 0;
    __syncwarp();
    int my_live = 0;
    for (int s = lane; s < st.n_slots; s += 32)
        if (st.slot_live[s]) {
            ++my_live;
            atomicAdd(&hist[st.slot_key[s] >> shift], 1);
        }
    const int count = __shfl_sync(FULL, warp_sum(my_live), 0);
    __syncwarp();
    {
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
            hist[lane * 8 + i] = start;
            start += c[i];
        }
    }
    __syncwarp();
    for (int s = lane; s < st.n_slots; s += 32)
        if (st.slot_live[s]) sslot[atomicAdd(&hist[st.slot_key[s] >> shift], 1)] = s;
    __syncwarp();
    for (int bkt = lane; bkt < 256; bkt += 32) {
        const int en = hist[bkt], s0 = bkt ? hist[bkt - 1] : 0;
        for (int i = s0 + 1; i < en; ++i) {
            const int v = sslot[i], kv = st.slot_key[v];
            int j = i - 1;
            while (j >= s0 && st.slot_key[sslot[j]] > kv) {
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
        unpack_key(st.slot_key[s], g, m);
        int *fo = out.freqs + (st.inst * kn.k_cap + r) * D;
#pragma unroll
        for (int k = 0; k < MAXD; ++k)
            if (k < D) fo[k] = m[k];
        double *ao = out.amps + (st.inst * kn.k_cap + r) * 2;
        ao[0] = (double)st.slot_amp[s].re;
        ao[1] = (double)st.slot_amp[s].im;
    }
    if (lane == 0) {
        out.count[st.inst] = count;
        out.iterations[st.inst] = st.it_run;
        out.samples_used[st.inst] = (long long)st.it_run * g.nlines * g.L;
        out.terminated_by[st.inst] = st.term;
    }
    __syncwarp();
    st.active = false;
}

// One iteration of an instance whose gather has landed; issues the next
// gather or finishes the instance.
template <class R, int LC, int DC>
__device__ __forceinline__ void il_step(IlInst<R> &st, const Geo &g, const Knobs &kn,
                                        const cpx<R> *roots, const OutPtrs &out, int lane,
                                        int H, int &seq) {
    constexpr bool PAD = true;
    const int L = LC, nl = DC + 1;
    const R mag_tol = (R)kn.mag_tol, round_tol = (R)kn.round_tol, verify_tol = (R)kn.verify_tol;
    const R prune = (R)kn.amp_prune_tol;
    const unsigned lt_mask = (1u << lane) - 1u;
    cpx<R> *spec = st.spec;
    const int it = st.it;
    int al[MAXD], ta[MAXD];
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
        al[k] = st.al[k];
        ta[k] = st.ta[k];
    }
    st.it_run = it + 1;

    // (2) DFT of the D+1 lines (float32 rounding floor from the first stage)
    const R e = fft_static<R, LC, DC + 1>(spec, roots, lane);
    R noise_floor = (R)0;
    if (kn.noise_coef > 0) noise_floor = (R)kn.noise_coef * sqrt(__shfl_sync(FULL, warp_sum(e), 0));

    // (3) construction-subtraction
    for (int c0 = 0; c0 < st.n_slots; c0 += 32) {
        const int s = c0 + lane;
        const bool valid = s < st.n_slots && st.slot_live[s];
        int b = -1 - lane;
        if (valid) {
            int m[MAXD];
            unpack_key(st.slot_key[s], g, m);
            b = bin_of(m, g, al);
            const int u0 = phase_of(m, g, ta);
#pragma unroll
            for (int i = 0; i < MAXD + 1; ++i)
                if (i < nl) st.scr_u[i * 32 + lane] = phase_step(u0, i, m, g);
            st.scr_amp[lane] = st.slot_amp[s];
        }
        __syncwarp();
        const unsigned grp = __match_any_sync(FULL, b);
        if (valid && lane == __ffs(grp) - 1) {
            cpx<R> P[MAXD + 1];
#pragma unroll
            for (int i = 0; i < MAXD + 1; ++i) P[i] = {(R)0, (R)0};
            for (unsigned rest = grp; rest; rest &= rest - 1) {
                const int j = __ffs(rest) - 1;
                const cpx<R> aj = st.scr_amp[j];
#pragma unroll
                for (int i = 0; i < MAXD + 1; ++i)
                    if (i < nl) P[i] = P[i] + aj * roots[st.scr_u[i * 32 + j]];
            }
#pragma unroll
            for (int i = 0; i < MAXD + 1; ++i)
                if (i < nl) spec[padi<PAD>(i * L + b)] = spec[padi<PAD>(i * L + b)] - P[i];
        }
        __syncwarp();
    }

    // (4) classify + (5) merge
    const R floor = max(max((R)kn.energy_floor_abs, (R)kn.energy_floor * st.amp_sum), noise_floor);
    int n_cand = 0, n_acc = 0;
    R resid = (R)0;
#pragma unroll 2
    for (int c0 = 0; c0 < L; c0 += 32) {
        const int b = c0 + lane;
        R top = (R)0;
        const bool ok = bin_is_candidate<R, PAD>(spec, g, b, mag_tol, floor, &top);
        if (!ok) resid = max(resid, top);
        const unsigned msk = __ballot_sync(FULL, ok);
        if (ok) st.cand[n_cand + __popc(msk & lt_mask)] = (unsigned short)b;
        n_cand += __popc(msk);
    }
    __syncwarp();
    bool overflow = false;
    for (int c0 = 0; c0 < n_cand; c0 += 32) {
        const int b = c0 + lane < n_cand ? st.cand[c0 + lane] : -1;
        int m[MAXD];
        cpx<R> a;
        int stt = 0;
        if (b >= 0)
            stt = decode_candidate<R, PAD>(spec, g, b, al, ta, roots, round_tol, verify_tol, m, &a);
        const unsigned acc = __ballot_sync(FULL, stt == 2);
        int key = 0, found = -1;
        if (stt == 2) {
            key = pack_key(m, g);
            found = hash16_find(st.hash, st.slot_key, H, key);
        }
        const unsigned fresh = __ballot_sync(FULL, stt == 2 && found < 0);
        if (st.n_slots + __popc(fresh) > kn.k_cap) {
            overflow = true;
            break;
        }
        n_acc += __popc(acc);
        if (stt == 2) {
            cpx<R> v = a;
            int s;
            if (found < 0) {
                s = st.n_slots + __popc(fresh & lt_mask);
                st.slot_key[s] = key;
                hash16_insert(st.hash, H, key, s);
            } else {
                s = found;
                v = st.slot_amp[s] + a;
            }
            const bool keep = !(cabs(v) <= prune);
            st.slot_amp[s] = keep ? v : cpx<R>{(R)0, (R)0};
            st.slot_live[s] = keep;
            const int u0 = phase_of(m, g, ta);
            for (int i = 0; i < nl; ++i)
                spec[padi<PAD>(i * L + b)] =
                    spec[padi<PAD>(i * L + b)] - a * roots[phase_step(u0, i, m, g)];
        }
        if (b >= 0) resid = max(resid, bin_residual<R, PAD>(spec, g, b));
        st.n_slots += __popc(fresh);
        __syncwarp();
    }
    if (overflow) {
        st.term = FPSSFT_TERM_K_CAP_OVERFLOW;
        if (lane == 0 && out.iter_stats) {
            int *sp = out.iter_stats + (st.inst * kn.t_max + it) * 3;
            sp[0] = n_cand;
            sp[1] = 0;
            sp[2] = n_cand;
        }
        il_finish(st, g, kn, out, lane);
        return;
    }
    __syncwarp();

    // (6) amp_sum, (7) termination
    R my = (R)0;
    for (int s = lane; s < st.n_slots; s += 32)
        if (st.slot_live[s]) my += cabs(st.slot_amp[s]);
    st.amp_sum = __shfl_sync(FULL, warp_sum(my), 0);
    st.stall = n_acc > 0 ? 0 : st.stall + 1;
    const R clean = max((R)kn.energy_floor_abs, (R)kn.residual_stop * st.amp_sum);
    const bool is_clean = warp_max(resid) <= clean * clean;
    if (lane == 0 && out.iter_stats) {
        int *sp = out.iter_stats + (st.inst * kn.t_max + it) * 3;
        sp[0] = n_cand;
        sp[1] = n_acc;
        sp[2] = n_cand - n_acc;
    }
    __syncwarp();
    if (is_clean) st.term = FPSSFT_TERM_RESIDUAL_CLEAN;
    else if (st.stall >= kn.stall_limit) st.term = FPSSFT_TERM_STALL;
    else if (it + 1 < kn.t_max) {
        st.it = it + 1;
        if (il_load_params(st, g, st.it)) {
            il_issue<LC>(st, g, lane, seq);
            return;
        }
        st.term = -1;
    }
    il_finish(st, g, kn, out, lane);
}

template <class R, int LC, int DC, int NI>
__global__ void __launch_bounds__(128, 2) recover_warp_il_kernel(
    const float2 *__restrict__ cubes, long long batch, long long batch_stride, Geo g_in, Knobs kn,
    const int *__restrict__ schedule, const int *__restrict__ sched_index, int n_sched,
    OutPtrs out) {
    static_assert(sizeof(R) == 4, "the interleaved kernel pipelines cp.async gathers (float32)");
    extern __shared__ __align__(16) unsigned char sm[];
    Geo g = g_in;
    g.L = LC;
    g.D = DC;
    g.nlines = DC + 1;
    const WarpLayout lay = make_warp_layout(DC, LC, kn.k_cap, (int)sizeof(cpx<R>));
    cpx<R> *roots = (cpx<R> *)sm;
    build_roots(roots, LC);
    __syncthreads();  // the only block-wide barrier

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long first = ((long long)blockIdx.x * (blockDim.x >> 5) + warp) * NI;
    const int H = lay.H;
    int seq = 0;
    IlInst<R> st[NI];
#pragma unroll
    for (int s = 0; s < NI; ++s) {
        unsigned char *base = sm + lay.roots + ((size_t)warp * NI + s) * lay.per_warp;
        IlInst<R> &q = st[s];
        q.spec = (cpx<R> *)(base + lay.spec);
        q.slot_amp = (cpx<R> *)(base + lay.slot_amp);
        q.slot_key = (int *)(base + lay.slot_key);
        q.hash = (unsigned short *)(base + lay.hash);
        q.slot_live = base + lay.slot_live;
        q.cand = (unsigned short *)(base + lay.cand);
        q.scr_u = (int *)(base + lay.scr_u);
        q.scr_amp = (cpx<R> *)(base + lay.scr_amp);
        q.inst = first + s;
        q.active = q.inst < batch;
        q.seq = -1;
        if (!q.active) continue;
        q.cube = cube_base(cubes, (long long)q.inst, batch_stride, kn.group);
        int sidx = sched_index ? sched_index[q.inst] : 0;
        const bool ok = sidx >= 0 && sidx < n_sched;
        q.sched = schedule + (long long)(ok ? sidx : 0) * kn.t_max * 2 * DC;
        q.it = 0;
        q.it_run = 0;
        q.n_slots = 0;
        q.stall = 0;
        q.amp_sum = (R)0;
        q.term = ok ? FPSSFT_TERM_MAX_ITERATIONS : -1;
        for (int h = lane; h < H; h += 32) q.hash[h] = HASH_EMPTY;
        __syncwarp();
        if (ok && il_load_params(q, g, 0)) {
            il_issue<LC>(q, g, lane, seq);
        } else {
            q.term = -1;
            il_finish(q, g, kn, out, lane);
        }
    }
    // round-robin over the in-flight instances; wait only for the oldest
    // gather needed now, leave the younger ones in flight
    while (true) {
        bool any = false;
#pragma unroll
        for (int s = 0; s < NI; ++s) {
            if (!st[s].active) continue;
            any = true;
            int younger = 0;
#pragma unroll
            for (int t = 0; t < NI; ++t)
                if (t != s && st[t].active && st[t].seq > st[s].seq) ++younger;
            if (younger >= 2) asm volatile("cp.async.wait_group 2;\n" ::: "memory");
            else if (younger == 1) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
            else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
            __syncwarp();
            il_step<R, LC, DC>(st[s], g, kn, roots, out, lane, H, seq);
        }
        if (!any) break;
    }
}
