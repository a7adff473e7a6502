// Device-resident recovery loop for one large problem (the imaging duality
// path: 512 x 576 cubes, L = 4608, ~20k recovered
// pixels, float64), the loop of driver.py:140-204 as ONE CUDA graph: a
// conditional WHILE node whose body is one iteration --
//   setup   (alpha, tau) of iteration `it` from the device schedule, the D+1
//           stepped offsets (lines.py:55-64), the energy floor (driver.py:156)
//   gather  the D+1 lines                        (lines.py:36-64)
//   DFT     1/L forward transform of each line   (transform.py:17-22)
//   peel    projection of the recovered set onto each line, subtracted
//           (decoder.py:172-191, driver.py:150-154)
//   decode  classifier + bin guard on every bin  (decoder.py:127-169,
//           driver.py:156-176), floor read on the device
//   merge   merge-by-sum / prune into the device slot table in ascending bin
//           order with the reference dict's semantics (driver.py:94-118),
//           peel of the accepted entries, amp_sum, max |S|, the iteration
//           log and termination (driver.py:189-204); it sets the WHILE
//           condition (cudaGraphSetConditional), so the host never syncs
//           inside the loop.
// Included by fpssft.cu (inside namespace fpssft) after the per-step kernels.
#pragma once

struct LargeState {
    int it;        // iterations completed
    int done;      // 1 once terminated
    int stall;     // consecutive iterations without an accepted entry
    int term;      // FPSSFT_TERM_*
    int n_slots;   // slots used (incl. zeroed ones: the projection sums them as +0)
    int overflow;  // a fresh entry found no slot (k_cap)
    int pad[2];
    double amp_total;  // sum |a| over the live entries (driver.py:108)
    double floor;      // this iteration's energy floor (driver.py:156)
};

// it-th (alpha, tau) and the D+1 stepped offsets -> at_all[(D+1)][2][D];
// the energy floor from the previous iteration's amp_total.
__global__ void large_setup_kernel(const int *__restrict__ schedule, Geo g, Knobs kn,
                                   LargeState *stt, int *at_all) {
    if (threadIdx.x != 0 || stt->done) return;
    const int D = g.D, it = stt->it;
    const int *s = schedule + (long long)it * 2 * D;
    for (int i = 0; i <= D; ++i)
        for (int k = 0; k < D; ++k) {
            at_all[(i * 2) * D + k] = s[k];
            int t = s[D + k];
            if (i == k + 1) t = t + 1 == g.N[k] ? 0 : t + 1;
            at_all[(i * 2 + 1) * D + k] = t;
        }
    stt->floor = fmax(kn.energy_floor_abs, kn.energy_floor * stt->amp_total);
}

// root e^{2 pi i u / L} as the projection computes it (sincospi in float64)
__device__ __forceinline__ cpx<double> root_exact(int u, int L) {
    double sn, c;
    sincospi(2.0 * (double)u / (double)L, &sn, &c);
    return {c, sn};
}

// Projection of the recovered set onto all D+1 lines in one pass (the bin
// of an entry is the same on every line; only the phase steps by
// c_k m_k, lines.py:55-64): CTA c owns bins [c BT, (c+1) BT), streams the
// slots in chunks of BT, keeps those landing in its bins in an in-order list
// (block-scan compaction) and each thread sums its bin's entries per line in
// slot order -- project_onto_bins' order, no sort, no atomics.
template <int BT, int CAP>
__global__ void __launch_bounds__(BT) large_project_kernel(const int *__restrict__ sfreqs,
                                                           const double *__restrict__ samps,
                                                           const LargeState *stt, Geo g,
                                                           const int *__restrict__ at_all,
                                                           double *proj) {
    __shared__ unsigned short lbin[CAP];
    __shared__ int lu[CAP][MAXD + 1];
    __shared__ cpx<double> lamp[CAP];
    __shared__ int red[32];
    if (stt->done) return;
    const int D = g.D, L = g.L, tid = threadIdx.x, b0 = blockIdx.x * BT;
    int al[MAXD], ta[MAXD];
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
        al[k] = k < D ? at_all[k] : 0;
        ta[k] = k < D ? at_all[D + k] : 0;
    }
    const int n = stt->n_slots;
    cpx<double> acc[MAXD + 1];
#pragma unroll
    for (int i = 0; i < MAXD + 1; ++i) acc[i] = {0.0, 0.0};
    int fill = 0;
    auto drain = [&](int cnt) {
        for (int j = 0; j < cnt; ++j) {
            if (lbin[j] == tid) {
#pragma unroll
                for (int i = 0; i < MAXD + 1; ++i)
                    if (i <= D) acc[i] = acc[i] + lamp[j] * root_exact(lu[j][i], L);
            }
        }
    };
    for (int c0 = 0; c0 < n; c0 += BT) {
        const int e = c0 + tid;
        bool mine = false;
        int bin = 0, m[MAXD] = {0, 0, 0, 0};
        if (e < n) {
#pragma unroll
            for (int k = 0; k < MAXD; ++k) m[k] = k < D ? sfreqs[e * D + k] : 0;
            bin = bin_of(m, g, al) - b0;
            mine = bin >= 0 && bin < BT;
        }
        int tot;
        const int pos = block_exscan(mine ? 1 : 0, red, &tot);
        if (fill + tot > CAP) {  // uniform: drain the list, in order
            __syncthreads();
            drain(fill);
            __syncthreads();
            fill = 0;
        }
        if (mine) {
            const int p = fill + pos;
            lbin[p] = (unsigned short)bin;
            const int u0 = phase_of(m, g, ta);
#pragma unroll
            for (int i = 0; i < MAXD + 1; ++i)
                if (i <= D) lu[p][i] = phase_step(u0, i, m, g);
            lamp[p] = {samps[2 * e], samps[2 * e + 1]};
        }
        fill += tot;
    }
    __syncthreads();
    drain(fill);
    const int b = b0 + tid;
    if (b < L)
#pragma unroll
        for (int i = 0; i < MAXD + 1; ++i)
            if (i <= D) {
                proj[((long long)i * L + b) * 2] = acc[i].re;
                proj[((long long)i * L + b) * 2 + 1] = acc[i].im;
            }
}

// spec -= proj over the D+1 lines (the recovered set's projection).
__global__ void large_subtract_kernel(cpx<double> *spec, const double *__restrict__ proj, int n,
                                      const LargeState *stt) {
    if (stt->done) return;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
        spec[e].re -= proj[2 * e];
        spec[e].im -= proj[2 * e + 1];
    }
}

// One CTA: merge (ascending bins), peel, amp_sum, max |S|, log, termination.
constexpr int LARGE_NT = 1024;
__global__ void __launch_bounds__(LARGE_NT, 1)
    large_merge_kernel(cpx<double> *spec, const int *__restrict__ status,
                       const int *__restrict__ dfreqs, const double *__restrict__ damps,
                       const int *__restrict__ ncand, const int *__restrict__ at_all, Geo g,
                       Knobs kn, LargeState *stt, int *slot_of, int *sfreqs, double *samps,
                       int *iter_stats, cudaGraphConditionalHandle cond) {
    __shared__ int ired[64];
    __shared__ double dred[64];
    const int tid = threadIdx.x, D = g.D, L = g.L;
    if (stt->done) {  // (a WHILE node never runs a body after a 0 condition)
        if (tid == 0) cudaGraphSetConditional(cond, 0);
        return;
    }
    int ta[MAXD];
#pragma unroll
    for (int k = 0; k < MAXD; ++k) ta[k] = k < D ? at_all[D + k] : 0;
    const int n0 = stt->n_slots;
    int carry = 0, n_acc = 0;
    bool ovf = false;
    for (int c0 = 0; c0 < L; c0 += LARGE_NT) {
        const int b = c0 + tid;
        const bool acc = b < L && status[b] == 2;
        int m[MAXD] = {0, 0, 0, 0};
        cpx<double> a = {0.0, 0.0};
        int lin = 0;
        bool fresh = false;
        if (acc) {
            long long li = 0;
#pragma unroll
            for (int k = 0; k < MAXD; ++k)
                if (k < D) {
                    m[k] = dfreqs[b * D + k];
                    li = li * g.N[k] + m[k];
                }
            lin = (int)li;
            a = {damps[2 * b], damps[2 * b + 1]};
            const int old = slot_of[lin];  // keys are distinct within an iteration
            if (old >= 0) {
                const cpx<double> v = {samps[2 * old] + a.re, samps[2 * old + 1] + a.im};
                if (cabs(v) <= kn.amp_prune_tol) {  // del entries[f]
                    samps[2 * old] = samps[2 * old + 1] = 0.0;
                    slot_of[lin] = -1;
                } else {
                    samps[2 * old] = v.re;
                    samps[2 * old + 1] = v.im;
                }
            } else {
                fresh = !(cabs(a) <= kn.amp_prune_tol);
            }
            // peel the accepted entry from its bin on every line (driver.py:189-194)
            const int u0 = phase_of(m, g, ta);
#pragma unroll
            for (int i = 0; i < MAXD + 1; ++i)
                if (i <= D) {
                    const cpx<double> r = root_exact(phase_step(u0, i, m, g), L);
                    spec[(long long)i * L + b] = spec[(long long)i * L + b] - a * r;
                }
        }
        int tot;
        const int pre = block_exscan((fresh ? 1 : 0) | ((acc ? 1 : 0) << 16), ired, &tot);
        if (fresh) {  // appended in ascending bin order (dict insertion order)
            const int s = n0 + carry + (pre & 0xFFFF);
            if (s < kn.k_cap) {
#pragma unroll
                for (int k = 0; k < MAXD; ++k)
                    if (k < D) sfreqs[s * D + k] = m[k];
                samps[2 * s] = a.re;
                samps[2 * s + 1] = a.im;
                slot_of[lin] = s;
            } else {
                ovf = true;
            }
        }
        carry += tot & 0xFFFF;
        n_acc += tot >> 16;
    }
    const int n_slots = min(n0 + carry, kn.k_cap);
    ovf = __syncthreads_or(ovf);
    // amp_sum over the live entries (slot_of points back at a live slot)
    double my = 0.0;
    for (int s = tid; s < n_slots; s += LARGE_NT) {
        long long li = 0;
#pragma unroll
        for (int k = 0; k < MAXD; ++k)
            if (k < D) li = li * g.N[k] + sfreqs[s * D + k];
        if (slot_of[li] == s) my += cabs(cpx<double>{samps[2 * s], samps[2 * s + 1]});
    }
    const double amp_total = block_sum(my, dred);
    // residual max |S| over the D+1 lines
    double mx = 0.0;
    for (int e = tid; e < (D + 1) * L; e += LARGE_NT) mx = fmax(mx, cabs(spec[e]));
    const double worst = block_max(mx, dred + 32);
    if (tid == 0) {
        const int it = stt->it;
        const int nc = *ncand;
        if (iter_stats) {
            iter_stats[it * 3] = nc;
            iter_stats[it * 3 + 1] = ovf ? 0 : n_acc;
            iter_stats[it * 3 + 2] = ovf ? nc : nc - n_acc;
        }
        stt->n_slots = n_slots;
        stt->amp_total = amp_total;
        stt->stall = n_acc > 0 ? 0 : stt->stall + 1;
        int term = -1;
        if (ovf) {
            stt->overflow = 1;
            term = FPSSFT_TERM_K_CAP_OVERFLOW;
        } else if (worst <= fmax(kn.energy_floor_abs, kn.residual_stop * amp_total)) {
            term = FPSSFT_TERM_RESIDUAL_CLEAN;
        } else if (stt->stall >= kn.stall_limit) {
            term = FPSSFT_TERM_STALL;
        }
        stt->it = it + 1;
        if (term >= 0) {
            stt->term = term;
            stt->done = 1;
        } else if (it + 1 >= kn.t_max) {
            stt->term = FPSSFT_TERM_MAX_ITERATIONS;
            stt->done = 1;
        }
        cudaGraphSetConditional(cond, stt->done ? 0 : 1);
    }
}

__global__ void large_init_kernel(LargeState *stt, int *slot_of, long long n_total, int t_max) {
    const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (long long i = i0; i < n_total; i += (long long)gridDim.x * blockDim.x) slot_of[i] = -1;
    if (i0 == 0) {
        *stt = LargeState{};
        stt->term = FPSSFT_TERM_MAX_ITERATIONS;
        stt->done = t_max <= 0;
    }
}

// The live entries in slot (insertion) order -> freqs / amps, and the report
// scalars.
__global__ void large_final_kernel(const LargeState *stt, const int *slot_of,
                                   const int *sfreqs, const double *samps, Geo g, int *freqs,
                                   double *amps, int *count, int *iterations,
                                   long long *samples_used, int *terminated_by) {
    __shared__ int ired[64];
    const int tid = threadIdx.x, D = g.D, n = stt->n_slots;
    int carry = 0;
    for (int c0 = 0; c0 < n; c0 += LARGE_NT) {
        const int s = c0 + tid;
        bool live = false;
        if (s < n) {
            long long li = 0;
#pragma unroll
            for (int k = 0; k < MAXD; ++k)
                if (k < D) li = li * g.N[k] + sfreqs[s * D + k];
            live = slot_of[li] == s;
        }
        int tot;
        const int pre = block_exscan(live ? 1 : 0, ired, &tot);
        if (live) {
            const int r = carry + pre;
#pragma unroll
            for (int k = 0; k < MAXD; ++k)
                if (k < D) freqs[r * D + k] = sfreqs[s * D + k];
            amps[2 * r] = samps[2 * s];
            amps[2 * r + 1] = samps[2 * s + 1];
        }
        carry += tot;
    }
    if (tid == 0) {
        *count = carry;
        *iterations = stt->it;
        *samples_used = (long long)stt->it * g.nlines * g.L;
        *terminated_by = stt->term;
    }
}

// Workspace carve-up (bytes, 256-aligned pieces).
struct LargeWs {
    size_t state, at_all, spec, proj, status, dfreqs, damps, ncand, slot_of, sfreqs, samps, total;
};
inline LargeWs large_ws(const Geo &g, int k_cap) {
    auto a = [](size_t x) { return (x + 255) & ~(size_t)255; };
    LargeWs w;
    long long n_total = 1;
    for (int k = 0; k < g.D; ++k) n_total *= g.N[k];
    const size_t nl = (size_t)g.nlines * g.L;
    size_t o = 0;
    w.state = o;   o += a(sizeof(LargeState));
    w.at_all = o;  o += a((size_t)g.nlines * 2 * g.D * 4);
    w.spec = o;    o += a(nl * 16);
    w.proj = o;    o += a(nl * 16);
    w.status = o;  o += a((size_t)g.L * 4);
    w.dfreqs = o;  o += a((size_t)g.L * g.D * 4);
    w.damps = o;   o += a((size_t)g.L * 16);
    w.ncand = o;   o += a(4);
    w.slot_of = o; o += a((size_t)n_total * 4);
    w.sfreqs = o;  o += a((size_t)k_cap * g.D * 4);
    w.samps = o;   o += a((size_t)k_cap * 16);
    w.total = o;
    return w;
}
