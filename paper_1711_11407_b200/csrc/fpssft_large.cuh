// Kernels for recovered sets and lines too large for shared memory (the
// imaging duality path: a 512 x 576 frequency cube,
// L = 4608, up to ~20k recovered pixels, float64).  The loop around them runs
// on the host (paper_1711_11407_b200/large.py), one step per launch; each
// kernel keeps the per-bin semantics of its shared-memory counterpart.
// Included by fpssft.cu after the per-step op kernels.
#pragma once
// (included inside namespace fpssft)

// Line samples of the D+1 offsets of one iteration, straight to global
// memory: out[b][i][l] = cube_b[(alpha l + tau + [i > 0] e_{i-1}) mod N]
// (lines.py:36-64, core.py:236-238).  T = float2 (complex64 cube) or double2
// (complex128 cube); one thread per sample.
template <class T, class R>
__global__ void __launch_bounds__(256) gather_lines_kernel(const T *__restrict__ cubes,
                                                           long long batch_stride, Geo g,
                                                           const int *__restrict__ alpha_tau,
                                                           int per_instance, cpx<R> *out) {
    const int inst = blockIdx.y, D = g.D, L = g.L, nl = g.nlines;
    const int *at = alpha_tau + (per_instance ? (long long)inst * 2 * D : 0);
    int al[MAXD], ta[MAXD];
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
        al[k] = k < D ? at[k] : 0;
        ta[k] = k < D ? at[D + k] : 0;
    }
    if (!line_params_ok(g, al, ta)) return;
    const T *cube = cubes + (long long)inst * batch_stride;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nl * L; e += gridDim.x * blockDim.x) {
        const int i = e / L, l = e - i * L;
        long long off = 0;
#pragma unroll
        for (int k = 0; k < MAXD; ++k) {
            if (k < D) {
                long long n = ((long long)al[k] * l + ta[k] + (i == k + 1)) % g.N[k];
                off += n * g.stride[k];
            }
        }
        const T v = cube[off];
        out[(long long)inst * nl * L + e] = {(R)v.x, (R)v.y};
    }
}

// Projection of a large sparse set onto the bins of one line.  CTA c owns
// bins [c BT, (c+1) BT), one per thread.  It streams the entries in chunks
// of BT, keeps those that land in its bins (block-scan compaction, so the
// kept list stays in entry order) in shared memory, and each thread then
// sums its bin's entries in that order -- exactly project_bins' per-bin
// order, with no sort, no global scratch and no atomics.  A full list is
// drained before it overflows (still in order).  Work per CTA: K bin
// computations + ~K BT / L list compares per thread.
template <class R, int BT, int CAP>
__global__ void __launch_bounds__(BT) project_global_kernel(const int *__restrict__ freqs,
                                                            const double *__restrict__ amps,
                                                            const int *__restrict__ counts,
                                                            int k_max, Geo g,
                                                            const int *__restrict__ alpha_tau,
                                                            int per_instance, double *out) {
    __shared__ unsigned short lbin[CAP];
    __shared__ int lu[CAP];
    __shared__ cpx<R> lamp[CAP];
    __shared__ int red[32];
    const int inst = blockIdx.y, D = g.D, L = g.L, tid = threadIdx.x;
    const int b0 = blockIdx.x * BT;
    const int *at = alpha_tau + (per_instance ? (long long)inst * 2 * D : 0);
    int al[MAXD], ta[MAXD];
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
        al[k] = k < D ? at[k] : 0;
        ta[k] = k < D ? at[D + k] : 0;
    }
    const int n = min(counts[inst], k_max);
    cpx<R> acc = {(R)0, (R)0};
    int fill = 0;
    auto drain = [&](int cnt) {
        for (int j = 0; j < cnt; ++j) {
            if (lbin[j] == tid) {
                double sn, c;  // the value build_roots puts in the table
                sincospi(2.0 * (double)lu[j] / (double)L, &sn, &c);
                acc = acc + lamp[j] * cpx<R>{(R)c, (R)sn};
            }
        }
    };
    for (int c0 = 0; c0 < n; c0 += BT) {
        const int e = c0 + tid;
        bool mine = false;
        int bin = 0, u = 0;
        cpx<R> a = {(R)0, (R)0};
        if (e < n) {
            const long long o = (long long)inst * k_max + e;
            int m[MAXD];
#pragma unroll
            for (int k = 0; k < MAXD; ++k) m[k] = k < D ? freqs[o * D + k] : 0;
            bin = bin_of(m, g, al) - b0;
            mine = bin >= 0 && bin < BT;
            if (mine) {
                u = phase_of(m, g, ta);
                a = {(R)amps[o * 2], (R)amps[o * 2 + 1]};
            }
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
            lbin[fill + pos] = (unsigned short)bin;
            lu[fill + pos] = u;
            lamp[fill + pos] = a;
        }
        fill += tot;
    }
    __syncthreads();
    drain(fill);
    const int b = b0 + tid;
    if (b < L) {
        out[((long long)inst * L + b) * 2] = (double)acc.re;
        out[((long long)inst * L + b) * 2 + 1] = (double)acc.im;
    }
}
