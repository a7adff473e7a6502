// Line staging for interleaved batches held in pinned HOST memory.
//
// The schedule (alpha_t, tau_t) is data-independent (driver.py:131,142-143),
// so the line samples of the first T0 iterations of every instance are known
// before the loop starts (extract_line, lines.py:36-64 + core.py:236-238).
// An SM load of host memory moves at most one 128-byte request per PCIe tag
// (~0.29 G requests/s on this pool whatever their size, tools/seg_probe.cu:
// 37 GB/s at 128 B), a TMA bulk copy of a 256-byte segment the same request
// rate at twice the bytes (51 GB/s, the link's bulk rate).  So for a batch
// interleaved by G (segment = 8 G bytes, G = 32: 256 B) this kernel copies
// the segments of iterations 0..T0-1 with one cp.async.bulk each into shared
// memory and writes them, in line order, to a staging buffer in HBM:
//     staged[group][t][line][l][G]   complex64
// The group-gather recovery kernel then reads iteration t < T0 from there
// (GroupGather::load_staged: contiguous, no index arithmetic) and only the
// straggler iterations t >= T0 from the host cube.
//
// One CTA = 256 consecutive (line, l) positions of one (group, t): 256 bulk
// copies in flight, one mbarrier, one bulk store of the 256 segments.
// (included inside namespace fpssft)
namespace stage {

constexpr int POS = 256;  // positions (= bulk copies) per CTA

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(POS) stage_lines_kernel(const float2 *__restrict__ cubes,
                                                          long long group_stride, Geo g, int G,
                                                          const int *__restrict__ schedule,
                                                          int t_stage, float2 *staged,
                                                          long long staged_group_stride) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) unsigned long long mbar;
    const int tid = threadIdx.x, D = g.D, NLL = g.nlines * g.L;
    const int chunk = blockIdx.x, t = blockIdx.y;
    const long long grp = blockIdx.z;
    const int q = chunk * POS + tid;  // position: line q / L, point q % L
    const int nq = min(POS, NLL - chunk * POS);
    const unsigned S = 8u * (unsigned)G;  // segment bytes
    const unsigned mb = smem_u32(&mbar);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(mb));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(mb),
                     "r"((unsigned)nq * S) : "memory");
    }
    __syncthreads();
    if (tid < nq) {
        const int *sc = schedule + (long long)t * 2 * D;
        const int line = q / g.L, l = q - line * g.L;
        long long off = 0;
#pragma unroll
        for (int k = 0; k < MAXD; ++k) {
            if (k < D) {
                int nk = (int)fastmod((unsigned)sc[k] * (unsigned)l + (unsigned)sc[D + k],
                                      g.magic[k], (unsigned)g.N[k]);
                if (k == line - 1) nk = nk + 1 == g.N[k] ? 0 : nk + 1;  // tau + e_k
                off += (long long)nk * g.stride[k];
            }
        }
        const float2 *src = cubes + grp * group_stride + off;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(smem_u32(sm + (size_t)tid * S)), "l"(src), "r"(S), "r"(mb) : "memory");
    }
    if (tid == 0) {
        unsigned done = 0;
        while (!done)
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared.b64 p, [%1], 0;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(mb) : "memory");
        float2 *dst = staged + grp * staged_group_stride +
                      ((long long)t * NLL + (long long)chunk * POS) * G;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                     "r"(smem_u32(sm)), "r"((unsigned)nq * S) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

}  // namespace stage
