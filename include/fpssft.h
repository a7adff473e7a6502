/*
 * fpssft.h -- C ABI of the B200-native FPS-SFT recovery loop.
 *
 * Plain pointers and sizes only; every device buffer is owned by the caller.
 * All entry points are stream-ordered and asynchronous, reentrant across
 * streams, threads and devices, and keep no global mutable state (the root
 * tables are built per CTA on chip).  Return value 0 = success; otherwise a
 * FPSSFT_E* code and fpssft_last_error() (thread-local) says why.
 *
 * The reference (fps-sft 0.1.0, pure Python) exposes this path as Python
 * functions; each entry point below names the reference interface it replaces
 * (paths under /root/reference/pkg/src/fps_sft/).  The Python mirror of that
 * interface, paper_1711_11407_b200, binds these symbols with ctypes.
 */
#ifndef FPSSFT_H_
#define FPSSFT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FPSSFT_MAX_DIMS 4

/* error codes (the Python mirror maps them to the reference's exceptions) */
#define FPSSFT_OK 0
#define FPSSFT_EINVAL 1       /* ValueError   (core.py:225-226, lines.py:30-31, driver.py:55-63) */
#define FPSSFT_EOVERFLOW 2    /* OverflowError (core.py:53-54, :197-198)                         */
#define FPSSFT_EUNSUPPORTED 3 /* shape/capacity beyond what one CTA holds on chip                */
#define FPSSFT_ECUDA 4        /* CUDA runtime error                                              */

/* arithmetic the path computes in (input cubes are always complex64) */
#define FPSSFT_F32 0
#define FPSSFT_F64 1
/* float32 arithmetic with the float64 reference's decisions: float64
 * amplitudes and line-0 transform, and every decision whose float32 statistic
 * lies within its error bound of the threshold re-evaluated in float64
 * (decoder.py:146-163, driver.py:103-108).  Shapes without a guarded kernel
 * run the float64 kernels. */
#define FPSSFT_F32_GUARDED 2

/* execution mode: one warp or one whole CTA per instance (AUTO picks) */
#define FPSSFT_MODE_AUTO 0
#define FPSSFT_MODE_CTA 1
#define FPSSFT_MODE_WARP 2

/* terminated_by codes (driver.py:24-26 plus capacity overflow) */
#define FPSSFT_TERM_RESIDUAL_CLEAN 0
#define FPSSFT_TERM_STALL 1
#define FPSSFT_TERM_MAX_ITERATIONS 2
#define FPSSFT_TERM_K_CAP_OVERFLOW 3

/* CubeShape (core.py:26-73) plus the element strides of one cube. */
typedef struct fpssft_shape {
    int32_t ndim;                      /* D, 1..FPSSFT_MAX_DIMS                     */
    int32_t dims[FPSSFT_MAX_DIMS];     /* N_k                                       */
    int64_t strides[FPSSFT_MAX_DIMS];  /* element strides (row-major: N_1*..., 1)  */
} fpssft_shape;

/* FpsSftConfig (driver.py:29-63) minus seed (the schedule is explicit),
 * plus the recovered-set capacity and the arithmetic precision. */
typedef struct fpssft_params {
    int32_t t_max;       /* iteration cap (driver.py:132, default :88-91)  */
    int32_t stall_limit; /* driver.py:44                                    */
    int32_t k_cap;       /* recovered-set capacity per instance (power of 2)*/
    int32_t precision;   /* FPSSFT_F32 | FPSSFT_F64 | FPSSFT_F32_GUARDED    */
    int32_t mode;        /* FPSSFT_MODE_*: which kernel owns an instance    */
    double mag_tol, verify_tol, round_tol, amp_prune_tol;
    double energy_floor, energy_floor_abs, residual_stop;
} fpssft_params;

/* RecoveryReport (driver.py:76-85), padded per instance. */
typedef struct fpssft_out {
    int32_t *freqs;        /* [B, k_cap, D]  lexicographic order (core.py:102) */
    double *amps;          /* [B, k_cap, 2]  complex128                         */
    int32_t *count;        /* [B]            len(recovered)                     */
    int32_t *iterations;   /* [B]            iterations_run                     */
    int64_t *samples_used; /* [B]            iterations*(D+1)*L                 */
    int32_t *terminated_by;/* [B]            FPSSFT_TERM_*                       */
    int32_t *iter_stats;   /* [B, t_max, 3]  (candidates, accepted, rejected) or NULL (driver.py:66-73) */
} fpssft_out;

/*
 * The whole recovery loop for a batch of independent complex64 cubes.
 * Replaces fps_sft(make_dense_source(cube, shape), config)
 * (driver.py:121-212, core.py:276-278) for every instance b:
 *   cube_b    = cubes + b*batch_stride                       (device, complex64;
 *               or pinned, mapped host memory: UVA zero copy -- the kernels gather
 *               only the sampled chunks over the host link)
 *   schedule  = int32 [n_sched, t_max, 2, D] (alpha, tau)     (device)
 *               the (alpha_t, tau_t) the reference draws from default_rng(seed)
 *               (driver.py:131,142-143); see paper_1711_11407_b200.schedule
 *   sched_index[b] in [0, n_sched) picks instance b's schedule (NULL = 0).
 */
int fpssft_run_batch(const void *cubes, int64_t batch, int64_t batch_stride,
                     const fpssft_shape *shape, const fpssft_params *params,
                     const int32_t *schedule, const int32_t *sched_index, int32_t n_sched,
                     const fpssft_out *out, void *stream);

/* The same loop over a batch stored with `group` instances interleaved sample
 * by sample: layout [ceil(B/group), *dims, group] complex64 (the 64-byte DRAM
 * segment of a sample then serves 8 instances at group = 8).  Instance b's
 * sample n sits at cubes + (b / group) * group_stride + (b % group) +
 * sum_k n_k * shape->strides[k] (elements; the strides include the factor
 * group).  group = 1 is fpssft_run_batch.  Same outputs, same errors. */
int fpssft_run_batch_grouped(const void *cubes, int64_t batch, int32_t group,
                             int64_t group_stride, const fpssft_shape *shape,
                             const fpssft_params *params, const int32_t *schedule,
                             const int32_t *sched_index, int32_t n_sched, const fpssft_out *out,
                             void *stream);

/*
 * The same loop over an interleaved batch (fpssft_run_batch_grouped, one
 * schedule for the batch) held in pinned, mapped HOST memory, with the line
 * samples of the first `stage_iterations` iterations staged through HBM: the
 * schedule is data-independent (driver.py:131,142-143), so those samples
 * (extract_line, lines.py:36-64 + core.py:236-238) are known before the loop
 * starts.  A staging kernel copies each needed 8*group-byte segment with one
 * TMA bulk copy (group = 32: 256-byte segments, the host link's bulk rate
 * instead of the request-rate bound of SM loads) into
 * staging[group][t][line][l][group]; the recovery kernel reads iterations
 * t < stage_iterations from there and later (straggler) iterations from the
 * host cube.  Outputs identical to fpssft_run_batch_grouped.  Served by the
 * warp-per-instance kernels (float32; guarded float32 on the 64^3 shape; the
 * group-gather kernel for 256 x 256 batches with group a multiple of 8) and
 * the float32 compile-time team kernels (L = 2048, 512); other shapes and
 * float64 return FPSSFT_EUNSUPPORTED.  cubes may also be device memory.
 *   staging: device buffer of fpssft_stage_bytes(shape, group, batch,
 *            min(stage_iterations, params->t_max)) bytes.
 */
int64_t fpssft_stage_bytes(const fpssft_shape *shape, int32_t group, int64_t batch,
                           int32_t stage_iterations);
int fpssft_run_batch_staged(const void *cubes, int64_t batch, int32_t group,
                            int64_t group_stride, const fpssft_shape *shape,
                            const fpssft_params *params, const int32_t *schedule,
                            const fpssft_out *out, void *staging, int64_t staging_bytes,
                            int32_t stage_iterations, int32_t already_staged, void *stream);
/* The staging pass alone (already_staged != 0 above then skips it): lets a
 * caller stage the next chunk of a batch on one stream while the previous
 * chunk recovers on another (hostpath.py). */
int fpssft_stage_lines(const void *cubes, int64_t batch, int32_t group, int64_t group_stride,
                       const fpssft_shape *shape, const fpssft_params *params,
                       const int32_t *schedule, void *staging, int64_t staging_bytes,
                       int32_t stage_iterations, void *stream);

/*
 * D+1 line spectra of one iteration per instance.  Replaces
 *   [dft_forward(extract_line(DenseSource(cube), LineParams(alpha, off, L)))
 *    for off in decoding_offsets(tau)]
 * (lines.py:36-64, core.py:236-238, transform.py:17-22).
 * alpha_tau: device int32 [B or 1, 2, D]; per_instance selects which.
 * spectra: [B, D+1, L] complex64 (F32) or complex128 (F64).
 */
int fpssft_line_spectra(const void *cubes, int64_t batch, int64_t batch_stride,
                        const fpssft_shape *shape, const int32_t *alpha_tau,
                        int32_t per_instance, void *spectra, int32_t precision, void *stream);

/*
 * Line samples only, into global memory (extract_line for the D+1 offsets,
 * lines.py:36-64 + core.py:236-238) -- the first half of
 * fpssft_line_spectra for lines too long to transform in one CTA's shared
 * memory (the imaging shape 512 x 576, L = 4608, in float64), followed by
 * fpssft_dft_forward.  cubes: complex64 (cube_precision FPSSFT_F32) or
 * complex128 (FPSSFT_F64) row-major with shape->strides; lines: [B, D+1, L]
 * complex of `precision`.  B <= 65535.
 */
int fpssft_gather_lines(const void *cubes, int32_t cube_precision, int64_t batch,
                        int64_t batch_stride, const fpssft_shape *shape,
                        const int32_t *alpha_tau, int32_t per_instance, void *lines,
                        int32_t precision, void *stream);

/*
 * Batched 1/L-normalised forward DFT (transform.py:17-22, dft_forward).
 * lines/out: [B, L] complex64 (F32) or complex128 (F64); may alias.
 */
int fpssft_dft_forward(const void *lines, int64_t batch, int32_t L, void *out,
                       int32_t precision, void *stream);

/*
 * Per-bin 1-sparse test + OFDM phase decode + verification, vectorised over
 * all L bins (decoder.py:127-169, decode_spectra) plus the driver's
 * bin-consistency guard (driver.py:166-176) when alpha is given.
 *   spectra: [B, D+1, L] complex (precision); alpha_tau: [B or 1, 2, D].
 *   floor:   the energy floor handed to decode_spectra (driver.py:156).
 *   status:  [B, L] int32: 0 not a candidate, 1 candidate rejected,
 *            2 accepted, 3 decoded but failed the bin guard.
 *   freqs:   [B, L, D] int32 decoded m (valid where status >= 2).
 *   amps:    [B, L, 2] double (valid where status >= 2).
 *   n_candidates: [B] int32.
 */
int fpssft_decode_spectra(const void *spectra, int64_t batch, const fpssft_shape *shape,
                          const int32_t *alpha_tau, int32_t per_instance,
                          const fpssft_params *params, double floor, int32_t *status,
                          int32_t *freqs, double *amps, int32_t *n_candidates,
                          void *stream);

/*
 * Project a sparse set onto the line bins (decoder.py:172-191,
 * project_onto_bins; bin map numtheory.py:139-153):
 *   out[b, bin(m)] += a * exp(2 pi j u_tau(m) / L), summed in entry order.
 *   freqs [B, k_max, D] int32, amps [B, k_max, 2] double, counts [B] int32,
 *   alpha_tau [B or 1, 2, D], out [B, L, 2] double.
 */
int fpssft_project_onto_bins(const int32_t *freqs, const double *amps, const int32_t *counts,
                             int64_t batch, int32_t k_max, const fpssft_shape *shape,
                             const int32_t *alpha_tau, int32_t per_instance, double *out,
                             int32_t precision, void *stream);

/*
 * The recovery loop of ONE large problem, device-resident (driver.py:121-212
 * for recovered sets / lines beyond one CTA's shared memory: the imaging
 * duality path, 512 x 576 cubes, L = 4608, ~20k entries; reference
 * imaging.py:104-143 calls fps_sft on such a cube).  The whole loop is one
 * CUDA graph launch: a conditional WHILE node whose body is one iteration
 * (gather, DFT, peel, classify, merge, termination); the device sets the
 * loop condition, the host waits once at the end.  float64 only
 * (params->precision = FPSSFT_F64).
 *   cube:      one complex64 (FPSSFT_F32) or complex128 (FPSSFT_F64) cube,
 *              strides from shape->strides.
 *   schedule:  [params->t_max, 2, D] int32 (alpha, tau) per iteration.
 *   workspace: device buffer of fpssft_recover_large_workspace(shape, k_cap)
 *              bytes (k_cap = params->k_cap).
 *   freqs [k_cap, D] int32, amps [k_cap, 2] double: the live entries in
 *   insertion order (the reference dict's); count, iterations,
 *   samples_used, terminated_by: scalars; iter_stats [t_max, 3] or NULL.
 * Blocks until the loop has finished (synchronises `stream`).
 */
int64_t fpssft_recover_large_workspace(const fpssft_shape *shape, int32_t k_cap);
int fpssft_recover_large(const void *cube, int32_t cube_precision, const fpssft_shape *shape,
                         const fpssft_params *params, const int32_t *schedule, void *workspace,
                         int64_t workspace_bytes, int32_t *freqs, double *amps, int32_t *count,
                         int32_t *iterations, int64_t *samples_used, int32_t *terminated_by,
                         int32_t *iter_stats, void *stream);

/*
 * Dense re-synthesis of recovered spectra on the full grid (config 5's
 * "inverse-synthesise each image"): for every instance b
 *   cube_b[n] = sum_{i < counts[b]} amps[b,i] * exp(+2 pi j sum_k n_k freqs[b,i,k] / N_k)
 * -- the dense equivalent of SyntheticSource.sample_many (core.py:176-217),
 * exact integer-phase roots.  freqs [B, k_cap, D] int32, amps [B, k_cap, 2]
 * double (the fpssft_run_batch outputs), cubes: complex64 row-major,
 * cube_b = cubes + b*batch_stride (elements).
 */
int fpssft_synthesize(const int32_t *freqs, const double *amps, const int32_t *counts,
                      int64_t batch, int32_t k_cap, const fpssft_shape *shape, void *cubes,
                      int64_t batch_stride, int32_t precision, void *stream);

/* Dynamic shared memory one fpssft_run_batch CTA needs (0 if unsupported). */
size_t fpssft_smem_bytes(const fpssft_shape *shape, const fpssft_params *params);

/* Threads per CTA of the CTA-per-instance kernel for this shape. */
int fpssft_block_threads(const fpssft_shape *shape, int32_t precision);

/* Launch plan fpssft_run_batch would use: mode (FPSSFT_MODE_CTA/WARP),
 * threads per CTA, instances per CTA, dynamic shared memory per CTA.
 * Returns 0, or an error code if the shape/params cannot run. */
int fpssft_plan(const fpssft_shape *shape, const fpssft_params *params, int32_t *mode,
                int32_t *threads_per_cta, int32_t *instances_per_cta, size_t *smem_bytes);

/* The plan of fpssft_run_batch_grouped for a batch stored `group` instances
 * interleaved, with (per_instance_schedules != 0) or without a sched_index:
 * a shared schedule over an interleaved batch lets the CTA's warps gather
 * their group's lines together (instances per CTA then divides `group`). */
int fpssft_plan_batch(const fpssft_shape *shape, const fpssft_params *params, int32_t group,
                      int32_t per_instance_schedules, int32_t *mode, int32_t *threads_per_cta,
                      int32_t *instances_per_cta, size_t *smem_bytes);

/* Number of kernel launches fpssft_run_batch issues per call (for accounting). */
int fpssft_launches_per_batch(void);

/*
 * Device-wide L2 fetch granularity (cudaLimitMaxL2FetchGranularity) for the
 * current device, in bytes (0 = driver default, else 32/64/128).  The line
 * gather touches isolated 8-byte samples, so 32 B keeps DRAM traffic near
 * one sector per sample.  Process-wide side effect: opt-in, never implicit.
 */
int fpssft_set_l2_fetch_granularity(int32_t bytes);
int fpssft_get_l2_fetch_granularity(void);

const char *fpssft_last_error(void);
int fpssft_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FPSSFT_H_ */
