/*
 * tnrd.h -- C ABI of the B200-native TNRD despeckling inference path.
 *
 * The reference (specklediff, pure Python) has no FFI; its "operator API" is
 * the Python function set below.  Each entry point here is what a binding of
 * that function would call (the ctypes binding lives in
 * paper_1702_07482_b200/_lib.py).  Reference paths are
 * relative to /root/reference/pkg/src/specklediff.
 *
 *   tnrd_model_create     <- DiffusionModel + StageParams (diffusion.py:46-130)
 *                            parameters uploaded once; kernels are the
 *                            reference's k_i = coeffs @ basis.T (diffusion.py:76-77)
 *   tnrd_despeckle        <- run_diffusion            (diffusion.py:227-242)
 *   tnrd_stage            <- diffusion_step           (diffusion.py:184-194)
 *                            (and diffusion_force, diffusion.py:171-181, with
 *                            TNRD_STAGE_FORCE)
 *   tnrd_plan_*_host      <- run_diffusion called with host arrays (the
 *                            reference's only calling convention)
 *   tnrd_conv2d           <- conv2d                   (imageops.py:53-72)
 *   tnrd_prox_idiv        <- prox_idiv                (speckle.py:111-121)
 *   tnrd_stage_backward   <- _stage_backward          (training.py:69-123)
 *   tnrd_conv2d_adjoint   <- conv2d_adjoint           (imageops.py:75-106)
 *   tnrd_patch_correlation<- patch_correlation        (imageops.py:109-127)
 *   tnrd_sample_speckle   <- sample_speckle/speckle_field (speckle.py:51-70),
 *                            statistical parity (own counter-based generator)
 *
 * Conventions
 *   - images are fp32, row-major, `ld` elements between rows and
 *     `image_stride` elements between images of a batch;
 *   - device entry points are stream-ordered and asynchronous, allocate
 *     nothing, and report data-dependent errors through a 2-word device
 *     status block (see tnrd_status_*);
 *   - return codes: 0 ok, TNRD_EINVAL (-> ValueError), TNRD_ENONFINITE
 *     (-> FloatingPointError "non-finite image after stage t"), TNRD_ECUDA
 *     (-> RuntimeError), TNRD_EUNSUPPORTED (-> NotImplementedError);
 *     tnrd_last_error() returns the thread's last message.
 */
#ifndef TNRD_H
#define TNRD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define TNRD_OK 0
#define TNRD_EINVAL 1
#define TNRD_ENONFINITE 2
#define TNRD_ECUDA 3
#define TNRD_EUNSUPPORTED 4

/* tnrd_stage flags */
#define TNRD_STAGE_FLOOR_INPUT 0x1u  /* u_in := max(u_in, 1e-6) on load (initial_state, diffusion.py:219-224) */
#define TNRD_STAGE_TOP_HALO 0x2u     /* rows -2r..-1 of u_in are real halo rows (row strip), not mirrored */
#define TNRD_STAGE_BOTTOM_HALO 0x4u  /* rows H..H+2r-1 of u_in are real halo rows */
#define TNRD_STAGE_FORCE 0x8u        /* write the diffusion force instead of the prox output */
#define TNRD_STAGE_CHECK_F 0x10u     /* validate f (finite, >= 0) -> status flags */
#define TNRD_STAGE_PROJECTED 0x20u   /* projected-variant reaction (set from the model's variant) */

#define TNRD_VARIANT_PROX 0
#define TNRD_VARIANT_PROJECTED 1

/* status block: 2 x uint32 in device memory, reset to 0xFF bytes */
#define TNRD_STATUS_WORDS 2
#define TNRD_STATUS_F_NONFINITE 0x1u /* f contained NaN/Inf   (imageops.py:25) */
#define TNRD_STATUS_F_NEGATIVE 0x2u  /* f contained values < 0 (diffusion.py:231-232) */

typedef struct tnrd_model tnrd_model;
typedef struct tnrd_plan tnrd_plan;

const char* tnrd_last_error(void);
const char* tnrd_version(void);

/* Upload one model.  kernels: T*nk*m*m (float64, the reference's true-
 * convolution kernels k_i); weights: T*nk*M; lam: T (lambda = exp(beta));
 * centres mu_j = mu0 + j*delta (RbfGrid.centers, influence.py:29-31);
 * gamma = RbfGrid.gamma (influence.py:33-37).  The handle is immutable after
 * creation and may be shared between threads/streams. */
int tnrd_model_create(int m, int nk, int T, int M, const double* kernels,
                      const double* weights, double mu0, double delta,
                      double gamma, const double* lam, int device,
                      tnrd_model** out);
int tnrd_model_destroy(tnrd_model* model);
/* Part of construction (call before sharing the handle): select the reaction
 * step -- TNRD_VARIANT_PROX (default, diffusion.py:184-194) or
 * TNRD_VARIANT_PROJECTED with its floor (diffusion.py:197-224: u_0 =
 * max(f, floor), u' = smooth_max(u - force - lam (1/u - f^2/u^3), floor)). */
int tnrd_model_set_variant(tnrd_model* model, int variant, double floor);
/* m, nk, T, M, rbf path (1 = piecewise-polynomial table, 0 = direct
 * all-centre sum) */
int tnrd_model_info(const tnrd_model* model, int* m, int* nk, int* T, int* M,
                    int* fast_rbf);
/* Accuracy of the polynomial RBF tables built at creation: max |p - phi|
 * over every interval/filter/stage with float64 and with the fp32-rounded
 * coefficients the kernel uses (both evaluated in float64), the largest
 * sum_j |w_ij|, and the interval count (0 on the direct path). */
int tnrd_model_rbf_fit(const tnrd_model* model, double* max_abs_err,
                       double* max_abs_err_fp32, double* max_sum_abs_w,
                       int* intervals);
/* Same for the cubic table the parameter-space-taps kernels evaluate
 * (intervals of width min(delta, gamma) / 10, one float4 of monomial
 * coefficients each): max |p - phi| with float64 and with the fp32
 * coefficients, and the number of intervals (0 = no cubic table: those
 * kernels are not used for this model). */
int tnrd_model_rbf_fit_cubic(const tnrd_model* model, double* max_abs_err,
                             double* max_abs_err_fp32, int* intervals);

/* Stage kernel selection (process-wide): 0 = auto (the kernel measured
 * fastest on B200 for the grid size), 1 = CUDA-core kernels
 * (same choice as auto), 2 = tcgen05 forward-GEMM kernel (error if the
 * model is unsupported: m > 7 or RBF tables too large), 3 / 4 = CUDA-core
 * tile kernel with its small (32x32) / large (64x64) tiles forced, 5 = the
 * phase-locked tcgen05 kernel, 6 / 7 = CUDA-core split kernel ((tile,
 * filter group) units + ordered reduction, 2 launches per stage) with
 * large / small tiles forced, 8 = z-field stage (tcgen05 forward filter
 * bank over the whole image into per-stream z planes, then a TMA-fed
 * CUDA-core RBF + adjoint + prox kernel; m <= 7, nk <= 128), 9 = fused dataflow despeckle (all stages of
 * tnrd_despeckle in one persistent launch, tiles of stage t+1 started as
 * their neighbourhood of stage t is reduced; opt-in, measured slower on
 * B200 than the per-stage split kernel), 10 / 11 = cluster kernel with
 * large / small tiles forced: ONE launch per stage on small grids -- the
 * CTAs of a thread-block cluster split a tile's filter groups, keep their
 * partial forces in shared memory and sum them in rank order through
 * distributed shared memory, each CTA finishing its share of the tile's
 * pixels (diffusion_step, diffusion.py:184-194, as one operator), 12 =
 * tensor-core adjoint (two launches per stage: a CUDA-core kernel writes
 * phi = RBF(conv(u, k)) once per pixel, a tcgen05 kernel runs the adjoint
 * filter bank as a 3xTF32 GEMM with the shifted sum and the reaction in its
 * epilogue; m = 5, 7; other models and strip launches silently use the
 * CUDA-core kernels; opt-in: parity-green but measured slower than the fused
 * kernel on B200; keeps a phi workspace per stream inside
 * the model).  Auto runs the tile kernel from 6 waves of large tiles and the
 * cluster kernel below (one launch per stage either way); the split kernel
 * (modes 6 / 7) keeps a partial-force workspace per stream inside the model
 * (allocated on first use, outside stream capture). */
int tnrd_set_stage_kernel(int mode);
/* CTAs per cluster of the cluster kernel: 0 = chosen from the grid size
 * (the largest cluster <= 8 whose CTAs fit one wave), 2..8 = forced.  The
 * partial forces are summed in cluster-rank order, so results are
 * bit-reproducible for a given cluster size and differ between sizes by
 * fp32 summation order only. */
int tnrd_set_cluster_size(int ctas);
/* Where the CUDA-core large-tile stage kernels read the filter taps
 * (process-wide): 1 (default) = the kernel parameter space, read by the
 * uniform datapath (m <= 7, nk <= 48 with m = 7); 0 = staged in shared memory
 * and held in registers.  Both give bit-identical results; the initial value
 * can be set with TNRD_PARAM_TAPS=0|1 in the environment. */
int tnrd_set_param_taps(int on);
/* z-field stage precision (process-wide): number of tf32 cross products of
 * the 3-piece splits of u and k -- 6 (default: below fp32 rounding), 4 or 3
 * (experiments). */
int tnrd_set_zfield_passes(int n);

/* Reset a device status block (stream-ordered memset). */
int tnrd_status_reset(uint32_t* d_status, void* stream);
/* Decode a HOST copy of the status block: returns TNRD_OK, TNRD_EINVAL (bad
 * f) or TNRD_ENONFINITE with *bad_stage set; also sets the last error. */
int tnrd_status_decode(const uint32_t* h_status, int* bad_stage);

/* One stage t of the model: u_out = prox(u_in - force(u_in), f, lam_t)
 * (or the force with TNRD_STAGE_FORCE).  u_in/f/u_out: device pointers, may
 * not alias.  For strips, u_in must be addressable 2r rows above row 0 /
 * below row H-1 on the halo edges. */
int tnrd_stage(const tnrd_model* model, int t, const float* u_in,
               const float* f, float* u_out, int batch, int H, int W,
               int64_t ld, int64_t image_stride, uint32_t flags,
               uint32_t* d_status, void* stream);

/* All T stages, ping-ponging between u_out and work (same shape), the
 * final stage landing in u_out.  Stage 0 reads f as u_0 with the 1e-6 floor
 * (initial_state) and validates f into the status block.  Large batches
 * may run their two halves on an internal second stream forked from and
 * joined back into `stream` (same bits; ordering on `stream` is kept, and
 * the call may be captured into a CUDA graph after one eager call on that
 * stream); TNRD_BATCH_FORK=0 in the environment disables it. */
/* tnrd_stage that also writes the stage's force (sum_i rot180(k_i) *
 * phi_i(k_i * u), diffusion.py:171-181) to force_out (same layout as u_out)
 * in the same launch: diffusion_step's u_next and its trace's
 * u~ = u - force without a second pass (CUDA-core kernels; not with
 * TNRD_STAGE_FORCE). */
int tnrd_stage_force(const tnrd_model* model, int t, const float* u_in,
                     const float* f, float* u_out, float* force_out, int batch,
                     int H, int W, int64_t ld, int64_t image_stride,
                     uint32_t flags, uint32_t* d_status, void* stream);
int tnrd_despeckle(const tnrd_model* model, const float* f, float* u_out,
                   float* work, int batch, int H, int W, int64_t ld,
                   int64_t image_stride, uint32_t* d_status, void* stream);

/* Plans own device buffers, a status block, pinned staging and a stream for
 * one (batch, H, W) shape; use one plan per host thread. */
int tnrd_plan_create(const tnrd_model* model, int batch, int H, int W,
                     tnrd_plan** out);
int tnrd_plan_destroy(tnrd_plan* plan);
/* Full despeckle from/to HOST buffers (batch*H*W fp32, dense): H2D, all T
 * stages, D2H, synchronise, decode status.  Host buffers may be pageable or
 * pinned.  A single image of >= 2 x 3 waves of 64x64 tiles (e.g. a 16384^2
 * scene) runs as up to 16 tile-aligned row bands on their own streams, each
 * band's H2D, T stages (neighbour rows read in place) and D2H ordered by
 * events only where data flows, so the copies overlap the stages (pinned
 * buffers needed for the overlap; TNRD_SCENE_BANDS overrides the count).
 * The result is bit-identical to the unbanded despeckle. */
int tnrd_plan_despeckle_host(tnrd_plan* plan, const float* f_host,
                             float* u_host);
/* A sequence of `count` host images (each batch*H*W fp32, dense, back to
 * back in f_host / u_host): image i's copies and stages run round-robin on
 * the plan and up to 5 internal twin plans (own streams and buffers; 6 plans
 * for plans of <= 64 MB per buffer, else 2; TNRD_STREAM_DEPTH overrides), so
 * one image's H2D / D2H overlap the next ones' stages and small images run
 * concurrently (pinned host buffers needed for the overlap).  Synchronous; returns the first failing image's
 * error with *bad_index set (-1 if none). */
int tnrd_plan_despeckle_host_many(tnrd_plan* plan, const float* f_host,
                                  float* u_host, int count, int* bad_index);
/* Device-resident variant on the plan's stream (no sync, no status check). */
int tnrd_plan_despeckle_device(tnrd_plan* plan, const float* f_dev,
                               float* u_dev);
/* Synchronise the plan's stream and decode its status block. */
int tnrd_plan_check(tnrd_plan* plan, int* bad_stage);
void* tnrd_plan_stream(tnrd_plan* plan);
/* Device buffers owned by the plan: f (input) and u (output). */
float* tnrd_plan_f_device(tnrd_plan* plan);
float* tnrd_plan_u_device(tnrd_plan* plan);

/* Same-size true convolution with half-sample mirror padding (conv2d,
 * imageops.py:53-72); k: m*m float64 host array, m odd, m <= 15. */
/* ---- training backward ---------------------------
 * One stage of training.py:69-123 (_stage_backward) on a dense H x W image:
 * device u_prev, f, g_next (= dL/du_next; NULL = zero), g_prev (device out,
 * may be NULL); host outputs (each may be NULL): grad_beta (scalar),
 * grad_k[nk][m*m] = the kernel-space gradient gk_i (training.py:108-109;
 * the caller maps it to coefficients with basis^T like training.py:110),
 * grad_w[nk][M].  Works for both reaction variants.  Synchronous; bit-
 * reproducible (fixed-order float64 reductions). */
int tnrd_stage_backward(const tnrd_model* model, int t, const float* u_prev,
                        const float* f, const float* g_next, float* g_prev,
                        int H, int W, double* grad_beta, double* grad_k,
                        double* grad_w, void* stream);
/* imageops.py:75-106: exact transpose of conv2d(., k) (mirror padded),
 * dense device images; k is m x m float64 (row-major). */
int tnrd_conv2d_adjoint(const float* img, float* out, int H, int W,
                        const double* k, int m, void* stream);
/* imageops.py:109-127: C[a][b] = sum_P pad(base)[P + (a, b)] adj[P], dense
 * device images, out = host m x m float64.  Synchronous. */
int tnrd_patch_correlation(const float* base, const float* adj, int H, int W,
                           int m, double* out, void* stream);

/* L-look amplitude speckle on the GPU (speckle.py:51-70, SURVEY §8(f) rank
 * 3): out = clean * sqrt(G / L), G ~ Gamma(L, 1) per pixel; clean == NULL
 * writes the field sqrt(G / L) itself.  Generator: Philox4x32-10 keyed by
 * `seed`, counter (pixel index, attempt, 0) with pixel index = image*H*W +
 * y*W + x, and Marsaglia-Tsang gamma (tnrd_speckle.cuh).  Bit-reproducible
 * for a given (seed, looks, shape) under any launch geometry; equal to the
 * reference's numpy Generator(Philox).gamma in distribution only (the
 * reference's sequential rejection stream has no parallel equivalent).
 * With d_status (may be NULL) a non-finite / negative clean pixel clears
 * bit 0 / 1 of d_status[1] (decoded by tnrd_status_decode as bad input). */
int tnrd_sample_speckle(const float* clean, float* out, int batch, int H,
                        int W, int64_t ld, int64_t image_stride, int looks,
                        uint64_t seed, uint32_t* d_status, void* stream);
/* The generator's integer core on the host (known-answer tests). */
void tnrd_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2],
                        uint32_t out[4]);

int tnrd_conv2d(const float* img, float* out, int H, int W, int64_t ld,
                const double* k, int m, void* stream);
/* Closed-form I-divergence prox (prox_idiv, speckle.py:111-121). */
int tnrd_prox_idiv(const float* u_tilde, const float* f, float* out,
                   int64_t n, double lam, void* stream);

/* Number of kernel launches issued by this library (process-wide) since
 * the last reset (instrumentation for bench.py's gpu_launches). */
uint64_t tnrd_launch_count(void);
/* Build features of this library: TNRD_FEATURE_EXPERIMENTS = the opt-in
 * tensor-core / dataflow stage kernels (modes 2, 5, 8, 9 of
 * tnrd_set_stage_kernel) are compiled in (-DTNRD_EXPERIMENTS; they are not
 * in the default build). */
#define TNRD_FEATURE_EXPERIMENTS 0x1u
uint32_t tnrd_build_features(void);
void tnrd_launch_count_reset(void);

/* Peak probes for the roofline denominators (not on the reference's path):
 * kind 0 = FP32 FFMA, 1 = MUFU ex2.  Launches one saturating kernel on
 * `stream` and returns its operation count in *ops (FLOP for kind 0). */
int tnrd_probe(int kind, int iters, int blocks_per_sm, void* stream,
               double* ops);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* TNRD_H */
