/* pnp_b200 — C ABI of the B200-native DSG-NLM / linearized PnP-ADMM hot path.
 *
 * Drop-in for the reference's hot path (arXiv 1901.06110, package
 * `pnprestore`, /root/reference/pkg/src/pnprestore).  The reference is pure
 * Python; its "FFI" for this path is the Python call surface listed per
 * function below.  The package `paper_1901_06110_b200` binds these symbols
 * with ctypes and keeps the reference's Python names/semantics on top.
 *
 * Conventions
 *  - float32 planes, row-major, contiguous; a batch of B images of H x W is
 *    B*H*W floats.  All data pointers are DEVICE pointers owned by the caller
 *    unless stated otherwise.  Work is stream-ordered on the context stream.
 *  - Return value: PNP_OK or an error code; pnp_last_error() gives a
 *    thread-local message.  PNP_EINVAL maps to ValueError, PNP_ECUDA to
 *    RuntimeError, PNP_ENONFINITE to ValueError / DivergenceError.
 *  - Patch taps: P host floats, normalized (sum 1).  taps = 1/P reproduces the
 *    reference's box patch distance; a sampled Gaussian gives the BASELINE
 *    "Gaussian patch weights" extension.  `bandwidth` is the reference's
 *    PatchParams.bandwidth (north-star h = sqrt(2) * bandwidth).
 */
#ifndef PNP_B200_H
#define PNP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PNP_OK 0
#define PNP_EINVAL 1
#define PNP_ECUDA 2
#define PNP_ENONFINITE 3
#define PNP_ENCCL 4

typedef struct pnp_ctx pnp_ctx;
typedef struct pnp_frozen pnp_frozen;

/* ---- context ------------------------------------------------------------ */
int pnp_version(void);
const char* pnp_last_error(void);
/* One context per device per host thread: owns scratch arenas and a stream
 * handle (default: the legacy stream 0 until pnp_ctx_set_stream). */
int pnp_ctx_create(int device, pnp_ctx** out);
int pnp_ctx_destroy(pnp_ctx* ctx);
/* stream = a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream). */
int pnp_ctx_set_stream(pnp_ctx* ctx, void* stream);
int pnp_ctx_synchronize(pnp_ctx* ctx);
/* k cache: the pair weights hat*k of sweep A are kept in HBM (half window,
 * 4 B per pixel and offset pair) when they fit, so sweep B / frozen applies
 * stream them instead of recomputing the patch filter; results are bitwise
 * identical either way.  bytes = 0 disables, < 0 = no limit (default).  When
 * the whole cache does not fit (the budget or free HBM less 4 GiB), the tile
 * rows that fit are cached and the rest recomputed (at least 1/8 of them, else
 * none).  A frozen guide uses the buffer bound with pnp_ctx_bind_kcache when
 * it is created (the buffer must then outlive the handle; the Python layer
 * binds torch memory and keeps it with the FrozenGuide), else allocates its
 * cache from the device's stream-ordered pool (cudaMallocAsync) and frees it
 * on the stream of its last use.  An adaptive
 * denoise holds its cache only for the duration of the call: a buffer the
 * caller bound with pnp_ctx_bind_kcache (the Python layer binds memory from
 * torch's caching allocator, so torch sees and reuses it), else a
 * stream-ordered pool allocation freed at the end of the call
 * (pnp_ctx_trim returns the pool's idle memory to the device). */
int pnp_ctx_set_cache_limit(pnp_ctx* ctx, int64_t bytes);
int pnp_ctx_bind_kcache(pnp_ctx* ctx, void* ptr, int64_t bytes);
int pnp_ctx_trim(pnp_ctx* ctx);
int pnp_frozen_cached(const pnp_frozen* fz);
/* Per-launch CUDA-event timing on the context stream (off by default).
 * profile_read syncs the stream, returns summed device ms and launch counts
 * for 6 categories (0 DSG recompute sweep, 1 DSG fixup/finalize, 2 forward
 * operators, 3 ADMM elementwise/reductions, 4 DSG k-cache sweep, 5 input
 * validation) since the last read, and resets them. */
int pnp_ctx_profile(pnp_ctx* ctx, int enable);
int pnp_ctx_profile_read(pnp_ctx* ctx, double* ms, int* launches);
/* Measured FFMA / MUFU.EX2 instruction throughput of the device (per second,
 * whole GPU) — the roofline denominators of the DSG sweep. */
int pnp_peak_rates(int device, double* ffma_per_s, double* ex2_per_s);
/* Pre-size scratch for (batch, H, W, R, P, box taps?) so later calls allocate
 * nothing (required before CUDA-graph capture). */
int pnp_ctx_reserve(pnp_ctx* ctx, int batch, int H, int W, int R, int P, int box);

/* ---- DSG-NLM ------------------------------------------------------------ */
/* dsg_nlm_denoise(image, params, guide) — reference denoise.py:272-288.
 * out = K x / m + (1 - d / m) x with K = D^-1/2 (hat o K_nlm) D^-1/2,
 * d = K 1 (normalized row sums), m = max d per image.
 * taps: P normalized 1-D patch taps.  Equal taps (1/P) are the reference's
 * box patch distance; from P = 11 they run the general sweep with
 * running-sum box filters (cost flat in P; any odd P <= 63, any R), below it
 * the P-templated sweep.  Other taps (Gaussian) run the P-templated sweep for
 * P <= 15, R <= 32 and the general sweep beyond.
 * guide may equal x.  d_out (B*H*W) and alpha_out (B floats, = m) are
 * optional device outputs. */
int pnp_dsg_denoise(pnp_ctx* ctx, const float* x, const float* guide, float* out,
                    int batch, int H, int W, int R, int P, const float* taps,
                    double bandwidth, float* d_out, float* alpha_out);

/* dsg_nlm_denoise(..., distances="direct") — the reference's brute-force
 * per-pixel path (denoise.py:291-355): three passes with the patch distance
 * summed directly over the P x P patch (cost window area x patch area); the
 * bench-denoiser timing baseline.  Same result as pnp_dsg_denoise within fp32
 * rounding (P <= 63). */
int pnp_dsg_denoise_direct(pnp_ctx* ctx, const float* x, const float* guide, float* out,
                           int batch, int H, int W, int R, int P, const float* taps,
                           double bandwidth);

/* freeze_guide(guide, params) -> FrozenGuide — denoise.py:358-386.  The
 * library-owned handle copies the guide and keeps rs = g^-1/2, d and m. */
int pnp_dsg_freeze(pnp_ctx* ctx, const float* guide, int batch, int H, int W, int R,
                   int P, const float* taps, double bandwidth, pnp_frozen** out);
/* FrozenGuide.apply(image) — denoise.py:375-381; bit-identical to
 * pnp_dsg_denoise(x, guide) with the frozen guide. */
int pnp_dsg_apply(pnp_ctx* ctx, const pnp_frozen* fz, const float* x, float* out);
int pnp_frozen_destroy(pnp_frozen* fz);
/* Copies of the handle's state: alpha (m) per image to HOST memory, the
 * guide / row sums d to caller device buffers (either may be null). */
int pnp_frozen_alpha(const pnp_frozen* fz, float* alpha_host);
int pnp_frozen_export(pnp_ctx* ctx, const pnp_frozen* fz, float* guide_out, float* d_out);
int pnp_frozen_shape(const pnp_frozen* fz, int* batch, int* H, int* W, int* R, int* P);
/* Residency of the handle's pair-weight (k) cache: tile rows per image it
 * covers (from the top; the rest recompute on apply), tile rows per image and
 * its bytes.  No reference counterpart (the reference recomputes weights). */
int pnp_frozen_cache(const pnp_frozen* fz, int* rows_cached, int* tile_rows,
                     unsigned long long* bytes);

/* nlm_denoise(image, params, guide) — denoise.py:254-269 (row-stochastic). */
int pnp_nlm_denoise(pnp_ctx* ctx, const float* x, const float* guide, float* out,
                    int batch, int H, int W, int R, int P, const float* taps,
                    double bandwidth);

/* Single-image denoise whose sweep A starts before the whole image is on the
 * device (pipelined uploads, DenoiseStream): the image is split into
 * `nbands` bands of tile rows (pnp_dsg_band_rows gives band j's last tile
 * row + 1 in tile_end[j] and the input rows [0, rows_needed[j]) it reads);
 * band j's sweep A waits for events[j] (a cudaEvent_t recorded once those
 * rows are uploaded; NULL = no wait), the rest of the denoise runs after the
 * last band.  Guide = x.  Bitwise equal to pnp_dsg_denoise. */
int pnp_dsg_band_rows(int H, int W, int R, int P, int box, int nbands, int* tile_end,
                      int* rows_needed);
int pnp_dsg_denoise_banded(pnp_ctx* ctx, const float* x, float* out, int H, int W, int R, int P,
                           const float* taps, double bandwidth, int nbands,
                           void* const* events);
/* The same denoise driven band by band by a caller that produces the image on
 * the host as it goes (the numpy drop-in path: cast + upload of band j+1
 * overlaps sweep A of band j).  Call pnp_dsg_band_sweep for j = 0 .. nbands-1
 * in order, each after the context stream is ordered behind the upload of
 * input rows [0, rows_needed[j]); then pnp_dsg_band_finish.  Band 0 sizes the
 * buffers and the k cache.  Guide = x.  Bitwise equal to pnp_dsg_denoise. */
int pnp_dsg_band_sweep(pnp_ctx* ctx, const float* x, int H, int W, int R, int P,
                       const float* taps, double bandwidth, int nbands, int j);
int pnp_dsg_band_finish(pnp_ctx* ctx, const float* x, float* out, int H, int W, int R, int P,
                        const float* taps, double bandwidth);

/* ---- row-strip building blocks (multi-GPU sharding) ---- *
 * A rank owns global rows [y0, y1) = whole tile rows of height TH
 * (pnp_dsg_geometry).  Per-pixel buffers are windows: rows [buf_r0, buf_r0 +
 * buf_rows) of the Hg x W image (own rows plus halos received from
 * neighbours).  Partial buffers hold part_ntr tile rows x pnp_dsg_groups()
 * offset groups x ceil(W/64) tiles of C*(TH+Rb)*(64+2Rb) floats
 * (pnp_dsg_partial_floats gives the total); slot 0 is
 * global tile row part_tr0 (a neighbour's rows are received into the
 * prefix).  A sharded run sums in exactly the single-GPU order, so its
 * output is bit-identical.
 *   sweep pass: 0 mass g (C=1), 1 Kx+d (C=2, needs x, rs), 2 d (C=1, rs),
 *               3 Kx (C=1, x, rs)
 *   fixup mode: 0 rs = g^-1/2, 1 Kx, d + per-rank max bits, 2 d + max,
 *               3 frozen apply (out = Kx inv_m + (1 - d inv_m) x)
 *   finalize:   out = Kx/m + (1 - d/m) x with m from (all-reduced) mbits.
 * kcache (nullable, pnp_dsg_kcache_floats(.., ntr) floats, caller-owned):
 * pass 0 also stores the strip's pair weights, passes 1-3 then stream them
 * instead of recomputing the patch filter (bitwise identical results). */
/* out[8] = {TH tile height, offset groups, Rb far band of a partial block
 * (R; 0 when blocks are tile-only), sweep path (0 P-templated, 1 general
 * half window, 2 general full window), input halo rows above, input halo
 * rows below, rows of the channel (rs) planes read below, 0}. */
int pnp_dsg_geometry(int Hg, int W, int R, int P, int box, int* out);
int pnp_dsg_groups(int Hg, int W, int R, int P, int box);
int64_t pnp_dsg_partial_floats(int Hg, int W, int R, int P, int box, int C, int ntr);
int64_t pnp_dsg_kcache_floats(int Hg, int W, int R, int P, int box, int ntr);
int pnp_dsg_strip_sweep(pnp_ctx* ctx, int pass, const float* guide, const float* x,
                        const float* rs, int Hg, int W, int buf_r0, int buf_rows, int tr0,
                        int ntr, int R, int P, const float* taps, double bandwidth,
                        float* partial, int part_off, int part_ntr, float* kcache);
int pnp_dsg_strip_fixup(pnp_ctx* ctx, int mode, const float* partial, int part_tr0,
                        int part_ntr, int Hg, int W, int R, int P, int box, int y0, int y1,
                        int buf_r0, int buf_rows, float* rs, float* kx, float* d, unsigned* mbits,
                        const float* inv_m, const float* x, float* out);
int pnp_dsg_strip_finalize(pnp_ctx* ctx, const float* kx, const float* d, const float* x,
                           float* out, const unsigned* mbits, int Hg, int W, int y0, int y1,
                           int buf_r0, int buf_rows);

/* ---- forward operators (forward.py) ------------------------------------- */
/* SR operator: separable blur k = ty tx^T given as 2(2r+1) host floats
 * (ty then tx; the reference's gaussian_kernel is such an outer product),
 * integer factor, boundary 0 = periodic (wrap), 1 = half-sample symmetric
 * (forward.py:98-148). */
int pnp_sr_apply(pnp_ctx* ctx, const float* x, float* y, int batch, int H, int W,
                 const float* taps, int radius, int factor, int boundary);
int pnp_sr_adjoint(pnp_ctx* ctx, const float* y, float* x, int batch, int H, int W,
                   const float* taps, int radius, int factor, int boundary);
/* grad = A^T (A x - y) (forward.py:183-185); if data_out != null it receives
 * 0.5 ||A x - y||^2 per image (double, device). */
int pnp_sr_grad(pnp_ctx* ctx, const float* x, const float* yobs, float* grad, int batch,
                int H, int W, const float* taps, int radius, int factor, int boundary,
                double* data_out);
/* QIS gradient (forward.py:322-327) and data term (312-319, double per image).
 * pnp_qis_grad: grad may be null (data only), data_out may be null. */
int pnp_qis_grad(pnp_ctx* ctx, const float* x, const float* ones, const float* zeros,
                 float* grad, int batch, int n, double gain_over_K, double floor_,
                 double* data_out);
int pnp_qis_data(pnp_ctx* ctx, const float* x, const float* ones, const float* zeros,
                 int batch, int n, double gain_over_K, double floor_, double* data_out);
/* qis_simulate Knuth loop on the HOST (forward.py:263-298): stop[i] =
 * exp(-gain*clip(x)/K) precomputed by the caller; ones[i] receives the count
 * of fired jots.  Bit-exact with the reference's raster-then-jot order. */
int pnp_qis_simulate_host(const double* stop, int64_t n, int K, uint64_t seed,
                          double* ones);

/* ---- linearized ADMM pieces (solver.py:199-235) ------------------------- */
/* x <- clamp(mu (alpha x + rho (v - u) - grad)), z = x + u; flags bit0 set
 * if the pre-projection x is non-finite, bit1 if z is non-finite.  lo/hi:
 * use -inf/+inf for no bound. */
int pnp_admm_xupdate(pnp_ctx* ctx, float* x, const float* v, const float* u,
                     const float* grad, float* z, int64_t n, double mu, double alpha,
                     double rho, double lo, double hi, int* flags);
/* u <- u + x - v; stats[b*4 + 0..3] = (sum (x-v)^2, sum (rho (v-v_prev))^2,
 * sum (gt-v)^2 (if gt), 0) per image (double); flags bit2 if v or u
 * non-finite.  v_prev may be null (then 0 is used). */
int pnp_admm_uupdate(pnp_ctx* ctx, float* u, const float* x, const float* v,
                     const float* v_prev, const float* gt, int batch, int64_t n,
                     double rho, double* stats, int* flags);
/* y = clamp(x) */
/* Fused ADMM steps (same per-pixel arithmetic as the unfused calls):
 * grad f(x) + x-update (x <- proj(mu (alpha x + rho (v - u) - grad)), z = x + u,
 * flags |= 1 / 2 on non-finite x / z) in the gradient kernel's epilogue, and
 * the frozen DSG apply v = W z + u-update (u += x - v, stats[b*4+0..2] =
 * sum (x-v)^2, sum (rho (v - v_prev))^2, sum (gt - v)^2, flags |= 4) in the
 * apply's fixup epilogue.  data_out (nullable): f(x) per image. */
int pnp_sr_grad_xupdate(pnp_ctx* ctx, float* x, const float* yobs, int batch, int H, int W,
                        const float* taps, int radius, int factor, int boundary, double* data_out,
                        const float* v, const float* u, float* z, double mu, double alpha,
                        double rho, double lo, double hi, int* flags);
int pnp_qis_grad_xupdate(pnp_ctx* ctx, float* x, const float* ones, const float* zeros, int batch,
                         int n, double gain_over_K, double floor_, double* data_out,
                         const float* v, const float* u, float* z, double mu, double alpha,
                         double rho, double lo, double hi, int* flags);
int pnp_dsg_apply_admm(pnp_ctx* ctx, const pnp_frozen* fz, const float* z, float* v, float* u,
                       const float* x, const float* v_prev, const float* gt, double rho,
                       double* stats, int* flags);
/* ---- float64 distance-engine helpers (reference image.py:97-143,
 * denoise.py:70-88, 106-174).  Off the fp32 sweep path; computed on the
 * device in float64.  All pointers are device pointers. ----
 * pad_symmetric: out ((H+2m) x (W+2m)) = half-sample mirror pad of img,
 *   0 <= margin <= min(H, W) (image.py:97-113).
 * integral_image: out ((H+1) x (W+1)) = summed-area table with a zero leading
 *   row / column, sequential cumsums like numpy's (image.py:116-126; bitwise).
 * patch_distance_map: out (H x W) = sum over the P x P patch of
 *   (G(s+ab) - G(s+t+ab))^2, t = (dy, dx), |t| <= R, reflected guide with
 *   margin R + (P-1)/2 <= min(H, W); the shifted-add order of the reference's
 *   method="direct" (denoise.py:131-142; bitwise).
 * patch_ssd_pairs: out[i] = patch SSD between pixels (pairs[4i], pairs[4i+1])
 *   and (pairs[4i+2], pairs[4i+3]) (nlm_kernel, denoise.py:70-88); pairs is
 *   a device int array. */
int pnp_pad_symmetric_f64(pnp_ctx* ctx, const double* img, int H, int W, int margin, double* out);
int pnp_integral_image_f64(pnp_ctx* ctx, const double* img, int H, int W, double* out);
int pnp_patch_distance_map_f64(pnp_ctx* ctx, const double* guide, int H, int W, int P, int R,
                               int dy, int dx, double* out);
int pnp_patch_ssd_pairs_f64(pnp_ctx* ctx, const double* guide, int H, int W, int P,
                            const int* pairs, int n, double* out);
/* build_dense_weights (denoise.py:389-418): out = the n x n (n = H*W) doubly
 * stochastic W of the guide in float64 -- hat * exp(-SSD/(2 P^2 bw^2)) on the
 * clipped window (direct SSD order), scaled by row^-1/2 and col^-1/2, divided
 * by the max row sum, diagonal completed to row sums of 1.  scratch: 2n+1
 * doubles.  Test-scale (the caller bounds n). */
int pnp_dense_weights_f64(pnp_ctx* ctx, const double* guide, int H, int W, int P, int R,
                          double bandwidth, double* out, double* scratch);

/* Native iteration loop of linearized_pnp_admm with a frozen guide
 * (reference solver.py:199-235): iterations k0..k1 (1-based) of
 *   x <- proj(mu (alpha x + rho (v - u) - grad f(x))), z = x + u   (fused)
 *   v <- W z, u += x - v, stats / flags                         (fused)
 * issuing, per iteration, exactly pnp_sr_grad_xupdate (kind 0: obs = y,
 * taps/radius/factor/boundary) or pnp_qis_grad_xupdate (kind 1: obs = ones,
 * obs2 = zeros, gain_over_K, floor_) followed by pnp_dsg_apply_admm, with the
 * same per-iteration pointers the Python loop uses: flags + k-1, stats +
 * (k-1)*batch*4, objv + (k-2)*batch (objective of the previous iterate; objv
 * may be NULL).  v0 holds the current v on entry; the new v alternates
 * between v1 and v0, *v_last tells which holds the final one (0 = v0).
 * ms_out (nullable, host, k1-k0+1 floats): device time from the call's start
 * to the end of each iteration (synchronizes once at the end). */
int pnp_admm_run(pnp_ctx* ctx, int kind, const float* obs, const float* obs2, int batch, int H,
                 int W, const float* taps, int radius, int factor, int boundary,
                 double gain_over_K, double floor_, const pnp_frozen* fz, int k0, int k1, float* x,
                 float* v0, float* v1, float* u, float* z, const float* gt, double mu,
                 double alpha, double rho, double lo, double hi, double* stats, double* objv,
                 int* flags, float* ms_out, int* v_last);
/* Standard PnP-ADMM baseline (reference solver.py:244-328): the Gram operator
 * out = A^T A x + shift x of the SR model, and conjugate gradients on
 * (A^T A + shift I) x = rhs per image of a batch (cg_solve semantics: stop
 * when ||r|| / ||rhs|| <= tol or after max_iters; warm = start from x, else
 * from 0; ||rhs|| = 0 -> x = 0).  Outputs per image: iterations, relative
 * residual, status (0 ok, 2 nonpositive curvature, 3 non-finite).  Device
 * resident: scalars stay on the GPU, the host polls completion every few
 * iterations. */
/* Row-strip SR operators (sharded ADMM; batch 1).  x / r buffers hold global
 * rows [in_r0, in_r0 + in_rows) (HR for the residual, LR for the adjoint,
 * halos included); outputs are global rows [out_r0, out_r0 + out_rows) (LR
 * for the residual, HR for the adjoint).  Boundary handling uses the global
 * height Hg, so strips reproduce the whole-image operator exactly.
 * data_out (nullable, device double): 0.5 ||A x - y||^2 over the window. */
int pnp_sr_strip_residual(pnp_ctx* ctx, const float* x, const float* y, float* r, int Hg, int W,
                          int in_r0, int in_rows, int out_r0, int out_rows, const float* taps,
                          int radius, int factor, int boundary, double* data_out);
int pnp_sr_strip_adjoint(pnp_ctx* ctx, const float* r, float* out, int Hg, int W, int in_r0,
                         int in_rows, int out_r0, int out_rows, const float* taps, int radius,
                         int factor, int boundary);
/* rhs = atb + rho (v - u); z = x + u with flags |= 1 / 2 on non-finite x / z. */
int pnp_admm_std_rhs(pnp_ctx* ctx, float* rhs, const float* atb, const float* v, const float* u,
                     int64_t n, double rho);
int pnp_admm_std_z(pnp_ctx* ctx, float* z, const float* x, const float* u, int64_t n,
                   int* flags);
int pnp_sr_gram(pnp_ctx* ctx, const float* x, float* out, int batch, int H, int W,
                const float* taps, int radius, int factor, int boundary, double shift);
int pnp_sr_cg(pnp_ctx* ctx, const float* rhs, float* x, int batch, int H, int W,
              const float* taps, int radius, int factor, int boundary, double shift, double tol,
              int max_iters, int warm, int* iters_out, double* resid_out, int* status_out);
int pnp_project(pnp_ctx* ctx, const float* x, float* y, int64_t n, double lo, double hi);
/* Validation helper (reference image.py:35-40): *all_finite = 1 when no
 * element of x (n floats, device, 16 B aligned) is NaN/Inf, else 0.  One
 * pass on the ctx stream, then a synchronizing 4-byte read-back. */
int pnp_check_finite(pnp_ctx* ctx, const float* x, int64_t n, int* all_finite);

/* Host casts of the numpy drop-in path (float64 numpy in / out around the
 * fp32 device compute; the reference's call shape, denoise.py:272-288):
 * AVX2 conversions with non-temporal stores on a persistent worker pool
 * (nthreads <= 0: all of it), round-to-nearest-even = a C cast, bit for bit.
 * Host pointers; no device work. */
int pnp_host_cast_f32_f64(const float* src, double* dst, int64_t n, int nthreads);
int pnp_host_cast_f64_f32(const double* src, float* dst, int64_t n, int nthreads);
/* Zero-fill (first touch) of a fresh float64 result on the same pool: the
 * numpy path faults the result's pages in while the device computes. */
int pnp_host_zero_f64(double* dst, int64_t n, int nthreads);
/* Stream-ordered variant for pipelines: *flag (device int) |= 1 when x holds
 * a NaN/Inf; no synchronization. */
int pnp_flag_nonfinite(pnp_ctx* ctx, const float* x, int64_t n, int* flag);

/* SplitMix64 on the device (reference forward.py:36-79, SplitMix64): the n
 * uniforms a host stream with state `state` would return next
 * (uniforms(n), forward.py:58-67), bit-identical; out = n device doubles.
 * Stream-ordered, no synchronization. */
int pnp_splitmix_uniforms(pnp_ctx* ctx, uint64_t state, int64_t n, double* out);
/* Noise step of sr_simulate (forward.py:205-212): y + sigma * normals(n) of
 * SplitMix64(seed) (Box-Muller, forward.py:70-79) over the flat y (n device
 * floats), in float64; written as float32 to out32 and/or float64 to out64
 * (either may be NULL, not both).  The transcendental calls are CUDA float64
 * (within 2 ulp of the host's libm). */
int pnp_sr_add_noise(pnp_ctx* ctx, const float* y, int64_t n, uint64_t seed, double sigma,
                     float* out32, double* out64);

#ifdef __cplusplus
}
#endif
#endif /* PNP_B200_H */
