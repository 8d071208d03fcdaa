// Float64 patch-distance primitives on the device: the public helpers of the
// reference's distance engine (pnprestore/image.py:97-143 pad_symmetric /
// integral_image, denoise.py:70-88 nlm_kernel, 106-174 _DistanceEngine /
// patch_distance_map).  They are not on the fp32 sweep path (the sweep kernel
// reflects indices at load and never materializes padded guides, SATs or
// per-offset maps); they exist so callers of those reference functions keep
// working, computed on the GPU in the reference's precision and, where the
// reference's order is sequential, in its exact summation order:
//   * pad_symmetric: a copy (exact);
//   * integral_image: column cumsums then row cumsums, each sequential like
//     numpy's cumsum -> bitwise equal;
//   * patch distances: the "direct" shifted-add order (py outer, px inner) of
//     _DistanceEngine.map, explicit _rn intrinsics so nothing is contracted
//     into FMAs -> bitwise equal to method="direct".
#include <cuda_runtime.h>
#include <stdint.h>

#include "pnp_internal.h"

namespace pnp {
namespace {

// half-sample symmetric index (np.pad mode="symmetric", single reflection)
__device__ __forceinline__ int reflect1(int i, int n) {
  if (i < 0) i = -i - 1;
  if (i >= n) i = 2 * n - 1 - i;
  return i;
}

__global__ void pad_symmetric_kernel(const double* __restrict__ img, int H, int W, int M,
                                     double* __restrict__ out) {
  const int Wo = W + 2 * M, Ho = H + 2 * M;
  const size_t n = (size_t)Ho * Wo;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / Wo), x = (int)(i % Wo);
    out[i] = img[(size_t)reflect1(y - M, H) * W + reflect1(x - M, W)];
  }
}

// out is (H+1) x (W+1) with a zero leading row / column.  Pass 1: thread per
// column, running sum down the rows (numpy cumsum axis 0); pass 2: thread per
// row, running sum along the columns (axis 1) in place.
__global__ void integral_cols_kernel(const double* __restrict__ img, int H, int W,
                                     double* __restrict__ out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int Wo = W + 1;
  if (x > W) return;
  out[x] = 0.0;
  if (x == 0) {
    for (int y = 1; y <= H; ++y) out[(size_t)y * Wo] = 0.0;
    return;
  }
  double s = 0.0;
  for (int y = 0; y < H; ++y) {
    s = __dadd_rn(s, img[(size_t)y * W + (x - 1)]);
    out[(size_t)(y + 1) * Wo + x] = s;
  }
}

__global__ void integral_rows_kernel(int H, int W, double* __restrict__ out) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (y > H) return;
  double* row = out + (size_t)y * (W + 1);
  double s = 0.0;
  for (int x = 1; x <= W; ++x) {
    s = __dadd_rn(s, row[x]);
    row[x] = s;
  }
}

// SSD between the P x P patches at s and s + t (reflected guide), in the
// shifted-add order of _DistanceEngine.map(method="direct")
__device__ __forceinline__ double patch_ssd(const double* __restrict__ g, int H, int W, int P,
                                            int sy, int sx, int dy, int dx) {
  const int h = (P - 1) / 2;
  double acc = 0.0;
  for (int py = 0; py < P; ++py) {
    const int ya = reflect1(sy + py - h, H), yb = reflect1(sy + py - h + dy, H);
    for (int px = 0; px < P; ++px) {
      const double d = __dsub_rn(g[(size_t)ya * W + reflect1(sx + px - h, W)],
                                 g[(size_t)yb * W + reflect1(sx + px - h + dx, W)]);
      acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
  }
  return acc;
}

__global__ void patch_distance_kernel(const double* __restrict__ g, int H, int W, int P, int dy,
                                      int dx, double* __restrict__ out) {
  const size_t n = (size_t)H * W;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    out[i] = patch_ssd(g, H, W, P, (int)(i / W), (int)(i % W), dy, dx);
}

__global__ void patch_ssd_pairs_kernel(const double* __restrict__ g, int H, int W, int P,
                                       const int* __restrict__ pairs, int n,
                                       double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int sy = pairs[4 * i], sx = pairs[4 * i + 1], ry = pairs[4 * i + 2], rx = pairs[4 * i + 3];
  out[i] = patch_ssd(g, H, W, P, sy, sx, ry - sy, rx - sx);
}

// ---- dense W (build_dense_weights, denoise.py:389-418), test-scale ----
// W[s][s+t] = hat_t * exp(-inv * ssd(s, t)) for every in-image pair of the
// clipped window; the scaling steps follow the reference's matrix transforms.
__global__ void dense_fill_kernel(const double* __restrict__ g, int H, int W, int P, int R,
                                  double inv, double* __restrict__ Wm) {
  const int n = H * W, side = 2 * R + 1;
  const size_t total = (size_t)n * side * side;
  const double scale = R + 1;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int s = (int)(i / ((size_t)side * side)), o = (int)(i % ((size_t)side * side));
    const int dy = o / side - R, dx = o % side - R;
    const int sy = s / W, sx = s % W, ry = sy + dy, rx = sx + dx;
    if (ry < 0 || ry >= H || rx < 0 || rx >= W) continue;
    const double k = exp(__dmul_rn(-inv, patch_ssd(g, H, W, P, sy, sx, dy, dx)));
    const double hat = __dmul_rn(1.0 - fabs((double)dy) / scale, 1.0 - fabs((double)dx) / scale);
    Wm[(size_t)s * n + (size_t)ry * W + rx] = __dmul_rn(hat, k);
  }
}

// per-row sums (one warp per row, fixed tree) and per-column sums (thread per
// column, rows in order): deterministic
__global__ void dense_rowsum_kernel(const double* __restrict__ Wm, int n, double* __restrict__ out) {
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
  if (row >= n) return;
  double s = 0.0;
  for (int j = lane; j < n; j += 32) s = __dadd_rn(s, Wm[(size_t)row * n + j]);
  for (int off = 16; off; off >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
  if (lane == 0) out[row] = s;
}

__global__ void dense_colsum_kernel(const double* __restrict__ Wm, int n, double* __restrict__ out) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= n) return;
  double s = 0.0;
  for (int i = 0; i < n; ++i) s = __dadd_rn(s, Wm[(size_t)i * n + col]);
  out[col] = s;
}

// W[i][j] = (W[i][j] * (1 / sqrt(row_i))) * (1 / sqrt(col_j))
__global__ void dense_scale_kernel(double* __restrict__ Wm, int n, const double* __restrict__ row,
                                   const double* __restrict__ col) {
  const size_t total = (size_t)n * n;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / n), c = (int)(i % n);
    Wm[i] = __dmul_rn(__dmul_rn(Wm[i], 1.0 / sqrt(row[r])), 1.0 / sqrt(col[c]));
  }
}

// m = max_i rowsum_i (single CTA), then W /= m
__global__ void dense_max_kernel(const double* __restrict__ v, int n, double* __restrict__ m) {
  __shared__ double red[32];
  double x = -1.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) x = fmax(x, v[i]);
  for (int off = 16; off; off >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, red[w]);
    *m = r;
  }
}

__global__ void dense_div_kernel(double* __restrict__ Wm, int n, const double* __restrict__ m) {
  const size_t total = (size_t)n * n;
  const double mm = *m;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x)
    Wm[i] = __ddiv_rn(Wm[i], mm);
}

// W[i][i] += 1 - rowsum_i
__global__ void dense_diag_kernel(double* __restrict__ Wm, int n, const double* __restrict__ row) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) Wm[(size_t)i * n + i] = __dadd_rn(Wm[(size_t)i * n + i], 1.0 - row[i]);
}

int grid_for(size_t n, int sms) {
  const size_t b = (n + 255) / 256;
  const size_t cap = (size_t)sms * 16;
  return (int)(b < cap ? (b > 0 ? b : 1) : cap);
}

}  // namespace
}  // namespace pnp

using namespace pnp;

extern "C" {

int pnp_pad_symmetric_f64(pnp_ctx* ctx, const double* img, int H, int W, int margin, double* out) {
  if (!ctx || !img || !out) return fail(PNP_EINVAL, "null argument");
  if (H < 1 || W < 1) return fail(PNP_EINVAL, "image must be at least 1x1");
  if (margin < 0) return fail(PNP_EINVAL, "margin must be >= 0, got " + std::to_string(margin));
  if (margin > (H < W ? H : W))
    return fail(PNP_EINVAL, "margin " + std::to_string(margin) + " exceeds min image extent " +
                                std::to_string(H < W ? H : W));
  const size_t n = (size_t)(H + 2 * margin) * (W + 2 * margin);
  pad_symmetric_kernel<<<grid_for(n, ctx->sms), 256, 0, ctx->stream>>>(img, H, W, margin, out);
  PNP_LAUNCH_CHECK("pad_symmetric_kernel");
  return PNP_OK;
}

int pnp_integral_image_f64(pnp_ctx* ctx, const double* img, int H, int W, double* out) {
  if (!ctx || !img || !out) return fail(PNP_EINVAL, "null argument");
  if (H < 1 || W < 1) return fail(PNP_EINVAL, "image must be at least 1x1");
  integral_cols_kernel<<<(W + 1 + 127) / 128, 128, 0, ctx->stream>>>(img, H, W, out);
  PNP_LAUNCH_CHECK("integral_cols_kernel");
  integral_rows_kernel<<<(H + 127) / 128, 128, 0, ctx->stream>>>(H, W, out);
  PNP_LAUNCH_CHECK("integral_rows_kernel");
  return PNP_OK;
}

int pnp_patch_distance_map_f64(pnp_ctx* ctx, const double* guide, int H, int W, int P, int R,
                               int dy, int dx, double* out) {
  if (!ctx || !guide || !out) return fail(PNP_EINVAL, "null argument");
  if (H < 1 || W < 1) return fail(PNP_EINVAL, "image must be at least 1x1");
  if (P < 1 || P % 2 == 0) return fail(PNP_EINVAL, "patch_side must be odd and >= 1");
  if (R < 1) return fail(PNP_EINVAL, "window_radius must be >= 1");
  if ((dy < 0 ? -dy : dy) > R || (dx < 0 ? -dx : dx) > R)
    return fail(PNP_EINVAL, "offset outside window radius " + std::to_string(R));
  const int margin = R + (P - 1) / 2;
  if (margin > (H < W ? H : W))
    return fail(PNP_EINVAL, "margin " + std::to_string(margin) + " exceeds min image extent " +
                                std::to_string(H < W ? H : W));
  const size_t n = (size_t)H * W;
  patch_distance_kernel<<<grid_for(n, ctx->sms), 256, 0, ctx->stream>>>(guide, H, W, P, dy, dx,
                                                                        out);
  PNP_LAUNCH_CHECK("patch_distance_kernel");
  return PNP_OK;
}

int pnp_dense_weights_f64(pnp_ctx* ctx, const double* guide, int H, int W, int P, int R,
                          double bandwidth, double* out, double* scratch) {
  if (!ctx || !guide || !out || !scratch) return fail(PNP_EINVAL, "null argument");
  if (H < 1 || W < 1) return fail(PNP_EINVAL, "image must be at least 1x1");
  if (P < 1 || P % 2 == 0 || R < 1 || !(bandwidth > 0)) return fail(PNP_EINVAL, "bad params");
  const int margin = R + (P - 1) / 2;
  if (margin > (H < W ? H : W))
    return fail(PNP_EINVAL, "margin " + std::to_string(margin) + " exceeds min image extent " +
                                std::to_string(H < W ? H : W));
  const int n = H * W;
  const size_t nn = (size_t)n * n;
  const double inv = 1.0 / (2.0 * P * P * bandwidth * bandwidth);
  double* row = scratch;
  double* col = scratch + n;
  double* m = scratch + 2 * (size_t)n;
  const int gb = grid_for(nn, ctx->sms);
  PNP_CUDA(cudaMemsetAsync(out, 0, nn * sizeof(double), ctx->stream));
  const size_t pairs = (size_t)n * (2 * R + 1) * (2 * R + 1);
  dense_fill_kernel<<<grid_for(pairs, ctx->sms), 256, 0, ctx->stream>>>(guide, H, W, P, R, inv, out);
  dense_rowsum_kernel<<<(n + 7) / 8, 256, 0, ctx->stream>>>(out, n, row);
  dense_colsum_kernel<<<(n + 127) / 128, 128, 0, ctx->stream>>>(out, n, col);
  dense_scale_kernel<<<gb, 256, 0, ctx->stream>>>(out, n, row, col);
  dense_rowsum_kernel<<<(n + 7) / 8, 256, 0, ctx->stream>>>(out, n, row);
  dense_max_kernel<<<1, 1024, 0, ctx->stream>>>(row, n, m);
  dense_div_kernel<<<gb, 256, 0, ctx->stream>>>(out, n, m);
  dense_rowsum_kernel<<<(n + 7) / 8, 256, 0, ctx->stream>>>(out, n, row);
  dense_diag_kernel<<<(n + 127) / 128, 128, 0, ctx->stream>>>(out, n, row);
  PNP_LAUNCH_CHECK("dense_weights kernels");
  return PNP_OK;
}

int pnp_patch_ssd_pairs_f64(pnp_ctx* ctx, const double* guide, int H, int W, int P,
                            const int* pairs, int n, double* out) {
  if (!ctx || !guide || (n > 0 && (!pairs || !out))) return fail(PNP_EINVAL, "null argument");
  if (H < 1 || W < 1 || n < 0) return fail(PNP_EINVAL, "bad shape");
  if (P < 1 || P % 2 == 0) return fail(PNP_EINVAL, "patch_side must be odd and >= 1");
  if ((P - 1) / 2 > (H < W ? H : W))
    return fail(PNP_EINVAL, "patch half-width exceeds min image extent");
  if (n == 0) return PNP_OK;
  patch_ssd_pairs_kernel<<<(n + 127) / 128, 128, 0, ctx->stream>>>(guide, H, W, P, pairs, n, out);
  PNP_LAUNCH_CHECK("patch_ssd_pairs_kernel");
  return PNP_OK;
}

}  // extern "C"
