// Forward operators and the fused linearized-ADMM elementwise steps.
//
// SR (reference forward.py:98-185): A = decimate_k o blur, blur = correlation
// with a separable normalized kernel under periodic (wrap) or half-sample
// symmetric padding; A^T = blur o zero-fill upsample (exact for symmetric
// kernels).  The residual kernel evaluates the blur only at the kept samples
// and fuses "- y" and the 0.5||.||^2 data-term partials; the adjoint kernel
// visits only the non-zero taps of the upsampled grid.
// QIS (forward.py:312-327): elementwise, evaluated in double.
// ADMM (solver.py:219-228): x-update + projection + x+u + finite flags in one
// pass; u-update + residual/PSNR partial sums in one pass.  All reductions
// are per-block partials summed in a fixed order (deterministic).
#include <math.h>
#include <stdint.h>

#include <vector>

#include "pnp_internal.h"

namespace pnp {

constexpr int kMaxTaps = 63;
struct Taps {
  float ty[kMaxTaps];  // vertical profile (row sums of the 2-D kernel)
  float tx[kMaxTaps];  // horizontal profile (column sums)
};

__device__ __forceinline__ int map_index(int i, int n, int symmetric) {
  if (symmetric) {
    if (i < 0) i = -i - 1;
    if (i >= n) i = 2 * n - 1 - i;
    return i;
  }
  i %= n;
  return i < 0 ? i + n : i;
}

// Deterministic block sum of doubles -> partial[blockIdx.y][blockIdx.x].
__device__ __forceinline__ void block_sum_store(double v, double* partial) {
  __shared__ double red[32];
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k];
    partial[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
  }
}

// out[b*stride + k] = scale * sum_j partial[b][j][k]  (fixed order)
__global__ void reduce_partials_kernel(const double* partial, int nblk, int nvec, double scale,
                                       double* out, int stride) {
  const int b = blockIdx.x;
  const int k = threadIdx.x;
  if (k >= nvec) return;
  double s = 0.0;
  for (int j = 0; j < nblk; ++j) s += partial[((size_t)b * nblk + j) * nvec + k];
  out[(size_t)b * stride + k] = scale * s;
}

// r = A x - y (or A x when y == null) on the low-res grid; optional data partials.
__global__ void __launch_bounds__(256)
sr_residual_kernel(const float* __restrict__ x, const float* __restrict__ y, float* __restrict__ r,
                   int H, int W, int k, int rad, int sym, const Taps taps, double* partial) {
  const int h = H / k, w = W / k;
  const int b = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double sq = 0.0;
  if (i < h * w) {
    const int oy = i / w, ox = i - oy * w;
    const float* xb = x + (size_t)b * H * W;
    float acc = 0.f;
    for (int a = -rad; a <= rad; ++a) {
      const float* row = xb + (size_t)map_index(k * oy + a, H, sym) * W;
      float s = 0.f;
      for (int c = -rad; c <= rad; ++c) s = fmaf(taps.tx[c + rad], row[map_index(k * ox + c, W, sym)], s);
      acc = fmaf(taps.ty[a + rad], s, acc);
    }
    if (y) acc -= y[(size_t)b * h * w + i];
    r[(size_t)b * h * w + i] = acc;
    sq = (double)acc * (double)acc;
  }
  if (partial) block_sum_store(sq, partial);
}

// x_out = A^T r = blur(upsample_k(r)) on the high-res grid.
__global__ void __launch_bounds__(256)
sr_adjoint_kernel(const float* __restrict__ r, float* __restrict__ out, int H, int W, int k,
                  int rad, int sym, const Taps taps) {
  const int h = H / k, w = W / k;
  const int b = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= H * W) return;
  const int py = i / W, px = i - py * W;
  const float* rb = r + (size_t)b * h * w;
  float acc = 0.f;
  for (int a = -rad; a <= rad; ++a) {
    const int uy = map_index(py + a, H, sym);
    if (uy % k) continue;
    const float* row = rb + (size_t)(uy / k) * w;
    float s = 0.f;
    for (int c = -rad; c <= rad; ++c) {
      const int ux = map_index(px + c, W, sym);
      if (ux % k) continue;
      s = fmaf(taps.tx[c + rad], row[ux / k], s);
    }
    acc = fmaf(taps.ty[a + rad], s, acc);
  }
  out[(size_t)b * H * W + i] = acc;
}

__global__ void __launch_bounds__(256)
qis_grad_kernel(const float* __restrict__ x, const float* __restrict__ ones,
                const float* __restrict__ zeros, float* __restrict__ grad, size_t n,
                double gk, double floor_, double* partial) {
  const int b = blockIdx.y;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  double term = 0.0;
  if (i < n) {
    const size_t o = (size_t)b * n + i;
    const double z = gk * fmax((double)x[o], floor_);
    const double k1 = ones[o], k0 = zeros[o];
    if (grad) grad[o] = (float)(gk * (k0 - k1 / expm1(z)));
    if (partial) term = k0 * z - k1 * log(-expm1(-z));
  }
  if (partial) block_sum_store(term, partial);
}

__global__ void __launch_bounds__(256)
admm_xupdate_kernel(float* __restrict__ x, const float* __restrict__ v, const float* __restrict__ u,
                    const float* __restrict__ grad, float* __restrict__ z, size_t n, double mu,
                    double alpha, double rho, float lo, float hi, int* flags) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  int f = 0;
  if (i < n) {
    const double xv = (double)x[i];
    const double uv = (double)u[i];
    const double xn = mu * (alpha * xv + rho * ((double)v[i] - uv) - (double)grad[i]);
    float xf = (float)xn;
    if (!isfinite(xf)) f |= 1;
    xf = fminf(fmaxf(xf, lo), hi);
    const float zf = (float)((double)xf + uv);
    if (!isfinite(zf)) f |= 2;
    x[i] = xf;
    z[i] = zf;
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if (f && (threadIdx.x & 31) == 0) atomicOr(flags, f);
}

// u += x - v ; partials (sum (x-v)^2, sum (rho (v - v_prev))^2, sum (gt - v)^2)
__global__ void __launch_bounds__(256)
admm_uupdate_kernel(float* __restrict__ u, const float* __restrict__ x, const float* __restrict__ v,
                    const float* __restrict__ vp, const float* __restrict__ gt, size_t n,
                    double rho, double* partial, int* flags) {
  const int b = blockIdx.y;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  int f = 0;
  if (i < n) {
    const size_t o = (size_t)b * n + i;
    const double xv = x[o], vv = v[o];
    const float un = (float)((double)u[o] + (xv - vv));
    if (!isfinite(vv) || !isfinite(un)) f = 4;
    u[o] = un;
    s0 = (xv - vv) * (xv - vv);
    const double dv = rho * (vv - (vp ? (double)vp[o] : 0.0));
    s1 = dv * dv;
    if (gt) {
      const double e = (double)gt[o] - vv;
      s2 = e * e;
    }
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if (f && (threadIdx.x & 31) == 0) atomicOr(flags, f);
  __shared__ double red[3][32];
  for (int off = 16; off; off >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, off);
    s1 += __shfl_xor_sync(0xffffffffu, s1, off);
    s2 += __shfl_xor_sync(0xffffffffu, s2, off);
  }
  const int wid = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][wid] = s0;
    red[1][wid] = s1;
    red[2][wid] = s2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a0 = 0, a1 = 0, a2 = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      a0 += red[0][k];
      a1 += red[1][k];
      a2 += red[2][k];
    }
    double* pp = partial + ((size_t)b * gridDim.x + blockIdx.x) * 3;
    pp[0] = a0;
    pp[1] = a1;
    pp[2] = a2;
  }
}

__global__ void project_kernel(const float* x, float* y, size_t n, float lo, float hi) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = fminf(fmaxf(x[i], lo), hi);
}

// ------------------------------------------------------------------ host ---

static int sr_check(int batch, int H, int W, const float* taps, int radius, int factor,
                    int boundary, Taps& t) {
  if (batch < 1 || H < 1 || W < 1) return fail(PNP_EINVAL, "bad shape");
  if (factor < 1) return fail(PNP_EINVAL, "factor must be >= 1");
  if (H % factor || W % factor) return fail(PNP_EINVAL, "dimensions not divisible by factor");
  if (radius < 0 || 2 * radius + 1 > kMaxTaps) return fail(PNP_EINVAL, "bad blur radius");
  if (radius > (H < W ? H : W)) return fail(PNP_EINVAL, "kernel radius exceeds image extent");
  if (boundary != 0 && boundary != 1) return fail(PNP_EINVAL, "boundary must be 0 or 1");
  if (!taps) return fail(PNP_EINVAL, "taps null");
  for (int i = 0; i < 2 * radius + 1; ++i) {
    t.ty[i] = taps[i];
    t.tx[i] = taps[2 * radius + 1 + i];
  }
  return PNP_OK;
}

static int ensure_partials(pnp_ctx* ctx, size_t doubles) {
  return ctx->stats.ensure(doubles * sizeof(double));
}

}  // namespace pnp

using namespace pnp;

extern "C" {

int pnp_sr_apply(pnp_ctx* ctx, const float* x, float* y, int batch, int H, int W,
                 const float* taps, int radius, int factor, int boundary) {
  if (!ctx || !x || !y) return fail(PNP_EINVAL, "null argument");
  Taps t;
  int rc = sr_check(batch, H, W, taps, radius, factor, boundary, t);
  if (rc) return rc;
  const int nl = (H / factor) * (W / factor);
  dim3 grid((nl + 255) / 256, batch);
  {
    ProfScope prof_(ctx, PROF_FORWARD);
    sr_residual_kernel<<<grid, 256, 0, ctx->stream>>>(x, nullptr, y, H, W, factor, radius, boundary,
                                                      t, nullptr);
  }
  PNP_LAUNCH_CHECK("sr_residual_kernel");
  return PNP_OK;
}

int pnp_sr_adjoint(pnp_ctx* ctx, const float* y, float* x, int batch, int H, int W,
                   const float* taps, int radius, int factor, int boundary) {
  if (!ctx || !x || !y) return fail(PNP_EINVAL, "null argument");
  Taps t;
  int rc = sr_check(batch, H, W, taps, radius, factor, boundary, t);
  if (rc) return rc;
  dim3 grid((H * W + 255) / 256, batch);
  {
    ProfScope prof_(ctx, PROF_FORWARD);
    sr_adjoint_kernel<<<grid, 256, 0, ctx->stream>>>(y, x, H, W, factor, radius, boundary, t);
  }
  PNP_LAUNCH_CHECK("sr_adjoint_kernel");
  return PNP_OK;
}

int pnp_sr_grad(pnp_ctx* ctx, const float* x, const float* yobs, float* grad, int batch, int H,
                int W, const float* taps, int radius, int factor, int boundary, double* data_out) {
  if (!ctx || !x || !yobs || !grad) return fail(PNP_EINVAL, "null argument");
  Taps t;
  int rc = sr_check(batch, H, W, taps, radius, factor, boundary, t);
  if (rc) return rc;
  const int nl = (H / factor) * (W / factor);
  const int nblk = (nl + 255) / 256;
  if ((rc = ctx->kx.ensure((size_t)batch * nl * sizeof(float)))) return rc;
  if (data_out && (rc = ensure_partials(ctx, (size_t)batch * nblk))) return rc;
  float* r = ctx->kx.as<float>();
  double* part = data_out ? ctx->stats.as<double>() : nullptr;
  {
    ProfScope prof_(ctx, PROF_FORWARD);
    sr_residual_kernel<<<dim3(nblk, batch), 256, 0, ctx->stream>>>(x, yobs, r, H, W, factor, radius,
                                                                   boundary, t, part);
  }
  PNP_LAUNCH_CHECK("sr_residual_kernel");
  if (data_out) {
    {
      ProfScope prof_(ctx, PROF_ADMM);
      reduce_partials_kernel<<<batch, 32, 0, ctx->stream>>>(part, nblk, 1, 0.5, data_out, 1);
    }
    PNP_LAUNCH_CHECK("reduce_partials_kernel");
  }
  {
    ProfScope prof_(ctx, PROF_FORWARD);
    sr_adjoint_kernel<<<dim3((H * W + 255) / 256, batch), 256, 0, ctx->stream>>>(
        r, grad, H, W, factor, radius, boundary, t);
  }
  PNP_LAUNCH_CHECK("sr_adjoint_kernel");
  return PNP_OK;
}

int pnp_qis_grad(pnp_ctx* ctx, const float* x, const float* ones, const float* zeros, float* grad,
                 int batch, int n, double gain_over_K, double floor_, double* data_out) {
  if (!ctx || !x || !ones || !zeros || (!grad && !data_out))
    return fail(PNP_EINVAL, "null argument");
  if (batch < 1 || n < 1) return fail(PNP_EINVAL, "bad shape");
  const int nblk = (n + 255) / 256;
  double* part = nullptr;
  if (data_out) {
    int rc = ensure_partials(ctx, (size_t)batch * nblk);
    if (rc) return rc;
    part = ctx->stats.as<double>();
  }
  {
    ProfScope prof_(ctx, PROF_FORWARD);
    qis_grad_kernel<<<dim3(nblk, batch), 256, 0, ctx->stream>>>(x, ones, zeros, grad, (size_t)n,
                                                                gain_over_K, floor_, part);
  }
  PNP_LAUNCH_CHECK("qis_grad_kernel");
  if (data_out) {
    {
      ProfScope prof_(ctx, PROF_ADMM);
      reduce_partials_kernel<<<batch, 32, 0, ctx->stream>>>(part, nblk, 1, 1.0, data_out, 1);
    }
    PNP_LAUNCH_CHECK("reduce_partials_kernel");
  }
  return PNP_OK;
}

int pnp_qis_data(pnp_ctx* ctx, const float* x, const float* ones, const float* zeros, int batch,
                 int n, double gain_over_K, double floor_, double* data_out) {
  if (!ctx || !x || !ones || !zeros || !data_out) return fail(PNP_EINVAL, "null argument");
  if (batch < 1 || n < 1) return fail(PNP_EINVAL, "bad shape");
  const int nblk = (n + 255) / 256;
  int rc = ensure_partials(ctx, (size_t)batch * nblk);
  if (rc) return rc;
  double* part = ctx->stats.as<double>();
  {
    ProfScope prof_(ctx, PROF_FORWARD);
    qis_grad_kernel<<<dim3(nblk, batch), 256, 0, ctx->stream>>>(x, ones, zeros, nullptr, (size_t)n,
                                                                gain_over_K, floor_, part);
  }
  PNP_LAUNCH_CHECK("qis_grad_kernel");
  reduce_partials_kernel<<<batch, 32, 0, ctx->stream>>>(part, nblk, 1, 1.0, data_out, 1);
  PNP_LAUNCH_CHECK("reduce_partials_kernel");
  return PNP_OK;
}

int pnp_admm_xupdate(pnp_ctx* ctx, float* x, const float* v, const float* u, const float* grad,
                     float* z, int64_t n, double mu, double alpha, double rho, double lo, double hi,
                     int* flags) {
  if (!ctx || !x || !v || !u || !grad || !z || !flags) return fail(PNP_EINVAL, "null argument");
  const float flo = isinf(lo) ? -INFINITY : (float)lo;
  const float fhi = isinf(hi) ? INFINITY : (float)hi;
  {
    ProfScope prof_(ctx, PROF_ADMM);
    admm_xupdate_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(
        x, v, u, grad, z, (size_t)n, mu, alpha, rho, flo, fhi, flags);
  }
  PNP_LAUNCH_CHECK("admm_xupdate_kernel");
  return PNP_OK;
}

int pnp_admm_uupdate(pnp_ctx* ctx, float* u, const float* x, const float* v, const float* v_prev,
                     const float* gt, int batch, int64_t n, double rho, double* stats,
                     int* flags) {
  if (!ctx || !u || !x || !v || !stats || !flags) return fail(PNP_EINVAL, "null argument");
  const int nblk = (int)((n + 255) / 256);
  int rc = ensure_partials(ctx, (size_t)batch * nblk * 3);
  if (rc) return rc;
  double* part = ctx->stats.as<double>();
  {
    ProfScope prof_(ctx, PROF_ADMM);
    admm_uupdate_kernel<<<dim3(nblk, batch), 256, 0, ctx->stream>>>(u, x, v, v_prev, gt, (size_t)n,
                                                                    rho, part, flags);
  }
  PNP_LAUNCH_CHECK("admm_uupdate_kernel");
  reduce_partials_kernel<<<batch, 32, 0, ctx->stream>>>(part, nblk, 3, 1.0, stats, 4);
  PNP_LAUNCH_CHECK("reduce_partials_kernel");
  return PNP_OK;
}

int pnp_project(pnp_ctx* ctx, const float* x, float* y, int64_t n, double lo, double hi) {
  if (!ctx || !x || !y) return fail(PNP_EINVAL, "null argument");
  const float flo = isinf(lo) ? -INFINITY : (float)lo;
  const float fhi = isinf(hi) ? INFINITY : (float)hi;
  {
    ProfScope prof_(ctx, PROF_ADMM);
    project_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(x, y, (size_t)n, flo, fhi);
  }
  PNP_LAUNCH_CHECK("project_kernel");
  return PNP_OK;
}

// Knuth product-method Poisson jots, bit-exact with forward.py:263-298 given
// the same stop thresholds (computed by the caller with numpy's exp).
int pnp_qis_simulate_host(const double* stop, int64_t n, int K, uint64_t seed, double* ones) {
  if (!stop || !ones || n < 0 || K < 1) return fail(PNP_EINVAL, "bad arguments");
  const uint64_t GOLDEN = 0x9E3779B97F4A7C15ull;
  uint64_t state = seed;
  auto next_uniform = [&]() {
    state += GOLDEN;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    return (double)(z >> 11) * 0x1.0p-53;
  };
  for (int64_t i = 0; i < n; ++i) {
    const double thr = stop[i];
    int fired = 0;
    for (int j = 0; j < K; ++j) {
      int count = 0;
      double prod = 1.0;
      for (;;) {
        prod *= next_uniform();
        if (prod <= thr) break;
        ++count;
      }
      if (count >= 1) ++fired;
    }
    ones[i] = (double)fired;
  }
  return PNP_OK;
}

}  // extern "C"
