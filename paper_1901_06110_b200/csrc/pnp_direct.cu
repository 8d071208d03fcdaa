// Brute-force DSG-NLM: the reference's distances="direct" path
// (denoise.py:291-355, `_dsg_per_pixel`): three per-pixel passes over the
// clipped window with the patch distance summed directly over all P x P patch
// elements -- cost window area x patch area per pixel, no separable filter,
// no running sums.  It exists as the timing baseline of bench-denoiser
// (bench.py:43-72: "fast vs brute-force"), exactly as in the reference.
//
// One thread per pixel; the guide is first mirror-padded (image.py:97-113)
// into a scratch plane so every patch read is a plain load.  The patch
// distance is taken as a sum of squared differences (the reference expands it
// into norms and a cross term, which cancels catastrophically in fp32; the
// value is the same quantity).  Pass 1: g = sum hat k; pass 2: d = rs sum hat
// k rs, max d -> m (int-ordered atomicMax, exact); pass 3: out = rs sum
// hat k rs x / m + (1 - d/m) x.
#include <float.h>
#include <math.h>

#include <string>

#include "pnp_internal.h"
#include "pnp_pdl.cuh"

namespace pnp {

namespace {

constexpr int kDirectMaxP = 63;

struct DirectArgs {
  const float* pad;  // [B][H+2M][W+2M]
  const float* x;    // [B][H][W]
  float* rs;         // [B][H][W]
  float* d;          // [B][H][W]
  float* out;        // [B][H][W]
  unsigned* mbits;   // [B]
  int H, W, R, P, M;
  float c;           // -log2(e) / (2 bw^2)
  float taps[kDirectMaxP];
};

__global__ void direct_pad_kernel(const float* g, float* pad, int H, int W, int M) {
  const int Hp = H + 2 * M, Wp = W + 2 * M, b = blockIdx.y;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < (size_t)Hp * Wp;
       i += (size_t)gridDim.x * blockDim.x) {
    const int py = (int)(i / Wp), px = (int)(i % Wp);
    int y = py - M, xx = px - M;
    if (y < 0) y = -y - 1;
    if (y >= H) y = 2 * H - 1 - y;
    if (xx < 0) xx = -xx - 1;
    if (xx >= W) xx = 2 * W - 1 - xx;
    pad[(size_t)b * Hp * Wp + i] = g[((size_t)b * H + y) * W + xx];
  }
}

// hat_t * k_t(s) for pixel (y, x) and offset (dy, dx): direct P x P sum
__device__ __forceinline__ float direct_weight(const DirectArgs& a, const float* pb, int y, int x,
                                               int dy, int dx) {
  const int Wp = a.W + 2 * a.M, p = (a.P - 1) / 2;
  const float* ps = pb + (size_t)(y + a.M - p) * Wp + (x + a.M - p);
  const float* pr = ps + (size_t)dy * Wp + dx;
  float ssd = 0.f;
  for (int i = 0; i < a.P; ++i) {
    float row = 0.f;
    for (int j = 0; j < a.P; ++j) {
      const float t = __fsub_rn(ps[(size_t)i * Wp + j], pr[(size_t)i * Wp + j]);
      row = __fmaf_rn(a.taps[j], __fmul_rn(t, t), row);
    }
    ssd = __fmaf_rn(a.taps[i], row, ssd);
  }
  const float s1 = a.R + 1.f;
  const float hat = (1.f - fabsf((float)dy) / s1) * (1.f - fabsf((float)dx) / s1);
  return hat * exp2f(a.c * ssd);
}

template <int PASS>
__global__ void direct_pass_kernel(const DirectArgs a) {
  const int b = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.H * a.W) return;
  const int y = i / a.W, x = i % a.W;
  const size_t plane = (size_t)a.H * a.W;
  const float* pb = a.pad + (size_t)b * (a.H + 2 * a.M) * (a.W + 2 * a.M);
  const float* rsb = a.rs + b * plane;
  const float* xb = a.x + b * plane;
  const int r0 = max(0, y - a.R), r1 = min(a.H - 1, y + a.R);
  const int c0 = max(0, x - a.R), c1 = min(a.W - 1, x + a.R);
  float acc = 0.f, mass = 0.f;
  for (int yy = r0; yy <= r1; ++yy)  // raster order over the clipped window
    for (int xx = c0; xx <= c1; ++xx) {
      const float k = direct_weight(a, pb, y, x, yy - y, xx - x);
      if (PASS == 0) {
        acc += k;
      } else {
        const float w = k * rsb[(size_t)yy * a.W + xx];
        mass += w;
        if (PASS == 2) acc = __fmaf_rn(w, xb[(size_t)yy * a.W + xx], acc);
      }
    }
  const size_t o = b * plane + i;
  if (PASS == 0) {
    a.rs[o] = 1.f / sqrtf(fmaxf(acc, FLT_MIN));
  } else if (PASS == 1) {
    const float dv = rsb[i] * mass;
    a.d[o] = dv;
    atomicMax(a.mbits + b, __float_as_uint(dv));  // d > 0: int order = float order
  } else {
    const float m = __uint_as_float(a.mbits[b]);
    const float kx = rsb[i] * acc;
    a.out[o] = kx / m + (1.f - a.d[o] / m) * xb[i];
  }
}

}  // namespace
}  // namespace pnp

using namespace pnp;

extern "C" int pnp_dsg_denoise_direct(pnp_ctx* ctx, const float* x, const float* guide,
                                      float* out, int batch, int H, int W, int R, int P,
                                      const float* taps, double bandwidth) {
  if (!ctx || !x || !out || !taps) return fail(PNP_EINVAL, "null argument");
  if (batch < 1 || H < 1 || W < 1) return fail(PNP_EINVAL, "bad shape");
  if (P < 1 || P % 2 == 0 || P > kDirectMaxP)
    return fail(PNP_EINVAL, "patch_side must be odd and <= " + std::to_string(kDirectMaxP));
  if (R < 1 || !(bandwidth > 0)) return fail(PNP_EINVAL, "bad window radius / bandwidth");
  const int M = R + (P - 1) / 2;
  if (M > (H < W ? H : W)) return fail(PNP_EINVAL, "margin exceeds min image extent");
  if (!guide) guide = x;
  PNP_CUDA(cudaSetDevice(ctx->device));
  const size_t n = (size_t)batch * H * W;
  const size_t npad = (size_t)batch * (H + 2 * M) * (W + 2 * M);
  float *pad = nullptr, *rs = nullptr, *d = nullptr;
  unsigned* mbits = nullptr;
  cudaStream_t st = ctx->stream;
  PNP_CUDA(cudaMallocAsync((void**)&pad, npad * sizeof(float), st));
  PNP_CUDA(cudaMallocAsync((void**)&rs, n * sizeof(float), st));
  PNP_CUDA(cudaMallocAsync((void**)&d, n * sizeof(float), st));
  PNP_CUDA(cudaMallocAsync((void**)&mbits, batch * sizeof(unsigned), st));
  PNP_CUDA(cudaMemsetAsync(mbits, 0, batch * sizeof(unsigned), st));
  direct_pad_kernel<<<dim3(1024, batch), 256, 0, st>>>(guide, pad, H, W, M);
  DirectArgs a{};
  a.pad = pad;
  a.x = x;
  a.rs = rs;
  a.d = d;
  a.out = out;
  a.mbits = mbits;
  a.H = H;
  a.W = W;
  a.R = R;
  a.P = P;
  a.M = M;
  a.c = (float)(-1.0 / (2.0 * log(2.0) * bandwidth * bandwidth));
  for (int i = 0; i < P; ++i) a.taps[i] = taps[i];
  const dim3 grid((unsigned)((H * W + 127) / 128), batch);
  direct_pass_kernel<0><<<grid, 128, 0, st>>>(a);
  direct_pass_kernel<1><<<grid, 128, 0, st>>>(a);
  direct_pass_kernel<2><<<grid, 128, 0, st>>>(a);
  PNP_LAUNCH_CHECK("direct_pass_kernel");
  for (void* p : {(void*)pad, (void*)rs, (void*)d, (void*)mbits}) cudaFreeAsync(p, st);
  return PNP_OK;
}
