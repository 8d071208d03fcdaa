// Host orchestration of the DSG-NLM pipeline + fixup/finalize kernels.
//
//   adaptive  (dsg_nlm_denoise, reference denoise.py:272-288)
//     sweep A  [C=1, y = mask]        -> partial -> fixup_rs   -> rs = g^-1/2
//     sweep B  [C=2, y = rs*x, rs]    -> partial -> fixup_kxd  -> Kx, d, max d
//     finalize                        -> out = Kx/m + (1 - d/m) x
//   freeze    (FrozenGuide.__init__, denoise.py:367-373): sweep A, fixup_rs,
//     sweep B [C=1, y = rs] -> fixup_d -> d, m
//   apply     (FrozenGuide.apply, denoise.py:375-381): sweep [C=1, y = rs*x]
//     -> fixup_apply (finalize fused).
// The Kx and d channels see exactly the same instruction sequence in every
// variant, so apply() is bit-identical to the adaptive call.
#include <float.h>
#include <math.h>

#include <cstring>
#include <string>
#include <vector>

#include "dsg_sweep.cuh"
#include "sweep_launch.cuh"
#include "pnp_internal.h"

namespace pnp {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
  return PNP_ECUDA;
}

int DevBuf::ensure(size_t want) {
  if (want <= bytes && ptr) return PNP_OK;
  release();
  size_t sz = want < 256 ? 256 : want;
  cudaError_t e = cudaMalloc(&ptr, sz);
  if (e != cudaSuccess) {
    ptr = nullptr;
    bytes = 0;
    return cuda_fail(e, "cudaMalloc(scratch)");
  }
  bytes = sz;
  return PNP_OK;
}
void DevBuf::release() {
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  bytes = 0;
}

// ---------------------------------------------------------------- kernels --

enum FixMode { FIX_RS = 0, FIX_KXD = 1, FIX_D = 2, FIX_APPLY = 3, FIX_NLM = 4 };

struct FixIO {
  float* rs;           // in (KXD, D, APPLY) / out (RS)
  float* kx;           // out (KXD)
  float* d;            // out (KXD, D) / in (APPLY)
  unsigned* mbits;     // per-image max bits (KXD, D)
  const float* inv_m;  // per image (APPLY)
  const float* x;      // (APPLY)
  float* out;          // (APPLY, NLM)
};

__device__ __forceinline__ float dsg_finish(float kx, float d, float inv_m, float x) {
  const float w = __fmul_rn(kx, inv_m);
  const float mass = __fmul_rn(d, inv_m);
  return __fmaf_rn(__fsub_rn(1.f, mass), x, w);
}

template <int MODE>
__global__ void __launch_bounds__(256) dsg_fixup_kernel(const FixGeo f, const FixIO io) {
  const int b = blockIdx.y;
  const size_t plane = (size_t)f.H * f.W;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  float dval = 0.f;
  if (i < plane) {
    const int y = (int)(i / f.W), x = (int)(i - (size_t)y * f.W);
    const size_t o = (size_t)b * plane + i;
    const float s0 = gather_partial(f, b, 0, y, x);
    if (MODE == FIX_RS) {
      io.rs[o] = __fdiv_rn(1.f, __fsqrt_rn(fmaxf(s0, FLT_MIN)));
    } else if (MODE == FIX_KXD) {
      const float s1 = gather_partial(f, b, 1, y, x);
      const float r = io.rs[o];
      io.kx[o] = __fmul_rn(r, s0);
      dval = __fmul_rn(r, s1);
      io.d[o] = dval;
    } else if (MODE == FIX_D) {
      dval = __fmul_rn(io.rs[o], s0);
      io.d[o] = dval;
    } else if (MODE == FIX_APPLY) {
      const float kx = __fmul_rn(io.rs[o], s0);
      io.out[o] = dsg_finish(kx, io.d[o], io.inv_m[b], io.x[o]);
    } else {  // FIX_NLM: num / den
      const float s1 = gather_partial(f, b, 1, y, x);
      io.out[o] = __fdiv_rn(s0, s1);
    }
  }
  if (MODE == FIX_KXD || MODE == FIX_D) {
    // d > 0, so the int ordering of the bits is the float ordering; max is
    // exact and order-free -> deterministic.
    __shared__ float red[8];
    float v = dval;
    for (int off = 16; off; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      float m = red[0];
      for (int k = 1; k < (int)(blockDim.x >> 5); ++k) m = fmaxf(m, red[k]);
      atomicMax(io.mbits + b, __float_as_uint(m));
    }
  }
}

__global__ void dsg_finalize_kernel(const float* kx, const float* d, const unsigned* mbits,
                                    const float* x, float* out, float* alpha_out, size_t plane) {
  const int b = blockIdx.y;
  const float m = __uint_as_float(mbits[b]);
  const float inv_m = __frcp_rn(m);
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (alpha_out && i == 0) alpha_out[b] = m;
  if (i < plane) {
    const size_t o = (size_t)b * plane + i;
    out[o] = dsg_finish(kx[o], d[o], inv_m, x[o]);
  }
}

__global__ void dsg_alpha_kernel(const unsigned* mbits, float* mv, int B) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) {
    const float m = __uint_as_float(mbits[b]);
    mv[b] = m;
    mv[B + b] = __frcp_rn(m);
  }
}

// ------------------------------------------------------------------ host ---

struct Plan {
  int B, H, W, R, P, TH, tiles_x, tiles_y, ntiles, nchunks, NG;
  const Chunk* chunks;  // hat-tapered table (DSG)
  const Chunk* chunks_nohat;  // same offsets, L = 0 (plain NLM)
  const int* grp;
};

// Half-window offsets grouped in chunks of KY consecutive dy sharing dx.
static void build_chunks(int R, bool hat, std::vector<Chunk>& out) {
  out.clear();
  for (int dx = -R; dx <= R; ++dx) {
    const int dy_first = dx > 0 ? 0 : 1;
    for (int dy0 = dy_first; dy0 <= R; dy0 += kKY) {
      Chunk ch;
      memset(&ch, 0, sizeof(ch));
      ch.dx = dx;
      ch.dy0 = dy0;
      ch.kc = (R - dy0 + 1) < kKY ? (R - dy0 + 1) : kKY;
      for (int k = 0; k < kKY && k < 4; ++k) {
        // log2 of the separable hat (denoise.py:199-201), in double, rounded once
        const int dy = dy0 + k;
        const double s = R + 1.0;
        const double hy = 1.0 - fabs((double)dy) / s, hx = 1.0 - fabs((double)dx) / s;
        ch.L[k] = (hat && k < ch.kc) ? (float)(log2(hy) + log2(hx)) : 0.f;
      }
      out.push_back(ch);
    }
  }
}

static int pick_groups(int ntiles, int nchunks) {
  // Offset-group split so small images still fill 148 SMs (~8 CTAs each).
  // Depends only on the image geometry -> identical for every call variant.
  const int target = 148 * 8;
  int ng = (target + ntiles - 1) / ntiles;
  if (ng > nchunks) ng = nchunks;
  if (ng > 64) ng = 64;
  return ng < 1 ? 1 : ng;
}

static int check_geometry(int B, int H, int W, int R, int P, double bw) {
  if (B < 1) return fail(PNP_EINVAL, "batch must be >= 1");
  if (H < 1 || W < 1) return fail(PNP_EINVAL, "image must be at least 1x1");
  if (P < 1 || P % 2 == 0)
    return fail(PNP_EINVAL, "patch_side must be odd and >= 1, got " + std::to_string(P));
  if (P > kMaxP)
    return fail(PNP_EINVAL, "patch_side > " + std::to_string(kMaxP) + " not supported");
  if (R < 1) return fail(PNP_EINVAL, "window_radius must be >= 1, got " + std::to_string(R));
  if (!(bw > 0)) return fail(PNP_EINVAL, "bandwidth must be > 0");
  const int margin = R + (P - 1) / 2;
  const int mn = H < W ? H : W;
  if (margin > mn)
    return fail(PNP_EINVAL, "margin " + std::to_string(margin) + " exceeds min image extent " +
                                std::to_string(mn));
  if (R > kMaxR)
    return fail(PNP_EINVAL, "window_radius > " + std::to_string(kMaxR) + " not supported");
  return PNP_OK;
}

static int make_plan(pnp_ctx* ctx, int B, int H, int W, int R, int P, Plan& pl) {
  pl.B = B;
  pl.H = H;
  pl.W = W;
  pl.R = R;
  pl.P = P;
  pl.TH = tile_height(P);
  pl.tiles_x = (W + kTW - 1) / kTW;
  pl.tiles_y = (H + pl.TH - 1) / pl.TH;
  pl.ntiles = pl.tiles_x * pl.tiles_y;
  std::vector<Chunk> ch, ch0;
  build_chunks(R, true, ch);
  build_chunks(R, false, ch0);
  pl.nchunks = (int)ch.size();
  pl.NG = pick_groups(pl.ntiles, pl.nchunks);
  auto key = std::make_pair(R, pl.NG);
  auto it = ctx->tables.find(key);
  const size_t cb = ch.size() * sizeof(Chunk);
  if (it == ctx->tables.end()) {
    std::vector<int> grp(pl.NG + 1);
    for (int g = 0; g <= pl.NG; ++g) grp[g] = (int)((long long)g * pl.nchunks / pl.NG);
    DevBuf buf;
    int rc = buf.ensure(2 * cb + grp.size() * sizeof(int));
    if (rc) return rc;
    PNP_CUDA(cudaMemcpy(buf.ptr, ch.data(), cb, cudaMemcpyHostToDevice));
    PNP_CUDA(cudaMemcpy(buf.as<char>() + cb, ch0.data(), cb, cudaMemcpyHostToDevice));
    PNP_CUDA(cudaMemcpy(buf.as<char>() + 2 * cb, grp.data(), grp.size() * sizeof(int),
                        cudaMemcpyHostToDevice));
    it = ctx->tables.emplace(key, buf).first;
  }
  pl.chunks = it->second.as<Chunk>();
  pl.chunks_nohat = reinterpret_cast<const Chunk*>(it->second.as<char>() + cb);
  pl.grp = reinterpret_cast<const int*>(it->second.as<char>() + 2 * cb);
  return PNP_OK;
}

static size_t partial_floats(const Plan& pl, int C) {
  return (size_t)pl.B * pl.NG * pl.ntiles * C * (pl.TH + pl.R) * (kTW + 2 * pl.R);
}

template <int RB, int C>
static cudaError_t launch_sweep_rc(const SweepArgs& a, int P, dim3 grid, cudaStream_t st) {
  switch (P) {
    case 1: return launch_sweep<1, RB, C>(a, grid, st);
    case 3: return launch_sweep<3, RB, C>(a, grid, st);
    case 5: return launch_sweep<5, RB, C>(a, grid, st);
    case 7: return launch_sweep<7, RB, C>(a, grid, st);
    case 9: return launch_sweep<9, RB, C>(a, grid, st);
    case 11: return launch_sweep<11, RB, C>(a, grid, st);
    case 13: return launch_sweep<13, RB, C>(a, grid, st);
    case 15: return launch_sweep<15, RB, C>(a, grid, st);
  }
  return cudaErrorInvalidValue;
}

template <int C>
static cudaError_t launch_sweep_c(const SweepArgs& a, const Plan& pl, cudaStream_t st) {
  dim3 grid(pl.ntiles, pl.NG, pl.B);
  switch (r_bucket(pl.R)) {
    case 5: return launch_sweep_rc<5, C>(a, pl.P, grid, st);
    case 10: return launch_sweep_rc<10, C>(a, pl.P, grid, st);
    case 16: return launch_sweep_rc<16, C>(a, pl.P, grid, st);
    default: return launch_sweep_rc<32, C>(a, pl.P, grid, st);
  }
}

static int run_sweep(pnp_ctx* ctx, const Plan& pl, int C, const float* guide, ChanSpec c0,
                     ChanSpec c1, const float* taps, double bw, bool use_hat) {
  SweepArgs a;
  memset(&a, 0, sizeof(a));
  a.guide = guide;
  a.ch[0] = c0;
  a.ch[1] = c1;
  int rc = ctx->partial.ensure(partial_floats(pl, 2) * sizeof(float));
  if (rc) return rc;
  a.partial = ctx->partial.as<float>();
  a.chunks = use_hat ? pl.chunks : pl.chunks_nohat;
  a.grp = pl.grp;
  a.H = pl.H;
  a.W = pl.W;
  a.R = pl.R;
  a.tiles_x = pl.tiles_x;
  a.tiles_y = pl.tiles_y;
  // k = exp(-sum w_a w_b D / (2 bw^2)) = ex2(-log2(e)/(2 bw^2) * ...)
  const double scale = -1.0 / (2.0 * log(2.0) * bw * bw);
  for (int i = 0; i < pl.P; ++i) {
    a.taps_h[i] = taps[i];
    a.taps_v[i] = (float)(scale * (double)taps[i]);
  }
  cudaError_t e = C == 1 ? launch_sweep_c<1>(a, pl, ctx->stream)
                         : launch_sweep_c<2>(a, pl, ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "dsg_sweep_kernel");
  return PNP_OK;
}

template <int MODE>
static int run_fixup(pnp_ctx* ctx, const Plan& pl, int C, const FixIO& io) {
  FixGeo f;
  f.partial = ctx->partial.as<float>();
  f.H = pl.H;
  f.W = pl.W;
  f.R = pl.R;
  f.TH = pl.TH;
  f.tiles_x = pl.tiles_x;
  f.tiles_y = pl.tiles_y;
  f.NG = pl.NG;
  f.C = C;
  const size_t plane = (size_t)pl.H * pl.W;
  dim3 grid((unsigned)((plane + 255) / 256), pl.B);
  dsg_fixup_kernel<MODE><<<grid, 256, 0, ctx->stream>>>(f, io);
  PNP_LAUNCH_CHECK("dsg_fixup_kernel");
  return PNP_OK;
}

static int ensure_planes(pnp_ctx* ctx, size_t n) {
  int rc;
  if ((rc = ctx->rs.ensure(n * sizeof(float)))) return rc;
  if ((rc = ctx->kx.ensure(n * sizeof(float)))) return rc;
  if ((rc = ctx->d.ensure(n * sizeof(float)))) return rc;
  return PNP_OK;
}

// g -> rs: sweep A + fixup (guide-only; shared by adaptive and freeze)
static int mass_and_rs(pnp_ctx* ctx, const Plan& pl, const float* guide, const float* taps,
                       double bw, float* rs) {
  int rc = run_sweep(ctx, pl, 1, guide, ChanSpec{nullptr, nullptr}, ChanSpec{nullptr, nullptr},
                     taps, bw, true);
  if (rc) return rc;
  FixIO io{};
  io.rs = rs;
  return run_fixup<FIX_RS>(ctx, pl, 1, io);
}

static int validate_taps(const float* taps, int P) {
  if (!taps) return fail(PNP_EINVAL, "taps must not be null");
  double s = 0;
  for (int i = 0; i < P; ++i) {
    if (!(taps[i] >= 0) || !isfinite(taps[i])) return fail(PNP_EINVAL, "taps must be finite, >= 0");
    s += taps[i];
  }
  if (fabs(s - 1.0) > 1e-5) return fail(PNP_EINVAL, "taps must sum to 1");
  return PNP_OK;
}

}  // namespace pnp

using namespace pnp;

extern "C" {

int pnp_version(void) { return 1; }
const char* pnp_last_error(void) { return g_last_error.c_str(); }

int pnp_ctx_create(int device, pnp_ctx** out) {
  if (!out) return fail(PNP_EINVAL, "out is null");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (device < 0 || device >= n) return fail(PNP_EINVAL, "invalid device index");
  PNP_CUDA(cudaSetDevice(device));
  pnp_ctx* c = new pnp_ctx();
  c->device = device;
  *out = c;
  return PNP_OK;
}

int pnp_ctx_destroy(pnp_ctx* ctx) {
  if (!ctx) return PNP_OK;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  ctx->partial.release();
  ctx->rs.release();
  ctx->kx.release();
  ctx->d.release();
  ctx->mbits.release();
  ctx->stats.release();
  ctx->flags.release();
  for (auto& kv : ctx->tables) kv.second.release();
  delete ctx;
  return PNP_OK;
}

int pnp_ctx_set_stream(pnp_ctx* ctx, void* stream) {
  if (!ctx) return fail(PNP_EINVAL, "ctx is null");
  ctx->stream = static_cast<cudaStream_t>(stream);
  return PNP_OK;
}

int pnp_ctx_synchronize(pnp_ctx* ctx) {
  if (!ctx) return fail(PNP_EINVAL, "ctx is null");
  PNP_CUDA(cudaStreamSynchronize(ctx->stream));
  return PNP_OK;
}

int pnp_ctx_reserve(pnp_ctx* ctx, int batch, int H, int W, int R, int P) {
  if (!ctx) return fail(PNP_EINVAL, "ctx is null");
  int rc = check_geometry(batch, H, W, R, P, 1.0);
  if (rc) return rc;
  PNP_CUDA(cudaSetDevice(ctx->device));
  Plan pl;
  if ((rc = make_plan(ctx, batch, H, W, R, P, pl))) return rc;
  if ((rc = ctx->partial.ensure(partial_floats(pl, 2) * sizeof(float)))) return rc;
  if ((rc = ensure_planes(ctx, (size_t)batch * H * W))) return rc;
  if ((rc = ctx->mbits.ensure(batch * sizeof(unsigned)))) return rc;
  return PNP_OK;
}

int pnp_dsg_denoise(pnp_ctx* ctx, const float* x, const float* guide, float* out, int batch,
                    int H, int W, int R, int P, const float* taps, double bandwidth,
                    float* d_out, float* alpha_out) {
  if (!ctx || !x || !out) return fail(PNP_EINVAL, "null argument");
  int rc = check_geometry(batch, H, W, R, P, bandwidth);
  if (rc) return rc;
  if ((rc = validate_taps(taps, P))) return rc;
  if (!guide) guide = x;
  PNP_CUDA(cudaSetDevice(ctx->device));
  Plan pl;
  if ((rc = make_plan(ctx, batch, H, W, R, P, pl))) return rc;
  const size_t n = (size_t)batch * H * W;
  if ((rc = ensure_planes(ctx, n))) return rc;
  if ((rc = ctx->mbits.ensure(batch * sizeof(unsigned)))) return rc;
  float* rs = ctx->rs.as<float>();
  float* kx = ctx->kx.as<float>();
  float* d = d_out ? d_out : ctx->d.as<float>();
  if ((rc = mass_and_rs(ctx, pl, guide, taps, bandwidth, rs))) return rc;
  if ((rc = run_sweep(ctx, pl, 2, guide, ChanSpec{rs, x}, ChanSpec{rs, nullptr}, taps, bandwidth,
                      true)))
    return rc;
  PNP_CUDA(cudaMemsetAsync(ctx->mbits.ptr, 0, batch * sizeof(unsigned), ctx->stream));
  FixIO io{};
  io.rs = rs;
  io.kx = kx;
  io.d = d;
  io.mbits = ctx->mbits.as<unsigned>();
  if ((rc = run_fixup<FIX_KXD>(ctx, pl, 2, io))) return rc;
  const size_t plane = (size_t)H * W;
  dim3 grid((unsigned)((plane + 255) / 256), batch);
  dsg_finalize_kernel<<<grid, 256, 0, ctx->stream>>>(kx, d, ctx->mbits.as<unsigned>(), x, out,
                                                     alpha_out, plane);
  PNP_LAUNCH_CHECK("dsg_finalize_kernel");
  return PNP_OK;
}

int pnp_dsg_freeze(pnp_ctx* ctx, const float* guide, int batch, int H, int W, int R, int P,
                   const float* taps, double bandwidth, pnp_frozen** out) {
  if (!ctx || !guide || !out) return fail(PNP_EINVAL, "null argument");
  int rc = check_geometry(batch, H, W, R, P, bandwidth);
  if (rc) return rc;
  if ((rc = validate_taps(taps, P))) return rc;
  PNP_CUDA(cudaSetDevice(ctx->device));
  Plan pl;
  if ((rc = make_plan(ctx, batch, H, W, R, P, pl))) return rc;
  const size_t n = (size_t)batch * H * W;
  pnp_frozen* fz = new pnp_frozen();
  fz->device = ctx->device;
  fz->B = batch;
  fz->H = H;
  fz->W = W;
  fz->R = R;
  fz->P = P;
  fz->bw = bandwidth;
  for (int i = 0; i < P; ++i) fz->taps[i] = taps[i];
  cudaError_t e = cudaMalloc(&fz->guide, n * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&fz->rs, n * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&fz->d, n * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&fz->mv, 2 * batch * sizeof(float));
  if (e != cudaSuccess) {
    pnp_frozen_destroy(fz);
    return cuda_fail(e, "cudaMalloc(frozen)");
  }
  auto bail = [&](int code) {
    pnp_frozen_destroy(fz);
    return code;
  };
  e = cudaMemcpyAsync(fz->guide, guide, n * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream);
  if (e != cudaSuccess) return bail(cuda_fail(e, "cudaMemcpyAsync(guide)"));
  if ((rc = ctx->mbits.ensure(batch * sizeof(unsigned)))) return bail(rc);
  if ((rc = mass_and_rs(ctx, pl, fz->guide, taps, bandwidth, fz->rs))) return bail(rc);
  if ((rc = run_sweep(ctx, pl, 1, fz->guide, ChanSpec{fz->rs, nullptr}, ChanSpec{nullptr, nullptr},
                      taps, bandwidth, true)))
    return bail(rc);
  e = cudaMemsetAsync(ctx->mbits.ptr, 0, batch * sizeof(unsigned), ctx->stream);
  if (e != cudaSuccess) return bail(cuda_fail(e, "cudaMemsetAsync"));
  FixIO io{};
  io.rs = fz->rs;
  io.d = fz->d;
  io.mbits = ctx->mbits.as<unsigned>();
  if ((rc = run_fixup<FIX_D>(ctx, pl, 1, io))) return bail(rc);
  dsg_alpha_kernel<<<(batch + 127) / 128, 128, 0, ctx->stream>>>(ctx->mbits.as<unsigned>(),
                                                                 fz->mv, batch);
  e = cudaGetLastError();
  if (e != cudaSuccess) return bail(cuda_fail(e, "dsg_alpha_kernel"));
  *out = fz;
  return PNP_OK;
}

int pnp_dsg_apply(pnp_ctx* ctx, const pnp_frozen* fz, const float* x, float* out) {
  if (!ctx || !fz || !x || !out) return fail(PNP_EINVAL, "null argument");
  if (fz->device != ctx->device) return fail(PNP_EINVAL, "handle belongs to another device");
  PNP_CUDA(cudaSetDevice(ctx->device));
  Plan pl;
  int rc = make_plan(ctx, fz->B, fz->H, fz->W, fz->R, fz->P, pl);
  if (rc) return rc;
  if ((rc = run_sweep(ctx, pl, 1, fz->guide, ChanSpec{fz->rs, x}, ChanSpec{nullptr, nullptr},
                      fz->taps, fz->bw, true)))
    return rc;
  FixIO io{};
  io.rs = fz->rs;
  io.d = fz->d;
  io.inv_m = fz->mv + fz->B;
  io.x = x;
  io.out = out;
  return run_fixup<FIX_APPLY>(ctx, pl, 1, io);
}

int pnp_frozen_destroy(pnp_frozen* fz) {
  if (!fz) return PNP_OK;
  cudaSetDevice(fz->device);
  if (fz->guide) cudaFree(fz->guide);
  if (fz->rs) cudaFree(fz->rs);
  if (fz->d) cudaFree(fz->d);
  if (fz->mv) cudaFree(fz->mv);
  delete fz;
  return PNP_OK;
}

int pnp_frozen_alpha(const pnp_frozen* fz, float* alpha_host) {
  if (!fz || !alpha_host) return fail(PNP_EINVAL, "null argument");
  PNP_CUDA(cudaSetDevice(fz->device));
  PNP_CUDA(cudaMemcpy(alpha_host, fz->mv, fz->B * sizeof(float), cudaMemcpyDeviceToHost));
  return PNP_OK;
}

int pnp_frozen_export(pnp_ctx* ctx, const pnp_frozen* fz, float* guide_out, float* d_out) {
  if (!ctx || !fz) return fail(PNP_EINVAL, "null argument");
  const size_t n = (size_t)fz->B * fz->H * fz->W * sizeof(float);
  PNP_CUDA(cudaSetDevice(ctx->device));
  if (guide_out)
    PNP_CUDA(cudaMemcpyAsync(guide_out, fz->guide, n, cudaMemcpyDeviceToDevice, ctx->stream));
  if (d_out) PNP_CUDA(cudaMemcpyAsync(d_out, fz->d, n, cudaMemcpyDeviceToDevice, ctx->stream));
  return PNP_OK;
}

int pnp_frozen_shape(const pnp_frozen* fz, int* batch, int* H, int* W, int* R, int* P) {
  if (!fz) return fail(PNP_EINVAL, "null argument");
  if (batch) *batch = fz->B;
  if (H) *H = fz->H;
  if (W) *W = fz->W;
  if (R) *R = fz->R;
  if (P) *P = fz->P;
  return PNP_OK;
}

int pnp_nlm_denoise(pnp_ctx* ctx, const float* x, const float* guide, float* out, int batch,
                    int H, int W, int R, int P, const float* taps, double bandwidth) {
  if (!ctx || !x || !out) return fail(PNP_EINVAL, "null argument");
  int rc = check_geometry(batch, H, W, R, P, bandwidth);
  if (rc) return rc;
  if ((rc = validate_taps(taps, P))) return rc;
  if (!guide) guide = x;
  PNP_CUDA(cudaSetDevice(ctx->device));
  Plan pl;
  if ((rc = make_plan(ctx, batch, H, W, R, P, pl))) return rc;
  // num = sum k x(s+t), den = sum k (no hat, no normalization; denoise.py:254-269)
  if ((rc = run_sweep(ctx, pl, 2, guide, ChanSpec{x, nullptr}, ChanSpec{nullptr, nullptr}, taps,
                      bandwidth, false)))
    return rc;
  FixIO io{};
  io.out = out;
  return run_fixup<FIX_NLM>(ctx, pl, 2, io);
}

}  // extern "C"
