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
#include <limits.h>
#include <math.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "admm_math.cuh"
#include "dsg_generic.cuh"
#include "dsg_sweep.cuh"
#include "sweep_launch.cuh"
#include "pnp_internal.h"
#include "pnp_reduce.cuh"

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

enum FixMode { FIX_RS = 0, FIX_KXD = 1, FIX_D = 2, FIX_APPLY = 3, FIX_NLM = 4, FIX_APPLY_U = 5 };

// Per-pixel buffers are windows [buf_r0, buf_r0 + buf_rows) x W (FixGeo).
struct FixIO {
  float* rs;           // in (KXD, D, APPLY) / out (RS)
  float* kx;           // out (KXD)
  float* d;            // out (KXD, D) / in (APPLY)
  unsigned* mbits;     // per-image max bits (KXD, D)
  const float* inv_m;  // per image (APPLY)
  const float* x;      // (APPLY)
  float* out;          // (APPLY, NLM)
  // FIX_APPLY_U: the ADMM u-update fused into the frozen apply (solver.py:
  // 222-228): v = out, u += x_admm - v, per-CTA partials of sum (x-v)^2,
  // sum (rho (v - v_prev))^2, sum (gt - v)^2, finite flags
  float* u;
  const float* xa;
  const float* vprev;
  const float* gt;
  double rho;
  double* part3;       // [B][gridDim.y * gridDim.x][3]
  int* flags;
  // when set, the last CTA reduces part3 into stats_out[b][0..2] (stride 4)
  double* stats_out;
  unsigned* counter;   // zero between launches (the last CTA resets it)
  // FIX_APPLY_U with grad set: the next iteration's x-update fused in
  // (solver.py:219-221): x = clamp(mu (alpha x + rho (v - u) - grad)) over
  // xa, z = x + u over the apply input; its finite flags into xflags
  const float* grad;
  double mu, alpha;
  float lo, hi;
  int* xflags;
};

// the fused x-update of one pixel (grad set): x_a and the apply input z are
// rewritten in place (this thread alone reads / writes them at o)
__device__ __forceinline__ int admm_x_next(const FixIO& io, size_t o, float xa, float v,
                                           float un) {
  float xf, zf;
  const int f = admm_xupdate(io.mu, io.alpha, io.rho, io.lo, io.hi, xa, v, un, io.grad[o], xf, zf);
  const_cast<float*>(io.xa)[o] = xf;
  const_cast<float*>(io.x)[o] = zf;
  return f;
}

// u-update of one pixel (same arithmetic as admm_uupdate_kernel)
__device__ __forceinline__ int admm_u_pixel(const FixIO& io, size_t o, float v, double& s0,
                                            double& s1, double& s2, float& xa_out, float& un_out) {
  const float xa = io.xa[o];
  const double xv = xa, vv = v;
  const float un = (float)((double)io.u[o] + (xv - vv));
  io.u[o] = un;
  xa_out = xa;
  un_out = un;
  s0 += (xv - vv) * (xv - vv);
  const double dv = io.rho * (vv - (io.vprev ? (double)io.vprev[o] : 0.0));
  s1 += dv * dv;
  if (io.gt) {
    const double e = (double)io.gt[o] - vv;
    s2 += e * e;
  }
  return (!isfinite(vv) || !isfinite(un)) ? 4 : 0;
}

// the same u-update from preloaded values (vprev / gt ignored when null)
__device__ __forceinline__ int admm_u_values(const FixIO& io, size_t o, float v, float u,
                                             float xa, float vprev, float gt, double& s0,
                                             double& s1, double& s2, float& un_out) {
  const double xv = xa, vv = v;
  const float un = (float)((double)u + (xv - vv));
  io.u[o] = un;
  un_out = un;
  s0 += (xv - vv) * (xv - vv);
  const double dv = io.rho * (vv - (io.vprev ? (double)vprev : 0.0));
  s1 += dv * dv;
  if (io.gt) {
    const double e = (double)gt - vv;
    s2 += e * e;
  }
  return (!isfinite(vv) || !isfinite(un)) ? 4 : 0;
}

// block-level epilogue of FIX_APPLY_U: flags + deterministic stats partials
__device__ __forceinline__ void admm_u_block(const FixIO& io, int b, int f, double s0, double s1,
                                             double s2) {
  f = __reduce_or_sync(0xffffffffu, f);
  if (f && (threadIdx.x & 31) == 0) atomicOr(io.flags, f);
  __shared__ double red3[3][8];
  for (int off = 16; off; off >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, off);
    s1 += __shfl_xor_sync(0xffffffffu, s1, off);
    s2 += __shfl_xor_sync(0xffffffffu, s2, off);
  }
  const int wid = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red3[0][wid] = s0;
    red3[1][wid] = s1;
    red3[2][wid] = s2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a0 = 0, a1 = 0, a2 = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      a0 += red3[0][k];
      a1 += red3[1][k];
      a2 += red3[2][k];
    }
    double* pp = io.part3 + (((size_t)b * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 3;
    pp[0] = a0;
    pp[1] = a1;
    pp[2] = a2;
  }
}

// The per-image sums of FIX_APPLY_U's partials, folded into the fixup: the
// last CTA to finish reduces them (same arithmetic as reduce_partials_kernel).
// One counter per image (blockIdx.z): the last CTA of each image reduces that
// image's sums, so a batch's reductions run in parallel instead of as one
// CTA's serial tail (config 5: 64 images).
__device__ __forceinline__ void admm_stats_last(const FixIO& io) {
  const int nblk = gridDim.x * gridDim.y;
  if (!io.stats_out || !cta_is_last_of(io.counter + blockIdx.z, (unsigned)nblk)) return;
  __shared__ double red[3][8];
  cta_reduce_partials3(io.part3, nblk, blockIdx.z, 1.0, io.stats_out, 4, red);
}

__device__ __forceinline__ float dsg_finish(float kx, float d, float inv_m, float x) {
  const float w = __fmul_rn(kx, inv_m);
  const float mass = __fmul_rn(d, inv_m);
  return __fmaf_rn(__fsub_rn(1.f, mass), x, w);
}

// Predicated read-only load (+0 when off).
__device__ __forceinline__ float ldg_pred(const float* p, bool on) {
  float v = 0.f;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
      "@q ld.global.nc.f32 %0, [%1];\n\t}"
      : "+f"(v)
      : "l"(p), "r"((int)on));
  return v;
}

// Small images (many offset groups): one thread per pixel; a CTA covers 4
// rows x 64 columns of one tile
// (blockIdx.y = tile row * ceil(TH/4) + row quarter).  A pixel is covered by
// at most 3 tile rows x 2 tile columns of partial blocks per offset group
// (only one side column lies within R <= 32 of the pixel); their offsets are
// computed once per pixel.  The
// loads of kFixGB groups are all issued before any add, then summed in the
// fixed order (group, tile row, tile col) that every variant (single GPU,
// strips, apply) shares -> bit-reproducible, and latency-tolerant when NG is
// large (small images split the offsets into many groups).  The epilogue's
// per-pixel inputs are loaded up front so their latency hides under the sums.
#ifndef PNP_FIXGB
#define PNP_FIXGB 2
#endif
#ifndef PNP_FIXLB
#define PNP_FIXLB 4  // min resident CTAs per SM (register cap)
#endif

template <int MODE>
__global__ void __launch_bounds__(256, PNP_FIXLB) dsg_fixup_px_kernel(const FixGeo f, const FixIO io) {
  pdl_begin();
  constexpr int C = (MODE == FIX_KXD || MODE == FIX_NLM) ? 2 : 1;
  constexpr int kFixGB = C == 1 ? PNP_FIXGB : PNP_FIXGB / 2;  // offset groups per batch of loads
  const int b = blockIdx.z;
  const int TH = f.TH, R = f.R, W = f.W;
  const int BR = TH + R, BC = kTW + 2 * R;
  const int RQ = (TH + 3) / 4;
  const int tq = blockIdx.y % RQ;
  const int ti = f.y0 / TH + blockIdx.y / RQ, tj = blockIdx.x;
  const int lx = threadIdx.x & (kTW - 1), ly = tq * 4 + (threadIdx.x >> 6);
  const int x = tj * kTW + lx, y = ti * TH + ly;
  const bool own = ly < TH && x < W && y >= f.y0 && y < f.y0 + f.nrows && y < f.Hg;
  const size_t blk = (size_t)f.C * BR * BC;
  const float* base = f.partial + (size_t)b * f.part_ntr * f.NP * f.tiles_x * blk;
  const int dti = (R + TH - 1) / TH;
  const int ti0 = max(max(f.part_tr0, 0), ti - dti), ti1 = min(ti, f.part_tr0 + f.part_ntr - 1);
  const int tj0 = max(0, tj - 1), tj1 = min(f.tiles_x - 1, tj + 1);

  // per-pixel epilogue inputs, issued before the partial sums
  const size_t o = (size_t)b * f.buf_rows * W + (size_t)(y - f.buf_r0) * W + x;
  float e_rs = 0.f, e_d = 0.f, e_x = 0.f, e_u = 0.f, e_xa = 0.f, e_vp = 0.f, e_gt = 0.f;
  if (own) {
    if (MODE == FIX_APPLY_U || MODE == FIX_KXD || MODE == FIX_D || MODE == FIX_APPLY)
      e_rs = io.rs[o];
    if (MODE == FIX_APPLY_U || MODE == FIX_APPLY) {
      e_d = io.d[o];
      e_x = io.x[o];
    }
    if (MODE == FIX_APPLY_U) {
      e_u = io.u[o];
      e_xa = io.xa[o];
      if (io.vprev) e_vp = io.vprev[o];
      if (io.gt) e_gt = io.gt[o];
    }
  }

  // covering blocks of this pixel, in (tile row, tile col) order: per tile
  // row, the own tile column and at most one side column (left when lx < R,
  // right when lx >= 64 - R; R <= 32 so never both) -> slots (i, 0..1).
  // 32-bit float offsets from the image's partial base (the host keeps an
  // image's partial array below 2^32 floats for this kernel).
  const bool sideL = lx < R, sideR = !sideL && lx >= kTW - R;
  unsigned boff[3][2];
  unsigned okm = 0;  // bit 2*i + k
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int t_i = ti0 + i;
      const int t_j = sideL ? tj - 1 + k : tj + k;
      const int br = y - t_i * TH, bc = x - t_j * kTW + R;
      const bool ok = own && (k == 0 || sideL || sideR) && t_i <= ti1 && t_j >= tj0 &&
                      t_j <= tj1 && br < BR && bc >= 0 && bc < BC;
      okm |= (ok ? 1u : 0u) << (2 * i + k);
      boff[i][k] = ok ? (unsigned)(((t_i - f.part_tr0) * f.NP * f.tiles_x + t_j) * blk) +
                            (unsigned)(br * BC + bc)
                      : 0u;
    }
  const unsigned gstride = (unsigned)(f.tiles_x * blk);  // next group, same tile
  const unsigned cstride = (unsigned)(BR * BC);

  float s[C] = {};
  for (int g0 = 0; g0 < f.NP; g0 += kFixGB) {
    const float* gb = base + (size_t)g0 * gstride;
    float v[kFixGB][3][2][C];
#pragma unroll
    for (int gg = 0; gg < kFixGB; ++gg)
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const bool ok = g0 + gg < f.NP && ((okm >> (2 * i + k)) & 1u);
          const unsigned off = (unsigned)gg * gstride + boff[i][k];
#pragma unroll
          for (int c_ = 0; c_ < C; ++c_) v[gg][i][k][c_] = ldg_pred(gb + (off + c_ * cstride), ok);
        }
#pragma unroll
    for (int gg = 0; gg < kFixGB; ++gg)
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 2; ++k)
          if (g0 + gg < f.NP && ((okm >> (2 * i + k)) & 1u))
#pragma unroll
            for (int c_ = 0; c_ < C; ++c_) s[c_] = __fadd_rn(s[c_], v[gg][i][k][c_]);
  }

  float dmax = 0.f;
  double u0 = 0.0, u1 = 0.0, u2 = 0.0;
  int uf = 0, xf = 0;
  if (own) {
    const float s0 = s[0];
    if (MODE == FIX_APPLY_U) {
      const float kx = __fmul_rn(e_rs, s0);
      const float v = dsg_finish(kx, e_d, io.inv_m[b], e_x);
      io.out[o] = v;
      float un;
      uf = admm_u_values(io, o, v, e_u, e_xa, e_vp, e_gt, u0, u1, u2, un);
      if (io.grad) xf = admm_x_next(io, o, e_xa, v, un);
    } else if (MODE == FIX_RS) {
      io.rs[o] = __fdiv_rn(1.f, __fsqrt_rn(fmaxf(s0, FLT_MIN)));
    } else if (MODE == FIX_KXD) {
      io.kx[o] = __fmul_rn(e_rs, s0);
      dmax = __fmul_rn(e_rs, s[C - 1]);
      io.d[o] = dmax;
    } else if (MODE == FIX_D) {
      dmax = __fmul_rn(e_rs, s0);
      io.d[o] = dmax;
    } else if (MODE == FIX_APPLY) {
      const float kx = __fmul_rn(e_rs, s0);
      io.out[o] = dsg_finish(kx, e_d, io.inv_m[b], e_x);
    } else {  // FIX_NLM: num / den
      io.out[o] = __fdiv_rn(s0, s[C - 1]);
    }
  }
  if (MODE == FIX_APPLY_U && io.grad) {
    xf = __reduce_or_sync(0xffffffffu, xf);
    if (xf && (threadIdx.x & 31) == 0) atomicOr(io.xflags, xf);
  }
  if (MODE == FIX_APPLY_U) admm_u_block(io, b, uf, u0, u1, u2), admm_stats_last(io);
  if (MODE == FIX_KXD || MODE == FIX_D) {
    // d > 0, so the int ordering of the bits is the float ordering; max is
    // exact and order-free -> deterministic.
    __shared__ float red[8];
    float v = dmax;
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

// Large images (few offset groups): one CTA per output tile (TH x 64 pixels of tile row blockIdx.y + the
// window's first tile row, tile column blockIdx.x).  Thread (lx, ly0) owns
// column lx and rows ly0, ly0+4, ... of the tile, so every covering partial
// block is visited by all threads in the same fixed order (group, tile row,
// tile col) -- the per-pixel summation order shared by all fixups -- while each
// thread keeps up to 8 independent loads in flight per block.
constexpr int kFixRows = 8;  // rows per thread (TH <= 32, 4 row phases)

// 4 resident CTAs per SM (64 registers): the fixups are latency-bound, and
// occupancy beats keeping more rows' loads in registers (8192^2 launch list:
// -12..-38% per mode against no register cap); FIX_NLM (two channels) at 3.
template <int MODE>
__global__ void __launch_bounds__(256, MODE == FIX_NLM ? 3 : 4) dsg_fixup_tile_kernel(const FixGeo f, const FixIO io) {
  pdl_begin();
  constexpr int C = (MODE == FIX_KXD || MODE == FIX_NLM) ? 2 : 1;
  const int b = blockIdx.z;
  const int TH = f.TH, R = f.R, W = f.W;
  const int BR = TH + R, BC = kTW + 2 * R;
  const int ti = f.y0 / TH + blockIdx.y, tj = blockIdx.x;
  const int lx = threadIdx.x & (kTW - 1), ly0 = threadIdx.x >> 6;
  const int x = tj * kTW + lx;
  const int ylo = max(f.y0, ti * TH), yhi = min(min(f.y0 + f.nrows, f.Hg), ti * TH + TH);
  const size_t blk = (size_t)f.C * BR * BC;
  const float* base = f.partial + (size_t)b * f.part_ntr * f.NP * f.tiles_x * blk;
  const int dti = (R + TH - 1) / TH, dtj = (R + kTW - 1) / kTW;
  const int ti0 = max(max(f.part_tr0, 0), ti - dti), ti1 = min(ti, f.part_tr0 + f.part_ntr - 1);
  const int tj0 = max(0, tj - dtj), tj1 = min(f.tiles_x - 1, tj + dtj);

  // Pull every covering block's row band into L2 with bulk prefetches first,
  // so the per-thread loads below see L2 latency rather than HBM latency.
  {
    const int nti = ti1 - ti0 + 1, ntj = tj1 - tj0 + 1;
    const int nq = f.NP * nti * ntj * C;
    for (int q = threadIdx.x; q < nq; q += blockDim.x) {
      int r_ = q;
      const int c_ = r_ % C; r_ /= C;
      const int t_j = tj0 + r_ % ntj; r_ /= ntj;
      const int t_i = ti0 + r_ % nti;
      const int gg = r_ / nti;
      const int br0 = ti * TH - t_i * TH, br1 = min(BR, br0 + TH);
      if (br0 >= br1) continue;
      const float* p = base + (((size_t)(t_i - f.part_tr0) * f.NP + gg) * f.tiles_x + t_j) * blk +
                       (size_t)c_ * BR * BC + (size_t)br0 * BC;
      const uintptr_t a0 = (uintptr_t)p & ~(uintptr_t)15;
      const uintptr_t a1 = ((uintptr_t)(p + (size_t)(br1 - br0) * BC) + 15) & ~(uintptr_t)15;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((unsigned)(a1 - a0))
                   : "memory");
    }
  }

  // per-pixel epilogue inputs of the plain modes, issued before the sums
  constexpr bool HOIST = MODE == FIX_KXD || MODE == FIX_D;  // (FIX_APPLY: measured slower)
  float e_rs[kFixRows];
#pragma unroll
  for (int k = 0; k < kFixRows; ++k) {
    const int y = ti * TH + ly0 + 4 * k;
    const bool ok = HOIST && ly0 + 4 * k < TH && y >= ylo && y < yhi && x < W;
    const size_t o = ok ? (size_t)b * f.buf_rows * W + (size_t)(y - f.buf_r0) * W + x : 0;
    e_rs[k] = ldg_pred(io.rs + o, ok);
  }

  float s[C][kFixRows];
#pragma unroll
  for (int c_ = 0; c_ < C; ++c_)
#pragma unroll
    for (int k = 0; k < kFixRows; ++k) s[c_][k] = 0.f;

  for (int gg = 0; gg < f.NP; ++gg)
    for (int t_i = ti0; t_i <= ti1; ++t_i) {
      const float* row = base + ((size_t)(t_i - f.part_tr0) * f.NP + gg) * f.tiles_x * blk;
      for (int t_j = tj0; t_j <= tj1; ++t_j) {
        const int bc = x - t_j * kTW + R;
        if (bc < 0 || bc >= BC || x >= W) continue;
        const float* p = row + (size_t)t_j * blk + bc;
        float v[C][kFixRows];
#pragma unroll
        for (int k = 0; k < kFixRows; ++k) {
          const int y = ti * TH + ly0 + 4 * k;
          const int br = y - t_i * TH;
          const bool ok = ly0 + 4 * k < TH && br < BR;
#pragma unroll
          for (int c_ = 0; c_ < C; ++c_) v[c_][k] = ldg_pred(p + (size_t)c_ * BR * BC + br * BC, ok);
        }
#pragma unroll
        for (int k = 0; k < kFixRows; ++k)
#pragma unroll
          for (int c_ = 0; c_ < C; ++c_)  // volatile: stays behind all the loads
            asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(s[c_][k]) : "f"(v[c_][k]));
      }
    }

  float dmax = 0.f;
  double u0 = 0.0, u1 = 0.0, u2 = 0.0;
  int uf = 0, xf = 0;
  if (MODE == FIX_APPLY_U) {
    // the fused ADMM epilogue reads 8 planes per pixel: the loads of 4 rows
    // are issued together before any of their stores (the stores could alias
    // the next row's loads for the compiler, which would otherwise serialize
    // one round trip per row); same per-pixel arithmetic, same row order
    constexpr int KB = 2;
#pragma unroll
    for (int k0 = 0; k0 < kFixRows; k0 += KB) {
      float ers[KB], ed[KB], ez[KB], exa[KB], eu[KB], evp[KB], egt[KB], egr[KB];
      size_t oo[KB];
      bool ok[KB];
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        const int k = k0 + j, y = ti * TH + ly0 + 4 * k;
        ok[j] = ly0 + 4 * k < TH && y >= ylo && y < yhi && x < W;
        oo[j] = ok[j] ? (size_t)b * f.buf_rows * W + (size_t)(y - f.buf_r0) * W + x : 0;
        ers[j] = ldg_pred(io.rs + oo[j], ok[j]);
        ed[j] = ldg_pred(io.d + oo[j], ok[j]);
        ez[j] = ldg_pred(io.x + oo[j], ok[j]);
        exa[j] = ldg_pred(io.xa + oo[j], ok[j]);
        eu[j] = ldg_pred(io.u + oo[j], ok[j]);
        evp[j] = ldg_pred(io.vprev + oo[j], ok[j] && io.vprev);
        egt[j] = ldg_pred(io.gt + oo[j], ok[j] && io.gt);
        egr[j] = ldg_pred(io.grad + oo[j], ok[j] && io.grad);
      }
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        if (!ok[j]) continue;
        const size_t o = oo[j];
        const float kx = __fmul_rn(ers[j], s[0][k0 + j]);
        const float v = dsg_finish(kx, ed[j], io.inv_m[b], ez[j]);
        io.out[o] = v;
        float un;
        uf |= admm_u_values(io, o, v, eu[j], exa[j], evp[j], egt[j], u0, u1, u2, un);
        if (io.grad) {
          float xn, zn;
          xf |= admm_xupdate(io.mu, io.alpha, io.rho, io.lo, io.hi, exa[j], v, un, egr[j], xn, zn);
          const_cast<float*>(io.xa)[o] = xn;
          const_cast<float*>(io.x)[o] = zn;
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kFixRows; ++k) {
    const int y = ti * TH + ly0 + 4 * k;
    if (MODE == FIX_APPLY_U || ly0 + 4 * k >= TH || y < ylo || y >= yhi || x >= W) continue;
    const size_t o = (size_t)b * f.buf_rows * W + (size_t)(y - f.buf_r0) * W + x;
    const float s0 = s[0][k];
    if (MODE == FIX_RS) {
      io.rs[o] = __fdiv_rn(1.f, __fsqrt_rn(fmaxf(s0, FLT_MIN)));
    } else if (MODE == FIX_KXD) {
      const float r = e_rs[k];
      io.kx[o] = __fmul_rn(r, s0);
      const float dv = __fmul_rn(r, s[C - 1][k]);
      io.d[o] = dv;
      dmax = fmaxf(dmax, dv);
    } else if (MODE == FIX_D) {
      const float dv = __fmul_rn(e_rs[k], s0);
      io.d[o] = dv;
      dmax = fmaxf(dmax, dv);
    } else if (MODE == FIX_APPLY) {
      const float kx = __fmul_rn(io.rs[o], s0);
      io.out[o] = dsg_finish(kx, io.d[o], io.inv_m[b], io.x[o]);
    } else {  // FIX_NLM: num / den
      io.out[o] = __fdiv_rn(s0, s[C - 1][k]);
    }
  }
  if (MODE == FIX_APPLY_U && io.grad) {
    xf = __reduce_or_sync(0xffffffffu, xf);
    if (xf && (threadIdx.x & 31) == 0) atomicOr(io.xflags, xf);
  }
  if (MODE == FIX_APPLY_U) admm_u_block(io, b, uf, u0, u1, u2), admm_stats_last(io);
  if (MODE == FIX_KXD || MODE == FIX_D) {
    // d > 0, so the int ordering of the bits is the float ordering; max is
    // exact and order-free -> deterministic.
    __shared__ float red[8];
    float v = dmax;
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

// out = Kx/m + (1 - d/m) x over output rows [y0, y0+nrows) of a window.
__global__ void dsg_finalize_kernel(const float* kx, const float* d, const unsigned* mbits,
                                    const float* x, float* out, float* alpha_out, int y0,
                                    int nrows, int W, int buf_r0, int buf_rows) {
  pdl_begin();
  const int b = blockIdx.y;
  const float m = __uint_as_float(mbits[b]);
  const float inv_m = __frcp_rn(m);
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (alpha_out && i == 0) alpha_out[b] = m;
  if (i < (size_t)nrows * W) {
    const size_t o = (size_t)b * buf_rows * W + (size_t)(y0 - buf_r0) * W + i;
    out[o] = dsg_finish(kx[o], d[o], inv_m, x[o]);
  }
}

// The same per pixel, four pixels per thread with 16-byte accesses (every
// plane 16-byte aligned and W % 4 == 0); grid-stride over the window.
__global__ void __launch_bounds__(256) dsg_finalize4_kernel(const float* kx, const float* d,
                                                            const unsigned* mbits, const float* x,
                                                            float* out, float* alpha_out, int y0,
                                                            int nrows, int W, int buf_r0,
                                                            int buf_rows) {
  pdl_begin();
  const int b = blockIdx.y;
  const float m = __uint_as_float(mbits[b]);
  const float inv_m = __frcp_rn(m);
  if (alpha_out && blockIdx.x == 0 && threadIdx.x == 0) alpha_out[b] = m;
  const size_t n4 = (size_t)nrows * W / 4;
  const size_t base = ((size_t)b * buf_rows * W + (size_t)(y0 - buf_r0) * W) / 4;
  const float4* k4 = reinterpret_cast<const float4*>(kx) + base;
  const float4* d4 = reinterpret_cast<const float4*>(d) + base;
  const float4* x4 = reinterpret_cast<const float4*>(x) + base;
  float4* o4 = reinterpret_cast<float4*>(out) + base;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (size_t)gridDim.x * blockDim.x) {
    const float4 a = __ldcs(k4 + i), dd = __ldcs(d4 + i), xx = __ldg(x4 + i);
    float4 r;
    r.x = dsg_finish(a.x, dd.x, inv_m, xx.x);
    r.y = dsg_finish(a.y, dd.y, inv_m, xx.y);
    r.z = dsg_finish(a.z, dd.z, inv_m, xx.z);
    r.w = dsg_finish(a.w, dd.w, inv_m, xx.w);
    __stcs(o4 + i, r);
  }
}

__global__ void dsg_alpha_kernel(const unsigned* mbits, float* mv, int B) {
  pdl_begin();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) {
    const float m = __uint_as_float(mbits[b]);
    mv[b] = m;
    mv[B + b] = __frcp_rn(m);
  }
}

// ------------------------------------------------------------------ host ---

// Global launch geometry: tile grid, offset table and offset-group split.
// Everything here depends only on (Hg, W, R, P), never on the window or the
// batch, so single-GPU and sharded runs sum in the same order.
struct Geom {
  int B, Hg, W, R, P, TH, tiles_x, tiles_y, nchunks, NG;
  int NP;            // partial groups per tile (= NG)
  int kind;          // PATH_FAST / PATH_GEN_SYM / PATH_GEN_NEAR
  bool box;          // equal patch taps: running-sum box filter (general kernel)
  int Rb;            // far band of a partial block (R, or 0 for tile-only blocks)
  int KG;            // general kernel: dy offsets per batch
  const Chunk* chunks;        // hat-tapered table (DSG), host (fast kernel)
  const Chunk* chunks_nohat;  // same offsets, L = 0 (plain NLM), host
  const int* grp;             // NG+1 group starts (chunks, or dy indices), host
  const float* ltab;          // general kernel: log2 hat per offset, device
};

// A window of the global image handled by one call.
struct Window {
  int buf_r0, buf_rows;  // per-pixel buffers: rows [buf_r0, buf_r0 + buf_rows)
  int tr0, ntr;          // tile rows swept
  int part_tr0, part_off, part_ntr;  // partial array: slot 0 = tile row part_tr0
  int y0, nrows;         // rows fixed up / finalized
};

static Window full_window(const Geom& g) {
  return Window{0, g.Hg, 0, g.tiles_y, 0, 0, g.tiles_y, 0, g.Hg};
}

// Half-window offsets grouped in chunks of KY consecutive dy sharing dx.
static void build_chunks(int R, bool hat, std::vector<Chunk>& out) {
  out.clear();
  int koff = 0;  // k-cache offset of the chunk in a tile's run (offset planes)
  for (int dx = -R; dx <= R; ++dx) {
    const int dy_first = dx > 0 ? 0 : 1;
    for (int dy0 = dy_first; dy0 <= R; dy0 += kKY) {
      Chunk ch;
      memset(&ch, 0, sizeof(ch));
      ch.dx = dx;
      ch.dy0 = dy0;
      ch.kc = (R - dy0 + 1) < kKY ? (R - dy0 + 1) : kKY;
      ch.koff = koff;
      koff += ch.kc;
      for (int k = 0; k < kKY; ++k) {
        // log2 of the separable hat (denoise.py:199-201), in double, rounded once
        const int dy = dy0 + k;
        const double s = R + 1.0;
        const double hy = 1.0 - fabs((double)dy) / s, hx = 1.0 - fabs((double)dx) / s;
        // slots past kc: -inf -> ex2 gives an exact +0 weight (packed pairs)
        ch.L[k] = k >= ch.kc ? -INFINITY : (hat ? (float)(log2(hy) + log2(hx)) : 0.f);
      }
      out.push_back(ch);
    }
  }
}

static int pick_groups(int ntiles, int nchunks) {
  // Offset groups per tile -- a function of the image geometry only, so every
  // path (adaptive, frozen, batched, sharded) sums in the same order.  Fitted
  // to B200 measurements of the frozen apply at R = 10 (k-cache sweep with
  // 4 CTAs/SM = 592 slots, then the fixup; profiles/sweep_history.md): about
  // 480 CTAs in all (one memory-bound wave; more groups cost more in the
  // per-pixel fixup than they gain), at most 7 groups, and 2 instead of 1
  // when one group per tile would spill a small tail wave.
  int ng = 480 / (ntiles > 0 ? ntiles : 1);
  if (ng > 7) ng = 7;
  if (ng < 1) ng = 1;
  if (ng == 1) {
    const double w = ntiles / (148.0 * 4);
    if (w > 1.0 && w < 4.0 && w - std::floor(w) < 0.35) ng = 2;
  }
  if (ng > nchunks) ng = nchunks;
#ifdef PNP_NG_OVERRIDE
  ng = PNP_NG_OVERRIDE;
#endif
  return ng < 1 ? 1 : ng;
}

// Which sweep kernel a geometry uses -- a function of (R, P, box) only, so
// adaptive, frozen, batched and sharded calls agree:
//   PATH_FAST      R <= 32 and Gaussian taps with P <= 15 / box taps with
//                  P <= 9: the P-templated sweep (dsg_sweep.cuh; k cache,
//                  packed f32x2 filter)
//   PATH_GEN_SYM   box taps (the reference's patch distance) from P = 11, and
//                  everything beyond the fast kernel: the general sweep
//                  (dsg_generic.cuh; running-sum box filter, cost flat in P),
//                  half window, tile + band blocks
//   PATH_GEN_NEAR  the general sweep over the full window, tile-only blocks
//                  (search radii whose far plane exceeds shared memory)
enum { PATH_FAST = 0, PATH_GEN_SYM = 1, PATH_GEN_NEAR = 2 };

static int choose_path(int R, int P, bool box, int& kind, int& TH, int& KG) {
#ifdef PNP_BOX_FAST  // A/B variant: box taps through the P-templated kernel too
  box = false;
#endif
  KG = 0;
  // Box patches (the reference's distance) run the general kernel from
  // P = 11 on -- one running-sum kernel over the reference's own Table-1 range
  // (P = 11..29, flat in P); below, and for Gaussian taps up to P = 15, the
  // P-templated kernel (its direct filter is the faster one there).
  if (P <= (box ? 9 : kMaxP) && R <= kMaxR) {
    kind = PATH_FAST;
    TH = tile_height(P);
    return PNP_OK;
  }
  if (P > kGenMaxP)
    return fail(PNP_EINVAL, "patch_side > " + std::to_string(kGenMaxP) + " not supported");
  auto bytes = [&](int th, bool sym, int kg) {
    return (size_t)gen_smem(th, P, R, 2, sym, kg).total * 4;
  };
  const size_t two = 113 * 1024, one = 227 * 1024;  // 2 / 1 CTAs per SM
  // (tile height, batch): taller tiles amortize the patch halo, bigger
  // batches the barriers; two resident CTAs per SM first
  const int cand[][2] = {{32, 4}, {16, 4}, {32, 2}, {16, 2}, {8, 4}, {8, 2}};
  for (size_t lim : {two, one})
    for (auto& c : cand)
      if (bytes(c[0], true, c[1]) <= lim) {
        kind = PATH_GEN_SYM;
        TH = c[0];
        KG = c[1];
        return PNP_OK;
      }
  for (auto& c : cand)
    if (bytes(c[0], false, c[1]) <= one) {
      kind = PATH_GEN_NEAR;
      TH = c[0];
      KG = c[1];
      return PNP_OK;
    }
  return fail(PNP_EINVAL, "patch / window too large for shared memory");
}

// The general kernel's offset groups: ranges of dy values, balanced by offset
// count, about 4 CTAs per SM over the whole grid.
static void gen_groups(int R, bool sym, int KG, int ntiles, std::vector<int>& grp) {
  // balanced by offset count over the dy values; a group's last batch of KG
  // may be partial (its missing offsets are masked in the kernel)
  (void)KG;
  const int ndy = sym ? R + 1 : 2 * R + 1;
  std::vector<long long> cnt(ndy);
  long long total = 0;
  for (int i = 0; i < ndy; ++i) {
    const int dy = sym ? i : i - R;
    cnt[i] = sym ? (dy == 0 ? R : 2 * R + 1) : (dy == 0 ? 2 * R : 2 * R + 1);
    total += cnt[i];
  }
  int ng = (4 * 148 + ntiles / 2) / (ntiles > 0 ? ntiles : 1);
  ng = std::max(1, std::min(std::min(ng, ndy), kMaxGroups));
  grp.assign(1, 0);
  long long acc = 0;
  int k = 1;
  for (int i = 0; i < ndy; ++i) {
    acc += cnt[i];
    if (k < ng && acc * ng >= total * k && i + 1 < ndy) {
      grp.push_back(i + 1);
      ++k;
    }
  }
  grp.push_back(ndy);
}

static int check_geometry(int B, int H, int W, int R, int P, double bw) {
  if (B < 1) return fail(PNP_EINVAL, "batch must be >= 1");
  if (H < 1 || W < 1) return fail(PNP_EINVAL, "image must be at least 1x1");
  if (P < 1 || P % 2 == 0)
    return fail(PNP_EINVAL, "patch_side must be odd and >= 1, got " + std::to_string(P));
  if (P > kGenMaxP)
    return fail(PNP_EINVAL, "patch_side > " + std::to_string(kGenMaxP) + " not supported");
  if (R < 1) return fail(PNP_EINVAL, "window_radius must be >= 1, got " + std::to_string(R));
  if (!(bw > 0)) return fail(PNP_EINVAL, "bandwidth must be > 0");
  const int margin = R + (P - 1) / 2;
  const int mn = H < W ? H : W;
  if (margin > mn)
    return fail(PNP_EINVAL, "margin " + std::to_string(margin) + " exceeds min image extent " +
                                std::to_string(mn));
  return PNP_OK;
}

// Equal taps select the box patch distance (the reference's own; general
// kernel with running sums), anything else the separable Gaussian filter.
static bool taps_box(const float* taps, int P) {
  for (int i = 1; i < P; ++i)
    if (taps[i] != taps[0]) return false;
  return true;
}

static int groups_for(int Hg, int W, int R, int P, bool box) {
  int kind = 0, TH = 0, KG = 0;
  if (choose_path(R, P, box, kind, TH, KG)) return -1;
  const int ntiles = ((W + kTW - 1) / kTW) * ((Hg + TH - 1) / TH);
  if (kind != PATH_FAST) {
    std::vector<int> grp;
    gen_groups(R, kind == PATH_GEN_SYM, KG, ntiles, grp);
    return (int)grp.size() - 1;
  }
  int nch = 0;
  for (int dx = -R; dx <= R; ++dx) nch += (R - (dx > 0 ? 0 : 1) + kKY) / kKY;
  return pick_groups(ntiles, nch);
}

static int make_geom(pnp_ctx* ctx, int B, int Hg, int W, int R, int P, bool box, Geom& g) {
  g.B = B;
  g.Hg = Hg;
  g.W = W;
  g.R = R;
  g.P = P;
  g.box = box;
  int rc = choose_path(R, P, box, g.kind, g.TH, g.KG);
  if (rc) return rc;
  g.Rb = g.kind == PATH_GEN_NEAR ? 0 : R;
  g.tiles_x = (W + kTW - 1) / kTW;
  g.tiles_y = (Hg + g.TH - 1) / g.TH;
  g.chunks = g.chunks_nohat = nullptr;
  g.ltab = nullptr;
  const int ntiles = g.tiles_x * g.tiles_y;
  if (g.kind != PATH_FAST) {
    std::vector<int> grp;
    gen_groups(R, g.kind == PATH_GEN_SYM, g.KG, ntiles, grp);
    g.NG = g.NP = (int)grp.size() - 1;
    g.nchunks = 0;
    auto key = std::make_tuple(R, g.NG * 8 + g.KG, g.kind);
    auto it = ctx->tables.find(key);
    if (it == ctx->tables.end()) {
      pnp_ctx::Tables t;
      t.grp = grp;
      // log2 of the separable hat (denoise.py:199-201) per offset, in double,
      // rounded once
      const int n = 2 * R + 1;
      std::vector<float> lt((size_t)n * n);
      const double sc = R + 1.0;
      for (int dy = -R; dy <= R; ++dy)
        for (int dx = -R; dx <= R; ++dx)
          lt[(size_t)(dy + R) * n + dx + R] =
              (float)(log2(1.0 - fabs((double)dy) / sc) + log2(1.0 - fabs((double)dx) / sc));
      if ((rc = t.ltab.ensure(lt.size() * sizeof(float)))) return rc;
      PNP_CUDA(cudaMemcpy(t.ltab.ptr, lt.data(), lt.size() * sizeof(float),
                          cudaMemcpyHostToDevice));
      it = ctx->tables.emplace(key, std::move(t)).first;
    }
    g.grp = it->second.grp.data();
    g.ltab = it->second.ltab.as<float>();
    return PNP_OK;
  }
  std::vector<Chunk> ch, ch0;
  build_chunks(R, true, ch);
  build_chunks(R, false, ch0);
  g.nchunks = (int)ch.size();
  g.NG = g.NP = pick_groups(ntiles, g.nchunks);
  auto key = std::make_tuple(R, g.NG, g.kind);
  auto it = ctx->tables.find(key);
  if (it == ctx->tables.end()) {
    if (g.NG > kMaxGroups) return fail(PNP_EINVAL, "too many offset groups");
    pnp_ctx::Tables t;
    const size_t cb = ch.size() * sizeof(Chunk);
    t.hat.resize(cb);
    t.nohat.resize(cb);
    memcpy(t.hat.data(), ch.data(), cb);
    memcpy(t.nohat.data(), ch0.data(), cb);
    t.grp.resize(g.NG + 1);
    for (int i = 0; i <= g.NG; ++i) t.grp[i] = (int)((long long)i * g.nchunks / g.NG);
    it = ctx->tables.emplace(key, std::move(t)).first;
  }
  g.chunks = reinterpret_cast<const Chunk*>(it->second.hat.data());
  g.chunks_nohat = reinterpret_cast<const Chunk*>(it->second.nohat.data());
  g.grp = it->second.grp.data();
  return PNP_OK;
}

static size_t block_floats(const Geom& g, int C) {
  return (size_t)C * (g.TH + g.Rb) * (kTW + 2 * g.Rb);
}

static size_t partial_floats(const Geom& g, int ntr, int C) {
  return (size_t)g.B * ntr * g.NP * g.tiles_x * block_floats(g, C);
}

// Stream-ordered allocation from the device's default memory pool, which is
// told once to keep freed memory (release threshold = max) so that frozen
// guides created and destroyed by successive ADMM runs reuse it without
// cudaMalloc / cudaFree (both can stall the host for milliseconds and the
// latter synchronizes the device).
static cudaError_t pool_alloc(pnp_ctx* ctx, void** p, size_t bytes) {
  static std::once_flag once[64];
  const int dev = ctx->device;
  if (dev >= 0 && dev < 64)
    std::call_once(once[dev], [dev] {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
    });
  return cudaMallocAsync(p, bytes, ctx->stream);
}

// Device counter of the last-CTA reductions: allocated and zeroed once; every
// kernel that uses it leaves it at zero.
static int ensure_counter(pnp_ctx* ctx, int n = 1) {
  if (ctx->counter.bytes >= (size_t)n * sizeof(unsigned)) return PNP_OK;
  int rc = ctx->counter.ensure((size_t)n * sizeof(unsigned));
  if (rc) return rc;
  PNP_CUDA(cudaMemsetAsync(ctx->counter.ptr, 0, ctx->counter.bytes, ctx->stream));
  return PNP_OK;
}

// Fixup variant: one thread per pixel when there are many partial groups or
// too few tiles to fill the GPU with one CTA per tile (same sums either way).
static bool fixup_px(const Geom& g) {
  // (32-bit offsets inside one image's partial array; a pixel covered by at
  // most 3 tile rows and one side column of blocks)
  if ((double)g.tiles_y * g.NP * g.tiles_x * 2 * (g.TH + g.Rb) * (kTW + 2 * g.Rb) >= 4294967295.0)
    return false;
  if (g.Rb > 32 || (g.Rb + g.TH - 1) / g.TH > 2) return false;
  return g.NP > 2 || (long long)g.B * g.tiles_x * g.tiles_y < 2 * 148;
}

template <int RB, int C, int MODE>
static cudaError_t launch_sweep_rc(const SweepArgs& a, const HostTab& t, int P, dim3 grid,
                                   cudaStream_t st, const CUtensorMap& m) {
  switch (P) {
    case 1: return launch_sweep<1, RB, C, MODE>(a, t, grid, st, m);
    case 3: return launch_sweep<3, RB, C, MODE>(a, t, grid, st, m);
    case 5: return launch_sweep<5, RB, C, MODE>(a, t, grid, st, m);
    case 7: return launch_sweep<7, RB, C, MODE>(a, t, grid, st, m);
    case 9: return launch_sweep<9, RB, C, MODE>(a, t, grid, st, m);
    case 11: return launch_sweep<11, RB, C, MODE>(a, t, grid, st, m);
    case 13: return launch_sweep<13, RB, C, MODE>(a, t, grid, st, m);
    case 15: return launch_sweep<15, RB, C, MODE>(a, t, grid, st, m);
  }
  return cudaErrorInvalidValue;
}

template <int C, int MODE>
static cudaError_t launch_sweep_cm(const SweepArgs& a, const HostTab& t, const Geom& g, dim3 grid,
                                   cudaStream_t st, const CUtensorMap& m) {
  switch (r_bucket(g.R)) {
    case 5: return launch_sweep_rc<5, C, MODE>(a, t, g.P, grid, st, m);
    case 10: return launch_sweep_rc<10, C, MODE>(a, t, g.P, grid, st, m);
    case 16: return launch_sweep_rc<16, C, MODE>(a, t, g.P, grid, st, m);
    default: return launch_sweep_rc<32, C, MODE>(a, t, g.P, grid, st, m);
  }
}

// The guide as a 3-D TMA tensor (W x buf_rows x B fp32) with the sweep
// tile's box (GCB x GR x 1) for the recompute / store sweeps' staging; false
// (no TMA: every tile gathers) when the layout does not allow it (row pitch
// not a multiple of 16 bytes, unaligned base) or the driver entry point is
// unavailable.
static bool guide_tmap(const Geom& g, const Window& w, const float* guide, CUtensorMap* m) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return (EncodeFn) nullptr;
    }
    return reinterpret_cast<EncodeFn>(fn);
  }();
  if (!encode || g.W % 4 || ((uintptr_t)guide & 15)) return false;
  const int p = (g.P - 1) / 2, RB = r_bucket(g.R);
  const int GC = kTW + 2 * (RB + p), GCB = (GC + 6) & ~3, GR = 33 + RB;  // Cfg::GCB
  if (GCB > 256 || GR > 256 || GCB > g.W || GR > w.buf_rows) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)g.W, (cuuint64_t)w.buf_rows, (cuuint64_t)g.B};
  const cuuint64_t strides[2] = {(cuuint64_t)g.W * 4, (cuuint64_t)w.buf_rows * g.W * 4};
  const cuuint32_t box[3] = {(cuuint32_t)GCB, (cuuint32_t)GR, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(guide), dims, strides,
                box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Half-window offsets (one k-cache plane of TH x 64 floats each per tile).
static int half_window(int R) { return 2 * R * R + 2 * R; }

// Floats of a k cache covering `ntr` tile rows of a (batched) image: exactly
// one float per pixel (of the tile grid) and half-window offset.
static size_t kcache_floats(const Geom& g, int ntr) {
  return (size_t)half_window(g.R) * g.B * ((size_t)ntr * g.TH) * (g.tiles_x * kTW);
}

// Decide whether the k cache of this call fits (ctx budget, free HBM).
static bool kcache_fits(pnp_ctx* ctx, size_t floats, size_t already) {
  if (ctx->cache_limit == 0) return false;
  const size_t bytes = floats * sizeof(float);
  if (bytes > ctx->cache_limit) return false;
  if (bytes <= already) return true;
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return false;
  return bytes - already + ((size_t)4 << 30) <= free_b;  // keep 4 GiB headroom
}

// Tile rows (counted from the top of every image) whose k cache fits: all of
// them when the whole cache fits, else as many as the budget allows (the
// rest is recomputed -- same bits either way), 0 below 1/8 of the image.
static int kcache_rows(pnp_ctx* ctx, const Geom& g, size_t already) {
  if (ctx->cache_limit == 0 || g.kind == PATH_GEN_NEAR) return 0;
  if (kcache_fits(ctx, kcache_floats(g, g.tiles_y), already)) return g.tiles_y;
  if (g.kind != PATH_FAST) return 0;  // the general sweep caches all tile rows or none
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return 0;
  const size_t head = (size_t)4 << 30, row_b = kcache_floats(g, 1) * sizeof(float);
  size_t budget = free_b + already > head ? free_b + already - head : 0;
  if (budget > ctx->cache_limit) budget = ctx->cache_limit;
  const int rows = (int)(budget / row_b);
  return rows * 8 >= g.tiles_y ? (rows < g.tiles_y ? rows : g.tiles_y) : 0;
}

// The k cache of one adaptive call: the caller-bound buffer (as many tile
// rows as fit), else a stream-ordered pool allocation released by
// kcache_release at the end of the call.  rows = 0: recompute (same bits).
static int kcache_acquire(pnp_ctx* ctx, const Geom& g, float** kc, int* rows) {
  *kc = nullptr;
  *rows = 0;
  ctx->kc_call = nullptr;
  ctx->kc_call_pooled = false;
  if (ctx->cache_limit == 0 || g.kind == PATH_GEN_NEAR) return PNP_OK;
  const size_t row_b = kcache_floats(g, 1) * sizeof(float);
  if (ctx->kc_ext) {
    size_t budget = ctx->kc_ext_bytes < ctx->cache_limit ? ctx->kc_ext_bytes : ctx->cache_limit;
    int r = (int)std::min<size_t>(budget / row_b, (size_t)g.tiles_y);
    if (r * 8 < g.tiles_y || (g.kind != PATH_FAST && r < g.tiles_y)) r = 0;
    *kc = r ? static_cast<float*>(ctx->kc_ext) : nullptr;
    *rows = r;
    ctx->kc_call = *kc;
    return PNP_OK;
  }
  const int r = kcache_rows(ctx, g, 0);
  if (r <= 0) return PNP_OK;
  void* p = nullptr;
  if (pool_alloc(ctx, &p, (size_t)r * row_b) != cudaSuccess) {
    cudaGetLastError();
    return PNP_OK;  // not fatal: recompute
  }
  *kc = static_cast<float*>(p);
  *rows = r;
  ctx->kc_call = *kc;
  ctx->kc_call_pooled = true;
  return PNP_OK;
}

static void kcache_release(pnp_ctx* ctx) {
  if (ctx->kc_call && ctx->kc_call_pooled) cudaFreeAsync(ctx->kc_call, ctx->stream);
  ctx->kc_call = nullptr;
  ctx->kc_call_pooled = false;
}

static int run_sweep_gen(pnp_ctx* ctx, const Geom& g, const Window& w, int C, const float* guide,
                         ChanSpec c0, ChanSpec c1, const float* taps, double bw, bool use_hat,
                         float* partial, int mode, float* kcache) {
  GenArgs a;
  memset(&a, 0, sizeof(a));
  if (mode != MODE_RECOMPUTE && (!kcache || g.kind != PATH_GEN_SYM))
    return fail(PNP_EINVAL, "k cache missing (or full-window general sweep)");
  a.kcache = mode != MODE_RECOMPUTE ? kcache : nullptr;
  a.kcache_floats = (long long)kcache_floats(g, w.ntr);
  a.guide = guide;
  a.ch[0] = c0;
  a.ch[1] = c1;
  a.partial = partial;
  a.ltab = use_hat ? g.ltab : nullptr;
  a.Hg = g.Hg;
  a.W = g.W;
  a.R = g.R;
  a.P = g.P;
  a.TH = g.TH;
  a.buf_r0 = w.buf_r0;
  a.buf_rows = w.buf_rows;
  a.tr0 = w.tr0;
  a.tiles_x = g.tiles_x;
  a.part_off = w.part_off;
  a.part_ntr = w.part_ntr;
  // k = exp(-SSD / (2 P^2 bw^2)) (box, denoise.py:186,194) = ex2(cv * SSD);
  // Gaussian: exp(-sum w_a w_b D / (2 bw^2)) with the scale folded into w_a
  const double scale = -1.0 / (2.0 * log(2.0) * bw * bw);
  a.cv = (float)(scale / ((double)g.P * g.P));
  for (int i = 0; i < g.P; ++i) {
    a.taps_h[i] = taps[i];
    a.taps_v[i] = (float)(scale * (double)taps[i]);
  }
  for (int i = 0; i <= g.NG; ++i) a.grp[i] = g.grp[i];
  a.partial_floats = partial == ctx->partial.ptr ? (long long)(ctx->partial.bytes / sizeof(float))
                                                 : LLONG_MAX;
  dim3 grid(w.ntr * g.tiles_x, g.NG, g.B);
  ProfScope prof(ctx, mode == MODE_CACHED ? PROF_SWEEP_CACHED : PROF_SWEEP);
  cudaError_t e =
      launch_generic(a, C, g.box, g.kind == PATH_GEN_SYM, g.KG, mode, grid, ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "dsg_generic_kernel");
  return PNP_OK;
}

static int run_sweep(pnp_ctx* ctx, const Geom& g, const Window& w, int C, const float* guide,
                     ChanSpec c0, ChanSpec c1, const float* taps, double bw, bool use_hat,
                     float* partial, int mode = MODE_RECOMPUTE, float* kcache = nullptr) {
  if (w.ntr <= 0) return PNP_OK;
  if (g.kind != PATH_FAST) {
    if (!kcache) mode = MODE_RECOMPUTE;
    return run_sweep_gen(ctx, g, w, C, guide, c0, c1, taps, bw, use_hat, partial, mode, kcache);
  }
  SweepArgs a;
  memset(&a, 0, sizeof(a));
  a.guide = guide;
  a.ch[0] = c0;
  a.ch[1] = c1;
  a.partial = partial;
  const HostTab tab{use_hat ? g.chunks : g.chunks_nohat, g.nchunks, g.grp, g.NG};
  a.Hg = g.Hg;
  a.W = g.W;
  a.R = g.R;
  a.buf_r0 = w.buf_r0;
  a.buf_rows = w.buf_rows;
  a.tr0 = w.tr0;
  a.tiles_x = g.tiles_x;
  a.part_off = w.part_off;
  a.part_ntr = w.part_ntr;
  a.kcache = kcache;
  a.kc_tile = (long long)half_window(g.R) * g.TH * kTW;
  a.kc_img = (long long)w.ntr * g.tiles_x * a.kc_tile;
  a.partial_floats = partial == ctx->partial.ptr ? (long long)(ctx->partial.bytes / sizeof(float))
                                                 : LLONG_MAX;
  a.kcache_floats = kcache ? (long long)g.B * a.kc_img : 0;
  // k = exp(-sum w_a w_b D / (2 bw^2)) = ex2(-log2(e)/(2 bw^2) * ...)
  const double scale = -1.0 / (2.0 * log(2.0) * bw * bw);
  for (int i = 0; i < g.P; ++i) {
    a.taps_h[i] = taps[i];
    a.taps_v[i] = (float)(scale * (double)taps[i]);
  }
  dim3 grid(w.ntr * g.tiles_x, g.NG, g.B);
  CUtensorMap gm;
  memset(&gm, 0, sizeof(gm));
  static const bool no_tma = getenv("PNP_NO_TMA") != nullptr;  // A/B switch
  a.tma = (!no_tma && mode != MODE_CACHED && guide_tmap(g, w, guide, &gm)) ? 1 : 0;
  ProfScope prof(ctx, mode == MODE_CACHED ? PROF_SWEEP_CACHED : PROF_SWEEP);
  cudaError_t e = cudaErrorInvalidValue;
  if (mode != MODE_RECOMPUTE && !kcache) return fail(PNP_EINVAL, "k cache missing");
  cudaStream_t st = ctx->stream;
  if (C == 1) {
    if (mode == MODE_RECOMPUTE) e = launch_sweep_cm<1, MODE_RECOMPUTE>(a, tab, g, grid, st, gm);
    else if (mode == MODE_STORE) e = launch_sweep_cm<1, MODE_STORE>(a, tab, g, grid, st, gm);
    else e = launch_sweep_cm<1, MODE_CACHED>(a, tab, g, grid, st, gm);
  } else {
    if (mode == MODE_RECOMPUTE) e = launch_sweep_cm<2, MODE_RECOMPUTE>(a, tab, g, grid, st, gm);
    else if (mode == MODE_CACHED) e = launch_sweep_cm<2, MODE_CACHED>(a, tab, g, grid, st, gm);
  }
  if (e != cudaSuccess) return cuda_fail(e, "dsg_sweep_kernel");
  return PNP_OK;
}

// A full-window sweep with the k cache covering tile rows [0, kc_rows):
// those run in `kmode` (STORE or CACHED) on the cache, the rest recompute.
static int run_sweep_kc(pnp_ctx* ctx, const Geom& g, int C, const float* guide, ChanSpec c0,
                        ChanSpec c1, const float* taps, double bw, float* partial, int kmode,
                        float* kc, int kc_rows) {
  const Window w = full_window(g);
  if (!kc || kc_rows <= 0 || (g.kind != PATH_FAST && kc_rows < g.tiles_y))
    return run_sweep(ctx, g, w, C, guide, c0, c1, taps, bw, true, partial, MODE_RECOMPUTE);
  if (kc_rows >= g.tiles_y)
    return run_sweep(ctx, g, w, C, guide, c0, c1, taps, bw, true, partial, kmode, kc);
  const Window wa{0, g.Hg, 0, kc_rows, 0, 0, g.tiles_y, 0, g.Hg};
  const Window wb{0, g.Hg, kc_rows, g.tiles_y - kc_rows, 0, kc_rows, g.tiles_y, 0, g.Hg};
  int rc = run_sweep(ctx, g, wa, C, guide, c0, c1, taps, bw, true, partial, kmode, kc);
  if (rc) return rc;
  return run_sweep(ctx, g, wb, C, guide, c0, c1, taps, bw, true, partial, MODE_RECOMPUTE);
}

template <int MODE>
static int run_fixup(pnp_ctx* ctx, const Geom& g, const Window& w, int C, const float* partial,
                     const FixIO& io) {
  if (w.nrows <= 0) return PNP_OK;
  FixGeo f;
  f.partial = partial;
  f.Hg = g.Hg;
  f.W = g.W;
  f.R = g.Rb;
  f.TH = g.TH;
  f.tiles_x = g.tiles_x;
  f.NP = g.NP;
  f.C = C;
  f.part_tr0 = w.part_tr0;
  f.part_ntr = w.part_ntr;
  f.y0 = w.y0;
  f.nrows = w.nrows;
  f.buf_r0 = w.buf_r0;
  f.buf_rows = w.buf_rows;
  const int tr_first = w.y0 / g.TH, tr_last = (w.y0 + w.nrows - 1) / g.TH;
  ProfScope prof(ctx, PROF_FIXUP);
  if (!fixup_px(g)) {  // same summation order either way
    dim3 grid(g.tiles_x, tr_last - tr_first + 1, g.B);
    PNP_CUDA(launch_pdl(dsg_fixup_tile_kernel<MODE>, grid, dim3(256), 0, ctx->stream, f, io));
  } else {
    dim3 grid(g.tiles_x, (tr_last - tr_first + 1) * ((g.TH + 3) / 4), g.B);
    PNP_CUDA(launch_pdl(dsg_fixup_px_kernel<MODE>, grid, dim3(256), 0, ctx->stream, f, io));
  }
  PNP_LAUNCH_CHECK("dsg_fixup_kernel");
  return PNP_OK;
}

static int run_finalize(pnp_ctx* ctx, const Geom& g, const Window& w, const float* kx,
                        const float* d, const unsigned* mbits, const float* x, float* out,
                        float* alpha_out) {
  const size_t npix = (size_t)w.nrows * g.W;
  ProfScope prof(ctx, PROF_FIXUP);
  auto a16 = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  if (g.W % 4 == 0 && a16(kx) && a16(d) && a16(x) && a16(out)) {
    const size_t n4 = npix / 4;
    const unsigned per_img = (unsigned)std::min<size_t>((n4 + 255) / 256,
                                                        (size_t)ctx->sms * 8 / g.B + 1);
    PNP_CUDA(launch_pdl(dsg_finalize4_kernel, dim3(per_img, g.B), dim3(256), 0, ctx->stream, kx,
                        d, mbits, x, out, alpha_out, w.y0, w.nrows, g.W, w.buf_r0, w.buf_rows));
    return PNP_OK;
  }
  dim3 grid((unsigned)((npix + 255) / 256), g.B);
  PNP_CUDA(launch_pdl(dsg_finalize_kernel, grid, dim3(256), 0, ctx->stream, kx, d, mbits, x, out,
                      alpha_out, w.y0, w.nrows, g.W, w.buf_r0, w.buf_rows));
  PNP_LAUNCH_CHECK("dsg_finalize_kernel");
  return PNP_OK;
}

static int ensure_planes(pnp_ctx* ctx, size_t n) {
  int rc;
  if ((rc = ctx->rs.ensure(n * sizeof(float)))) return rc;
  if ((rc = ctx->kx.ensure(n * sizeof(float)))) return rc;
  if ((rc = ctx->d.ensure(n * sizeof(float)))) return rc;
  return PNP_OK;
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

// sweep A + fixup: g -> rs (guide-only; shared by adaptive and freeze)
static int mass_and_rs(pnp_ctx* ctx, const Geom& g, const float* guide, const float* taps,
                       double bw, float* rs, float* kcache = nullptr, int kc_rows = 0) {
  const Window w = full_window(g);
  float* part = ctx->partial.as<float>();
  int rc = run_sweep_kc(ctx, g, 1, guide, ChanSpec{nullptr, nullptr}, ChanSpec{nullptr, nullptr},
                        taps, bw, part, MODE_STORE, kcache, kc_rows);
  if (rc) return rc;
  FixIO io{};
  io.rs = rs;
  return run_fixup<FIX_RS>(ctx, g, w, 1, part, io);
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
  PNP_CUDA(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device));
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
  kcache_release(ctx);
  ctx->cg.release();
  ctx->counter.release();
  for (auto& kv : ctx->tables) kv.second.ltab.release();
  for (auto& sl : ctx->slots) {
    cudaEventDestroy(sl.a);
    cudaEventDestroy(sl.b);
  }
  for (cudaEvent_t e : ctx->iter_events) cudaEventDestroy(e);
  if (ctx->ev_x) cudaEventDestroy(ctx->ev_x);
  if (ctx->ev_g) cudaEventDestroy(ctx->ev_g);
  if (ctx->ev_switch) cudaEventDestroy(ctx->ev_switch);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  ctx->admm_r.release();
  ctx->admm_part.release();
  ctx->admm_g.release();
  delete ctx;
  return PNP_OK;
}

int pnp_ctx_set_stream(pnp_ctx* ctx, void* stream) {
  if (!ctx) return fail(PNP_EINVAL, "ctx is null");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (s != ctx->stream) {
    // Calls are stream-ordered and share the context's scratch: a call issued
    // on the new stream must not start before the context's work queued on
    // the old one (two host streams driving one context would race on it).
    // Skipped when either stream is being captured into a graph: the capture
    // orders its own work, and an event from outside it cannot be joined.
    cudaStreamCaptureStatus c0 = cudaStreamCaptureStatusNone, c1 = cudaStreamCaptureStatusNone;
    const bool ok = cudaStreamIsCapturing(ctx->stream, &c0) == cudaSuccess &&
                    cudaStreamIsCapturing(s, &c1) == cudaSuccess;
    if (!ok) (void)cudaGetLastError();
    if (ok && c0 == cudaStreamCaptureStatusNone && c1 == cudaStreamCaptureStatusNone) {
      PNP_CUDA(cudaSetDevice(ctx->device));
      if (!ctx->ev_switch)
        PNP_CUDA(cudaEventCreateWithFlags(&ctx->ev_switch, cudaEventDisableTiming));
      PNP_CUDA(cudaEventRecord(ctx->ev_switch, ctx->stream));
      PNP_CUDA(cudaStreamWaitEvent(s, ctx->ev_switch, 0));
    }
    ctx->stream = s;
  }
  return PNP_OK;
}

int pnp_ctx_synchronize(pnp_ctx* ctx) {
  if (!ctx) return fail(PNP_EINVAL, "ctx is null");
  PNP_CUDA(cudaStreamSynchronize(ctx->stream));
  return PNP_OK;
}

int pnp_ctx_set_cache_limit(pnp_ctx* ctx, int64_t bytes) {
  if (!ctx) return fail(PNP_EINVAL, "ctx is null");
  ctx->cache_limit = bytes < 0 ? (size_t)-1 : (size_t)bytes;
  return PNP_OK;
}

int pnp_ctx_bind_kcache(pnp_ctx* ctx, void* ptr, int64_t bytes) {
  if (!ctx) return fail(PNP_EINVAL, "ctx is null");
  if (ptr && bytes > 0) {
    ctx->kc_ext = ptr;
    ctx->kc_ext_bytes = (size_t)bytes;
  } else {
    ctx->kc_ext = nullptr;
    ctx->kc_ext_bytes = 0;
  }
  return PNP_OK;
}

int pnp_ctx_trim(pnp_ctx* ctx) {
  if (!ctx) return fail(PNP_EINVAL, "ctx is null");
  PNP_CUDA(cudaSetDevice(ctx->device));
  PNP_CUDA(cudaStreamSynchronize(ctx->stream));
  cudaMemPool_t pool;
  PNP_CUDA(cudaDeviceGetDefaultMemPool(&pool, ctx->device));
  PNP_CUDA(cudaMemPoolTrimTo(pool, 0));
  return PNP_OK;
}

int pnp_frozen_cached(const pnp_frozen* fz) { return fz && fz->kcache ? 1 : 0; }

int pnp_ctx_profile(pnp_ctx* ctx, int enable) {
  if (!ctx) return fail(PNP_EINVAL, "ctx is null");
  ctx->prof = enable != 0;
  ctx->nslots = 0;
  return PNP_OK;
}

int pnp_ctx_profile_read(pnp_ctx* ctx, double* ms, int* launches) {
  if (!ctx || !ms || !launches) return fail(PNP_EINVAL, "null argument");
  for (int c = 0; c < PROF_NCAT; ++c) {
    ms[c] = 0.0;
    launches[c] = 0;
  }
  PNP_CUDA(cudaStreamSynchronize(ctx->stream));
  for (size_t i = 0; i < ctx->nslots; ++i) {
    float t = 0.f;
    PNP_CUDA(cudaEventElapsedTime(&t, ctx->slots[i].a, ctx->slots[i].b));
    ms[ctx->slots[i].cat] += t;
    launches[ctx->slots[i].cat] += 1;
  }
  ctx->nslots = 0;
  return PNP_OK;
}

int pnp_ctx_reserve(pnp_ctx* ctx, int batch, int H, int W, int R, int P, int box) {
  if (!ctx) return fail(PNP_EINVAL, "ctx is null");
  int rc = check_geometry(batch, H, W, R, P, 1.0);
  if (rc) return rc;
  PNP_CUDA(cudaSetDevice(ctx->device));
  Geom g;
  if ((rc = make_geom(ctx, batch, H, W, R, P, box != 0, g))) return rc;
  if ((rc = ctx->partial.ensure(partial_floats(g, g.tiles_y, 2) * sizeof(float)))) return rc;
  if ((rc = ensure_planes(ctx, (size_t)batch * H * W))) return rc;
  if ((rc = ctx->mbits.ensure(batch * sizeof(unsigned)))) return rc;
  return PNP_OK;
}

int pnp_dsg_denoise(pnp_ctx* ctx, const float* x, const float* guide, float* out, int batch,
                    int H, int W, int R, int P, const float* taps, double bandwidth,
                    float* d_out, float* alpha_out) {
  Nvtx range("dsg_denoise");
  if (!ctx || !x || !out) return fail(PNP_EINVAL, "null argument");
  int rc = check_geometry(batch, H, W, R, P, bandwidth);
  if (rc) return rc;
  if ((rc = validate_taps(taps, P))) return rc;
  if (!guide) guide = x;
  PNP_CUDA(cudaSetDevice(ctx->device));
  Geom g;
  if ((rc = make_geom(ctx, batch, H, W, R, P, taps_box(taps, P), g))) return rc;
  const size_t n = (size_t)batch * H * W;
  if ((rc = ensure_planes(ctx, n))) return rc;
  if ((rc = ctx->mbits.ensure(batch * sizeof(unsigned)))) return rc;
  if ((rc = ctx->partial.ensure(partial_floats(g, g.tiles_y, 2) * sizeof(float)))) return rc;
  float* rs = ctx->rs.as<float>();
  float* kx = ctx->kx.as<float>();
  float* d = d_out ? d_out : ctx->d.as<float>();
  float* part = ctx->partial.as<float>();
  const Window w = full_window(g);
  float* kc = nullptr;
  int kc_rows = 0;
  if ((rc = kcache_acquire(ctx, g, &kc, &kc_rows))) return rc;
  rc = mass_and_rs(ctx, g, guide, taps, bandwidth, rs, kc, kc_rows);
  if (!rc)
    rc = run_sweep_kc(ctx, g, 2, guide, ChanSpec{rs, x}, ChanSpec{rs, nullptr}, taps, bandwidth,
                      part, MODE_CACHED, kc, kc_rows);
  kcache_release(ctx);  // stream-ordered: after sweep B
  if (rc) return rc;
  PNP_CUDA(cudaMemsetAsync(ctx->mbits.ptr, 0, batch * sizeof(unsigned), ctx->stream));
  FixIO io{};
  io.rs = rs;
  io.kx = kx;
  io.d = d;
  io.mbits = ctx->mbits.as<unsigned>();
  if ((rc = run_fixup<FIX_KXD>(ctx, g, w, 2, part, io))) return rc;
  return run_finalize(ctx, g, w, kx, d, ctx->mbits.as<unsigned>(), x, out, alpha_out);
}

// Row bands of a single image for pnp_dsg_denoise_banded: band j sweeps tile
// rows [tile_end[j-1], tile_end[j]) and needs input rows [0, rows_needed[j]).
// The first bands ramp up (1/4, 1/4, 1/2, 3/4 of the others): the sweep starts
// as soon as a quarter band is uploaded, and the uploads (faster than the
// sweep per row) get ahead during the ramp (8192^2: sweep A of the numpy call
// ends ~1 ms earlier than with equal bands).
static void band_split(int H, int R, int P, int nbands, int* tile_end, int* rows_needed) {
  const int TH = tile_height(P), T = (H + TH - 1) / TH, p = (P - 1) / 2, RB = r_bucket(R);
  auto wt = [](int j) { return j < 2 ? 1 : j == 2 ? 2 : j == 3 ? 3 : 4; };  // quarters
  long long tot = 0;
  for (int j = 0; j < nbands; ++j) tot += wt(j);
  long long acc = 0;
  int prev = 0;
  for (int j = 0; j < nbands; ++j) {
    acc += wt(j);
    int tb = (int)(acc * T / tot);
    // at least one tile row per band, and room for the bands after it
    if (tb < prev + 1) tb = prev + 1;
    if (tb > T - (nbands - 1 - j)) tb = T - (nbands - 1 - j);
    prev = tb;
    tile_end[j] = tb;
    // the guide tile of tile row tb-1 reads rows up to (tb-1)*TH - p + 32 + RB
    const int need = (tb - 1) * TH - p + 33 + RB;
    rows_needed[j] = j == nbands - 1 ? H : (need < H ? need : H);
  }
}

int pnp_dsg_band_rows(int H, int W, int R, int P, int box, int nbands, int* tile_end,
                      int* rows_needed) {
  if (!tile_end || !rows_needed || nbands < 1) return fail(PNP_EINVAL, "bad arguments");
  int rc = check_geometry(1, H, W, R, P, 1.0);
  if (rc) return rc;
  int kind = 0, th = 0, kg = 0;
  if ((rc = choose_path(R, P, box != 0, kind, th, kg))) return rc;
  if (kind != PATH_FAST) return fail(PNP_EINVAL, "banded denoise needs the P-templated sweep");
  if (nbands > (H + tile_height(P) - 1) / tile_height(P))
    return fail(PNP_EINVAL, "more bands than tile rows");
  band_split(H, R, P, nbands, tile_end, rows_needed);
  return PNP_OK;
}

// Incremental banded denoise: band j's sweep A (tile rows [tile_end[j-1],
// tile_end[j])) is enqueued by pnp_dsg_band_sweep; the caller orders the
// context stream behind the upload of the rows it reads first.  Band 0 sizes
// the buffers and the k cache and pins the cached tile-row count for the
// rest of the call.  Same tiles, partial slots and k-cache runs as the
// one-launch sweep -> same bits.
int pnp_dsg_band_sweep(pnp_ctx* ctx, const float* x, int H, int W, int R, int P,
                       const float* taps, double bandwidth, int nbands, int j) {
  if (!ctx || !x || nbands < 1) return fail(PNP_EINVAL, "null argument");
  int rc = check_geometry(1, H, W, R, P, bandwidth);
  if (rc) return rc;
  if ((rc = validate_taps(taps, P))) return rc;
  if (j < 0 || j >= nbands) return fail(PNP_EINVAL, "band index out of range");
  if (j > 0 && ctx->band_next != j) return fail(PNP_EINVAL, "bands must be swept in order from 0");
  PNP_CUDA(cudaSetDevice(ctx->device));
  Geom g;
  if ((rc = make_geom(ctx, 1, H, W, R, P, taps_box(taps, P), g))) return rc;
  if (g.kind != PATH_FAST) return fail(PNP_EINVAL, "banded denoise needs the P-templated sweep");
  if (nbands > g.tiles_y) return fail(PNP_EINVAL, "more bands than tile rows");
  if (j == 0) {
    if ((rc = ensure_planes(ctx, (size_t)H * W))) return rc;
    if ((rc = ctx->mbits.ensure(sizeof(unsigned)))) return rc;
    if ((rc = ctx->partial.ensure(partial_floats(g, g.tiles_y, 2) * sizeof(float)))) return rc;
    kcache_release(ctx);  // an abandoned earlier banded call
    float* kc0 = nullptr;
    int kc_rows = 0;
    if ((rc = kcache_acquire(ctx, g, &kc0, &kc_rows))) return rc;
    ctx->band_kc_rows = kc_rows;
  }
  float* part = ctx->partial.as<float>();
  const int kc_rows = ctx->band_kc_rows;
  float* kc = kc_rows > 0 ? ctx->kc_call : nullptr;
  std::vector<int> tend(nbands), need(nbands);
  band_split(H, R, P, nbands, tend.data(), need.data());
  const size_t kc_row = (size_t)g.tiles_x * half_window(g.R) * g.TH * kTW;
  const int t0 = j ? tend[j - 1] : 0, t1 = tend[j];
  // cached tile rows [t0, min(t1, kc_rows)) store, the rest recompute
  const int tm = kc ? (t1 < kc_rows ? t1 : (t0 > kc_rows ? t0 : kc_rows)) : t0;
  ctx->band_next = -1;
  if (tm > t0) {
    Window wj{0, H, t0, tm - t0, 0, t0, g.tiles_y, 0, H};
    if ((rc = run_sweep(ctx, g, wj, 1, x, ChanSpec{nullptr, nullptr}, ChanSpec{nullptr, nullptr},
                        taps, bandwidth, true, part, MODE_STORE, kc + (size_t)t0 * kc_row)))
      return rc;
  }
  if (t1 > tm) {
    Window wj{0, H, tm, t1 - tm, 0, tm, g.tiles_y, 0, H};
    if ((rc = run_sweep(ctx, g, wj, 1, x, ChanSpec{nullptr, nullptr}, ChanSpec{nullptr, nullptr},
                        taps, bandwidth, true, part, MODE_RECOMPUTE)))
      return rc;
  }
  ctx->band_next = j + 1 < nbands ? j + 1 : nbands;
  ctx->band_count = nbands;
  return PNP_OK;
}

// The rest of a banded denoise once every band is swept: rs fixup, cached
// sweep B, Kx / d fixup, finalize.
int pnp_dsg_band_finish(pnp_ctx* ctx, const float* x, float* out, int H, int W, int R, int P,
                        const float* taps, double bandwidth) {
  if (!ctx || !x || !out) return fail(PNP_EINVAL, "null argument");
  int rc = check_geometry(1, H, W, R, P, bandwidth);
  if (rc) return rc;
  if ((rc = validate_taps(taps, P))) return rc;
  if (ctx->band_next < 0 || ctx->band_next != ctx->band_count)
    return fail(PNP_EINVAL, "pnp_dsg_band_finish before every band was swept");
  ctx->band_next = -1;
  PNP_CUDA(cudaSetDevice(ctx->device));
  Geom g;
  if ((rc = make_geom(ctx, 1, H, W, R, P, taps_box(taps, P), g))) return rc;
  float* rs = ctx->rs.as<float>();
  float* kx = ctx->kx.as<float>();
  float* d = ctx->d.as<float>();
  float* part = ctx->partial.as<float>();
  const int kc_rows = ctx->band_kc_rows;
  float* kc = kc_rows > 0 ? ctx->kc_call : nullptr;
  const Window w = full_window(g);
  {
    FixIO io{};
    io.rs = rs;
    if ((rc = run_fixup<FIX_RS>(ctx, g, w, 1, part, io))) return kcache_release(ctx), rc;
  }
  rc = run_sweep_kc(ctx, g, 2, x, ChanSpec{rs, x}, ChanSpec{rs, nullptr}, taps, bandwidth, part,
                    MODE_CACHED, kc, kc_rows);
  kcache_release(ctx);
  if (rc) return rc;
  PNP_CUDA(cudaMemsetAsync(ctx->mbits.ptr, 0, sizeof(unsigned), ctx->stream));
  FixIO io{};
  io.rs = rs;
  io.kx = kx;
  io.d = d;
  io.mbits = ctx->mbits.as<unsigned>();
  if ((rc = run_fixup<FIX_KXD>(ctx, g, w, 2, part, io))) return rc;
  return run_finalize(ctx, g, w, kx, d, ctx->mbits.as<unsigned>(), x, out, nullptr);
}

int pnp_dsg_denoise_banded(pnp_ctx* ctx, const float* x, float* out, int H, int W, int R, int P,
                           const float* taps, double bandwidth, int nbands,
                           void* const* events) {
  if (!ctx || !x || !out || !events || nbands < 1) return fail(PNP_EINVAL, "null argument");
  // sweep A band by band, each after its rows arrived
  for (int j = 0; j < nbands; ++j) {
    if (events[j]) PNP_CUDA(cudaStreamWaitEvent(ctx->stream, (cudaEvent_t)events[j], 0));
    int rc = pnp_dsg_band_sweep(ctx, x, H, W, R, P, taps, bandwidth, nbands, j);
    if (rc) return rc;
  }
  return pnp_dsg_band_finish(ctx, x, out, H, W, R, P, taps, bandwidth);
}

int pnp_dsg_freeze(pnp_ctx* ctx, const float* guide, int batch, int H, int W, int R, int P,
                   const float* taps, double bandwidth, pnp_frozen** out) {
  Nvtx range("dsg_freeze");
  if (!ctx || !guide || !out) return fail(PNP_EINVAL, "null argument");
  int rc = check_geometry(batch, H, W, R, P, bandwidth);
  if (rc) return rc;
  if ((rc = validate_taps(taps, P))) return rc;
  PNP_CUDA(cudaSetDevice(ctx->device));
  Geom g;
  if ((rc = make_geom(ctx, batch, H, W, R, P, taps_box(taps, P), g))) return rc;
  if ((rc = ctx->partial.ensure(partial_floats(g, g.tiles_y, 2) * sizeof(float)))) return rc;
  const size_t n = (size_t)batch * H * W;
  pnp_frozen* fz = new pnp_frozen();
  fz->device = ctx->device;
  fz->B = batch;
  fz->H = H;
  fz->W = W;
  fz->R = R;
  fz->P = P;
  fz->bw = bandwidth;
  fz->tiles_y = g.tiles_y;
  for (int i = 0; i < P; ++i) fz->taps[i] = taps[i];
  fz->stream = ctx->stream;
  cudaError_t e = pool_alloc(ctx, (void**)&fz->guide, n * sizeof(float));
  if (e == cudaSuccess) e = pool_alloc(ctx, (void**)&fz->rs, n * sizeof(float));
  if (e == cudaSuccess) e = pool_alloc(ctx, (void**)&fz->d, n * sizeof(float));
  if (e == cudaSuccess) e = pool_alloc(ctx, (void**)&fz->mv, 2 * batch * sizeof(float));
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
  fz->kc_stream = ctx->stream;
  if (ctx->kc_ext && ctx->cache_limit != 0 && g.kind != PATH_GEN_NEAR) {
    // caller-bound cache (torch memory on the Python side): as many tile
    // rows as it holds, none below 1/8 of them
    const size_t row_b = kcache_floats(g, 1) * sizeof(float);
    size_t budget = ctx->kc_ext_bytes < ctx->cache_limit ? ctx->kc_ext_bytes : ctx->cache_limit;
    int r = (int)std::min<size_t>(budget / row_b, (size_t)g.tiles_y);
    if (r * 8 < g.tiles_y || (g.kind != PATH_FAST && r < g.tiles_y)) r = 0;
    if (r > 0) {
      fz->kcache = static_cast<float*>(ctx->kc_ext);
      fz->kc_ext = true;
      fz->kc_rows = r;
      fz->kc_bytes = (size_t)r * row_b;
    }
  }
  const int kc_rows = fz->kc_ext ? 0 : kcache_rows(ctx, g, 0);
  if (kc_rows > 0) {
    e = pool_alloc(ctx, (void**)&fz->kcache, kcache_floats(g, kc_rows) * sizeof(float));
    if (e != cudaSuccess) {
      cudaGetLastError();
      fz->kcache = nullptr;  // not fatal: recompute instead
    } else {
      fz->kc_rows = kc_rows;
      fz->kc_bytes = kcache_floats(g, kc_rows) * sizeof(float);
    }
  }
  if ((rc = mass_and_rs(ctx, g, fz->guide, taps, bandwidth, fz->rs, fz->kcache, fz->kc_rows)))
    return bail(rc);
  const Window w = full_window(g);
  float* part = ctx->partial.as<float>();
  if ((rc = run_sweep_kc(ctx, g, 1, fz->guide, ChanSpec{fz->rs, nullptr},
                         ChanSpec{nullptr, nullptr}, taps, bandwidth, part, MODE_CACHED,
                         fz->kcache, fz->kc_rows)))
    return bail(rc);
  e = cudaMemsetAsync(ctx->mbits.ptr, 0, batch * sizeof(unsigned), ctx->stream);
  if (e != cudaSuccess) return bail(cuda_fail(e, "cudaMemsetAsync"));
  FixIO io{};
  io.rs = fz->rs;
  io.d = fz->d;
  io.mbits = ctx->mbits.as<unsigned>();
  if ((rc = run_fixup<FIX_D>(ctx, g, w, 1, part, io))) return bail(rc);
  e = launch_pdl(dsg_alpha_kernel, dim3((batch + 127) / 128), dim3(128), 0, ctx->stream,
                 ctx->mbits.as<unsigned>(), fz->mv, batch);
  if (e != cudaSuccess) return bail(cuda_fail(e, "dsg_alpha_kernel"));
  *out = fz;
  return PNP_OK;
}

int pnp_dsg_apply(pnp_ctx* ctx, const pnp_frozen* fz, const float* x, float* out) {
  Nvtx range("dsg_apply");
  if (fz && ctx) fz->stream = ctx->stream;
  if (!ctx || !fz || !x || !out) return fail(PNP_EINVAL, "null argument");
  if (fz->device != ctx->device) return fail(PNP_EINVAL, "handle belongs to another device");
  PNP_CUDA(cudaSetDevice(ctx->device));
  Geom g;
  int rc = make_geom(ctx, fz->B, fz->H, fz->W, fz->R, fz->P, taps_box(fz->taps, fz->P), g);
  if (rc) return rc;
  if ((rc = ctx->partial.ensure(partial_floats(g, g.tiles_y, 2) * sizeof(float)))) return rc;
  const Window w = full_window(g);
  float* part = ctx->partial.as<float>();
  if ((rc = run_sweep_kc(ctx, g, 1, fz->guide, ChanSpec{fz->rs, x}, ChanSpec{nullptr, nullptr},
                         fz->taps, fz->bw, part, MODE_CACHED, fz->kcache, fz->kc_rows)))
    return rc;
  FixIO io{};
  io.rs = fz->rs;
  io.d = fz->d;
  io.inv_m = fz->mv + fz->B;
  io.x = x;
  io.out = out;
  return run_fixup<FIX_APPLY>(ctx, g, w, 1, part, io);
}

int pnp_dsg_apply_admm(pnp_ctx* ctx, const pnp_frozen* fz, const float* z, float* v,
                       float* u, const float* x, const float* v_prev, const float* gt,
                       double rho, double* stats, int* flags) {
  return pnp::dsg_apply_admm_x(ctx, fz, z, v, u, x, v_prev, gt, rho, stats, flags, nullptr);
}

}  // extern "C"

namespace pnp {

int dsg_apply_admm_x(pnp_ctx* ctx, const pnp_frozen* fz, const float* z, float* v, float* u,
                     const float* x, const float* v_prev, const float* gt, double rho,
                     double* stats, int* flags, const AdmmXNext* xn) {
  if (fz && ctx) fz->stream = ctx->stream;
  if (!ctx || !fz || !z || !v || !u || !x || !stats || !flags)
    return fail(PNP_EINVAL, "null argument");
  if (fz->device != ctx->device) return fail(PNP_EINVAL, "handle belongs to another device");
  PNP_CUDA(cudaSetDevice(ctx->device));
  Geom g;
  int rc = make_geom(ctx, fz->B, fz->H, fz->W, fz->R, fz->P, taps_box(fz->taps, fz->P), g);
  if (rc) return rc;
  if ((rc = ctx->partial.ensure(partial_floats(g, g.tiles_y, 2) * sizeof(float)))) return rc;
  const Window w = full_window(g);
  const int rows = fixup_px(g) ? g.tiles_y * ((g.TH + 3) / 4) : g.tiles_y;
  const size_t nblk = (size_t)g.tiles_x * rows;
  if ((rc = ctx->stats.ensure((size_t)g.B * nblk * 3 * sizeof(double)))) return rc;
  float* part = ctx->partial.as<float>();
  if ((rc = run_sweep_kc(ctx, g, 1, fz->guide, ChanSpec{fz->rs, z}, ChanSpec{nullptr, nullptr},
                         fz->taps, fz->bw, part, MODE_CACHED, fz->kcache, fz->kc_rows)))
    return rc;
  FixIO io{};
  io.rs = fz->rs;
  io.d = fz->d;
  io.inv_m = fz->mv + fz->B;
  io.x = z;
  io.out = v;
  io.u = u;
  io.xa = x;
  io.vprev = v_prev;
  io.gt = gt;
  io.rho = rho;
  io.part3 = ctx->stats.as<double>();
  io.flags = flags;
  if ((rc = ensure_counter(ctx, g.B))) return rc;
  io.stats_out = stats;
  io.counter = ctx->counter.as<unsigned>();
  if (xn) {  // the next x-update fused in, once its gradient is ready
    if (!xn->grad || !xn->flags) return fail(PNP_EINVAL, "null argument");
    if (xn->ready) PNP_CUDA(cudaStreamWaitEvent(ctx->stream, xn->ready, 0));
    io.grad = xn->grad;
    io.mu = xn->mu;
    io.alpha = xn->alpha;
    io.lo = (float)xn->lo;
    io.hi = (float)xn->hi;
    io.xflags = xn->flags;
  }
  return run_fixup<FIX_APPLY_U>(ctx, g, w, 1, part, io);
}

}  // namespace pnp

extern "C" {

int pnp_frozen_destroy(pnp_frozen* fz) {
  if (!fz) return PNP_OK;
  cudaSetDevice(fz->device);
  if (fz->kc_ext && fz->kcache && fz->stream != fz->kc_stream) {
    // the caller frees the bound cache on the stream it was handed out on:
    // order that stream after the handle's last use
    cudaEvent_t ev;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess) {
      if (cudaEventRecord(ev, fz->stream) != cudaSuccess ||
          cudaStreamWaitEvent(fz->kc_stream, ev, 0) != cudaSuccess) {
        cudaGetLastError();
        cudaStreamSynchronize(fz->stream);
      }
      cudaEventDestroy(ev);
    } else {
      cudaGetLastError();
      cudaStreamSynchronize(fz->stream);
    }
  }
  for (void* p : {(void*)fz->guide, (void*)fz->rs, (void*)fz->d, (void*)fz->mv,
                  fz->kc_ext ? nullptr : (void*)fz->kcache})
    if (p && cudaFreeAsync(p, fz->stream) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(p);  // stream gone: synchronous free
    }
  delete fz;
  return PNP_OK;
}

int pnp_frozen_alpha(const pnp_frozen* fz, float* alpha_host) {
  if (!fz || !alpha_host) return fail(PNP_EINVAL, "null argument");
  PNP_CUDA(cudaSetDevice(fz->device));
  // mv is written on the handle's stream (which may be a non-blocking one)
  PNP_CUDA(cudaMemcpyAsync(alpha_host, fz->mv, fz->B * sizeof(float), cudaMemcpyDeviceToHost,
                           fz->stream));
  PNP_CUDA(cudaStreamSynchronize(fz->stream));
  return PNP_OK;
}

int pnp_frozen_export(pnp_ctx* ctx, const pnp_frozen* fz, float* guide_out, float* d_out) {
  if (!ctx || !fz) return fail(PNP_EINVAL, "null argument");
  fz->stream = ctx->stream;
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

int pnp_frozen_cache(const pnp_frozen* fz, int* rows_cached, int* tile_rows,
                     unsigned long long* bytes) {
  if (!fz) return fail(PNP_EINVAL, "null argument");
  if (rows_cached) *rows_cached = fz->kcache ? fz->kc_rows : 0;
  if (tile_rows) *tile_rows = fz->tiles_y;
  if (bytes) *bytes = fz->kcache ? (unsigned long long)fz->kc_bytes : 0ull;
  return PNP_OK;
}

int pnp_nlm_denoise(pnp_ctx* ctx, const float* x, const float* guide, float* out, int batch,
                    int H, int W, int R, int P, const float* taps, double bandwidth) {
  Nvtx range("nlm_denoise");
  if (!ctx || !x || !out) return fail(PNP_EINVAL, "null argument");
  int rc = check_geometry(batch, H, W, R, P, bandwidth);
  if (rc) return rc;
  if ((rc = validate_taps(taps, P))) return rc;
  if (!guide) guide = x;
  PNP_CUDA(cudaSetDevice(ctx->device));
  Geom g;
  if ((rc = make_geom(ctx, batch, H, W, R, P, taps_box(taps, P), g))) return rc;
  if ((rc = ctx->partial.ensure(partial_floats(g, g.tiles_y, 2) * sizeof(float)))) return rc;
  const Window w = full_window(g);
  float* part = ctx->partial.as<float>();
  // num = sum k x(s+t), den = sum k (no hat, no normalization; denoise.py:254-269)
  if ((rc = run_sweep(ctx, g, w, 2, guide, ChanSpec{x, nullptr}, ChanSpec{nullptr, nullptr}, taps,
                      bandwidth, false, part)))
    return rc;
  FixIO io{};
  io.out = out;
  return run_fixup<FIX_NLM>(ctx, g, w, 2, part, io);
}

// ---------------------------------------------------------------- strips ---

int pnp_dsg_geometry(int Hg, int W, int R, int P, int box, int* out) {
  if (!out) return fail(PNP_EINVAL, "null argument");
  int rc = check_geometry(1, Hg, W, R, P, 1.0);
  if (rc) return rc;
  int kind = 0, TH = 0, KG = 0;
  if ((rc = choose_path(R, P, box != 0, kind, TH, KG))) return rc;
  const int p = (P - 1) / 2;
  out[0] = TH;
  out[1] = groups_for(Hg, W, R, P, box != 0);
  out[2] = kind == PATH_GEN_NEAR ? 0 : R;  // far band of a partial block
  out[3] = kind;
  // input rows a tile row reads above / below its own rows, and rows of the
  // channel planes (rs) below
  if (kind == PATH_FAST) {
    out[4] = p;
    out[5] = R + (p > kKY ? p : kKY);
    out[6] = R + kKY - 1;
  } else if (kind == PATH_GEN_SYM) {
    out[4] = p;
    out[5] = R + p;
    out[6] = R;
  } else {
    out[4] = R + p;
    out[5] = R + p;
    out[6] = R;
  }
  out[7] = KG;
  return PNP_OK;
}

int pnp_dsg_groups(int Hg, int W, int R, int P, int box) {
  if (check_geometry(1, Hg, W, R, P, 1.0)) return -1;
  return groups_for(Hg, W, R, P, box != 0);
}

int64_t pnp_dsg_partial_floats(int Hg, int W, int R, int P, int box, int C, int ntr) {
  if (check_geometry(1, Hg, W, R, P, 1.0) || C < 1 || C > 2 || ntr < 0) return -1;
  int kind = 0, TH = 0, KG = 0;
  if (choose_path(R, P, box != 0, kind, TH, KG)) return -1;
  const int Rb = kind == PATH_GEN_NEAR ? 0 : R;
  const int64_t blk = (int64_t)C * (TH + Rb) * (kTW + 2 * Rb);
  return (int64_t)ntr * groups_for(Hg, W, R, P, box != 0) * ((W + kTW - 1) / kTW) * blk;
}

int64_t pnp_dsg_kcache_floats(int Hg, int W, int R, int P, int box, int ntr) {
  if (check_geometry(1, Hg, W, R, P, 1.0) || ntr < 0) return -1;
  int kind = 0, TH = 0, KG = 0;
  if (choose_path(R, P, box != 0, kind, TH, KG)) return -1;
  if (kind != PATH_FAST) return 0;  // the general sweep recomputes its weights
  return (int64_t)half_window(R) * ntr * TH * (((W + kTW - 1) / kTW) * kTW);
}

int pnp_dsg_strip_sweep(pnp_ctx* ctx, int pass, const float* guide, const float* x,
                        const float* rs, int Hg, int W, int buf_r0, int buf_rows, int tr0,
                        int ntr, int R, int P, const float* taps, double bandwidth,
                        float* partial, int part_off, int part_ntr, float* kcache) {
  if (!ctx || !guide || !partial) return fail(PNP_EINVAL, "null argument");
  int rc = check_geometry(1, Hg, W, R, P, bandwidth);
  if (rc) return rc;
  if ((rc = validate_taps(taps, P))) return rc;
  if (buf_r0 < 0 || buf_rows < 1 || buf_r0 + buf_rows > Hg) return fail(PNP_EINVAL, "bad window");
  if (ntr < 0 || part_off < 0 || part_off + ntr > part_ntr) return fail(PNP_EINVAL, "bad tiles");
  PNP_CUDA(cudaSetDevice(ctx->device));
  Geom g;
  if ((rc = make_geom(ctx, 1, Hg, W, R, P, taps_box(taps, P), g))) return rc;
  if (tr0 < 0 || tr0 + ntr > g.tiles_y) return fail(PNP_EINVAL, "tile rows out of range");
  if (kcache && g.kind != PATH_FAST)
    return fail(PNP_EINVAL, "strips of the general sweep have no k cache");
  Window w{buf_r0, buf_rows, tr0, ntr, 0, part_off, part_ntr, 0, 0};
  const int use = kcache ? MODE_CACHED : MODE_RECOMPUTE;
  switch (pass) {
    case 0:  // mass g: y = in-image mask
      return run_sweep(ctx, g, w, 1, guide, ChanSpec{nullptr, nullptr},
                       ChanSpec{nullptr, nullptr}, taps, bandwidth, true, partial,
                       kcache ? MODE_STORE : MODE_RECOMPUTE, kcache);
    case 1:  // Kx and d: y = rs*x, rs
      if (!x || !rs) return fail(PNP_EINVAL, "pass 1 needs x and rs");
      return run_sweep(ctx, g, w, 2, guide, ChanSpec{rs, x}, ChanSpec{rs, nullptr}, taps,
                       bandwidth, true, partial, use, kcache);
    case 2:  // d only: y = rs
      if (!rs) return fail(PNP_EINVAL, "pass 2 needs rs");
      return run_sweep(ctx, g, w, 1, guide, ChanSpec{rs, nullptr}, ChanSpec{nullptr, nullptr},
                       taps, bandwidth, true, partial, use, kcache);
    case 3:  // Kx only: y = rs*x
      if (!x || !rs) return fail(PNP_EINVAL, "pass 3 needs x and rs");
      return run_sweep(ctx, g, w, 1, guide, ChanSpec{rs, x}, ChanSpec{nullptr, nullptr}, taps,
                       bandwidth, true, partial, use, kcache);
  }
  return fail(PNP_EINVAL, "unknown pass");
}

int pnp_dsg_strip_fixup(pnp_ctx* ctx, int mode, const float* partial, int part_tr0,
                        int part_ntr, int Hg, int W, int R, int P, int box, int y0, int y1, int buf_r0,
                        int buf_rows, float* rs, float* kx, float* d, unsigned* mbits,
                        const float* inv_m, const float* x, float* out) {
  if (!ctx || !partial) return fail(PNP_EINVAL, "null argument");
  int rc = check_geometry(1, Hg, W, R, P, 1.0);
  if (rc) return rc;
  if (y0 < buf_r0 || y1 > buf_r0 + buf_rows || y0 > y1) return fail(PNP_EINVAL, "bad rows");
  PNP_CUDA(cudaSetDevice(ctx->device));
  Geom g;
  if ((rc = make_geom(ctx, 1, Hg, W, R, P, box != 0, g))) return rc;
  Window w{buf_r0, buf_rows, 0, 0, part_tr0, 0, part_ntr, y0, y1 - y0};
  FixIO io{};
  io.rs = rs;
  io.kx = kx;
  io.d = d;
  io.mbits = mbits;
  io.inv_m = inv_m;
  io.x = x;
  io.out = out;
  switch (mode) {
    case 0:
      if (!rs) return fail(PNP_EINVAL, "mode 0 needs rs");
      return run_fixup<FIX_RS>(ctx, g, w, 1, partial, io);
    case 1:
      if (!rs || !kx || !d || !mbits) return fail(PNP_EINVAL, "mode 1 needs rs, kx, d, mbits");
      return run_fixup<FIX_KXD>(ctx, g, w, 2, partial, io);
    case 2:
      if (!rs || !d || !mbits) return fail(PNP_EINVAL, "mode 2 needs rs, d, mbits");
      return run_fixup<FIX_D>(ctx, g, w, 1, partial, io);
    case 3:
      if (!rs || !d || !inv_m || !x || !out) return fail(PNP_EINVAL, "mode 3 needs rs,d,inv_m,x,out");
      return run_fixup<FIX_APPLY>(ctx, g, w, 1, partial, io);
  }
  return fail(PNP_EINVAL, "unknown mode");
}

int pnp_dsg_strip_finalize(pnp_ctx* ctx, const float* kx, const float* d, const float* x,
                           float* out, const unsigned* mbits, int Hg, int W, int y0, int y1,
                           int buf_r0, int buf_rows) {
  if (!ctx || !kx || !d || !x || !out || !mbits) return fail(PNP_EINVAL, "null argument");
  if (y0 < buf_r0 || y1 > buf_r0 + buf_rows || y0 > y1 || y1 > Hg) return fail(PNP_EINVAL, "bad rows");
  PNP_CUDA(cudaSetDevice(ctx->device));
  Geom g{};
  g.B = 1;
  g.Hg = Hg;
  g.W = W;
  Window w{buf_r0, buf_rows, 0, 0, 0, 0, 0, y0, y1 - y0};
  return run_finalize(ctx, g, w, kx, d, mbits, x, out, nullptr);
}

}  // extern "C"
