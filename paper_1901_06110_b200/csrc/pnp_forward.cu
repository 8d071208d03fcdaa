// Forward operators and the fused linearized-ADMM elementwise steps.
//
// SR (reference forward.py:98-185): A = decimate_k o blur, blur = correlation
// with a separable normalized kernel under periodic (wrap) or half-sample
// symmetric padding; A^T = blur o zero-fill upsample (exact for symmetric
// kernels).  Both are SMEM-tiled separable filters; the residual kernel
// evaluates the blur only at the kept samples and fuses "- y" and the
// 0.5||.||^2 data-term partials; the adjoint stages the zero-filled
// upsampled tile.
// QIS (forward.py:312-327): elementwise, evaluated in double.
// ADMM (solver.py:219-228): x-update + projection + x+u + finite flags in one
// pass; u-update + residual/PSNR partial sums in one pass.  All reductions
// are per-block partials summed in a fixed order (deterministic).
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "admm_math.cuh"
#include "pnp_internal.h"
#include "pnp_pdl.cuh"
#include "pnp_reduce.cuh"

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

// out[b*stride + k] = scale * sum_j partial[b][j][k]: one CTA per (b, k),
// thread t sums j = t, t+256, ... in order, then a fixed shuffle/SMEM tree
// (deterministic; latency-tolerant for many partials).
__global__ void __launch_bounds__(256) reduce_partials_kernel(const double* partial, int nblk,
                                                              int nvec, double scale, double* out,
                                                              int stride) {
  __shared__ double red[8];
  cta_reduce_partials(partial, nblk, nvec, blockIdx.x, blockIdx.y, scale, out, stride, red);
}

// A reduce_partials_kernel launch folded into the next kernel: its CTA
// (0, 0, 0) reduces partials the previous kernel wrote (out[b] = scale *
// sum_j partial[b][j], b < batch) -- same arithmetic, one launch fewer.
struct RedEpi {
  const double* part;
  double* out;
  double scale;
  int nblk, batch;
};

// CTA (0, 0, z) reduces images z, z + gridDim.z, ... (one image per CTA when the
// grid's z is the batch): a batch's reductions run in parallel.
__device__ __forceinline__ void red_epilogue(const RedEpi& e) {
  if (!e.out || blockIdx.x || blockIdx.y) return;
  __shared__ double red[8];
  for (int b = blockIdx.z; b < e.batch; b += gridDim.z)
    cta_reduce_partials(e.part, e.nblk, 1, b, 0, e.scale, e.out, 1, red);
}

// The linearized-ADMM x-update (solver.py:219-221) fused into a gradient
// kernel's epilogue: x <- proj(mu (alpha x + rho (v - u) - grad)), z = x + u,
// finite flags -- the arithmetic of admm_xupdate_kernel, per pixel.
struct XUpd {
  float* x;
  const float* v;
  const float* u;
  float* z;
  double mu, alpha, rho;
  float lo, hi;
  int* flags;
};

__device__ __forceinline__ int xupdate_pixel(const XUpd& q, size_t i, float grad) {
  float xf, zf;
  const int f = admm_xupdate(q.mu, q.alpha, q.rho, q.lo, q.hi, q.x[i], q.v[i], q.u[i], grad, xf,
                             zf);
  q.x[i] = xf;
  q.z[i] = zf;
  return f;
}

__device__ __forceinline__ void flags_or(int* flags, int f) {
  f = __reduce_or_sync(0xffffffffu, f);
  if (f && (threadIdx.x & 31) == 0) atomicOr(flags, f);
}

// SR blur kernels, SMEM tiled: the image region of a tile (+ radius halo,
// boundary-mapped once at staging) is filtered separably -- horizontal taps
// into a row buffer, then vertical taps -- in the reference's summation order
// (forward.py:_convolve: rows outer, columns inner).
// per-image conjugate-gradients scalars (device; see cg_* kernels below)
struct CgState {
  double rs, pap, bnorm, beta;
  int done, iters, status, stepped;  // status: 0 ok, 2 breakdown (p.Ap <= 0), 3 non-finite
};

// Row window of an SR kernel call (row strips of a sharded image; the full
// image is the window [0, Hg)).  Input rows are a buffer holding global rows
// [in_r0, in_r0 + in_rows) (HR rows for the residual, LR rows for the
// adjoint); outputs are global rows [out_r0, out_r0 + out_rows) (LR for the
// residual, HR for the adjoint).  Boundary mapping uses the global height.
struct SrWin {
  int Hg, in_r0, in_rows, out_r0, out_rows;
};

constexpr int kSrT = 16;   // low-res outputs per tile side (residual)
constexpr int kSrTA = 32;  // high-res outputs per tile side (adjoint)

// r = A x - y (or A x when y == null) on the low-res grid; optional
// 0.5||r||^2 partials, one per tile: partial[b][tile].
__global__ void __launch_bounds__(256)
sr_residual_kernel(const float* __restrict__ x, const float* __restrict__ y, float* __restrict__ r,
                   const SrWin win, int W, int k, int rad, int sym, const Taps taps,
                   double* partial, const CgState* skip = nullptr) {
  pdl_begin();
  extern __shared__ float sm[];
  const int H = win.Hg, w = W / k, b = blockIdx.z;
  if (skip && skip[b].done) return;  // CG: image already converged
  const int S = k * (kSrT - 1) + 1 + 2 * rad;  // staged hi-res rows / cols
  float* X = sm;                               // [S][S]
  float* Hh = sm + S * S;                      // [S][kSrT]
  const int oy0 = win.out_r0 + blockIdx.y * kSrT, ox0 = blockIdx.x * kSrT;
  const int y0 = k * oy0 - rad, x0 = k * ox0 - rad;
  const float* xb = x + (size_t)b * win.in_rows * W;
  // this thread's output and its observation, loaded before the staging so
  // the two global round trips overlap
  const int ty = threadIdx.x / kSrT, tx = threadIdx.x - ty * kSrT;
  const int oy = oy0 + ty, ox = ox0 + tx;
  const bool own = oy < win.out_r0 + win.out_rows && ox < w;
  const size_t o = own ? (size_t)b * win.out_rows * w + (size_t)(oy - win.out_r0) * w + ox : 0;
  const float yo = (own && y) ? y[o] : 0.f;
  // The configs' operator (factor 2, 9x9 kernel) runs with compile-time tile
  // sizes and unrolled taps; tiles whose staged window needs no boundary map
  // copy it row by row.  Same products in the same order as the generic
  // loops below -> the same bits.
  constexpr int FS = 2 * (kSrT - 1) + 1 + 8;
  const bool fast = k == 2 && rad == 4;
  if (fast && y0 >= 0 && y0 + FS <= H && y0 - win.in_r0 >= 0 &&
      y0 - win.in_r0 + FS <= win.in_rows && x0 >= 0 && x0 + FS <= W) {
    // thread (warp w, lane l): rows w + 8m, columns l and l + 32; every load
    // of the thread in flight before its first shared store
    const int wq = threadIdx.x >> 5, l = threadIdx.x & 31;
    const float* src = xb + (size_t)(y0 - win.in_r0 + wq) * W + x0 + l;
    float v[5][2];
#pragma unroll
    for (int m = 0; m < 5; ++m)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const bool in = wq + 8 * m < FS && l + 32 * h < FS;
        PNP_CHECK(!in || (y0 - win.in_r0 + wq + 8 * m < win.in_rows && x0 + l + 32 * h < W &&
                          x0 + l + 32 * h >= 0 && S == FS));
        v[m][h] = in ? src[(size_t)8 * m * W + 32 * h] : 0.f;
      }
#pragma unroll
    for (int m = 0; m < 5; ++m)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (wq + 8 * m < FS && l + 32 * h < FS) X[(wq + 8 * m) * FS + l + 32 * h] = v[m][h];
  } else {
    // boundary tiles: the (separable) index maps once per staged row / column
    int* rmap = reinterpret_cast<int*>(Hh + S * kSrT);
    int* cmap = rmap + S;
    for (int t = threadIdx.x; t < S; t += blockDim.x) {
      int sy = map_index(min(y0 + t, H - 1 + rad), H, sym) - win.in_r0;
      rmap[t] = sy < 0 ? 0 : (sy >= win.in_rows ? win.in_rows - 1 : sy);  // halo rows only: never hit
      cmap[t] = map_index(min(x0 + t, W - 1 + rad), W, sym);
    }
    __syncthreads();
    for (int yy = threadIdx.x >> 5; yy < S; yy += blockDim.x >> 5) {
      const float* src = xb + (size_t)rmap[yy] * W;
      for (int xx = threadIdx.x & 31; xx < S; xx += 32) {
        PNP_CHECK(rmap[yy] >= 0 && rmap[yy] < win.in_rows && cmap[xx] >= 0 && cmap[xx] < W);
        X[yy * S + xx] = src[cmap[xx]];
      }
    }
  }
  __syncthreads();
  if (fast) {  // thread t: filtered row (t >> 4) + 16 m, low-res column t & 15
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const int yy = (threadIdx.x >> 4) + 16 * m;
      if (yy < FS) {
        const float* row = X + yy * FS + 2 * (threadIdx.x & 15);
        PNP_CHECK(row + 8 < X + S * S);
        float s = 0.f;
#pragma unroll
        for (int c = 0; c <= 8; ++c) s = fmaf(taps.tx[c], row[c], s);
        Hh[yy * kSrT + (threadIdx.x & 15)] = s;
      }
    }
  } else {
    for (int i = threadIdx.x; i < S * kSrT; i += blockDim.x) {
      const int yy = i / kSrT, tx = i - yy * kSrT;
      const float* row = X + yy * S + k * tx;
      float s = 0.f;
      for (int c = 0; c <= 2 * rad; ++c) s = fmaf(taps.tx[c], row[c], s);
      Hh[i] = s;
    }
  }
  __syncthreads();
  double sq = 0.0;
  if (own) {
    float acc = 0.f;
    if (fast) {
      PNP_CHECK((2 * ty + 8) * kSrT + tx < S * kSrT);
#pragma unroll
      for (int a = 0; a <= 8; ++a) acc = fmaf(taps.ty[a], Hh[(2 * ty + a) * kSrT + tx], acc);
    } else {
      for (int a = 0; a <= 2 * rad; ++a) acc = fmaf(taps.ty[a], Hh[(k * ty + a) * kSrT + tx], acc);
    }
    if (y) acc -= yo;
    r[o] = acc;
    sq = (double)acc * (double)acc;
  }
  if (partial) {
    __shared__ double red[8];
    for (int off = 16; off; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q];
      partial[((size_t)b * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
    }
  }
}

// x_out = A^T r = blur(upsample_k(r)) on the high-res grid: the zero-filled
// upsampled tile (+ halo, boundary-mapped) is staged, then filtered.
// Conjugate-gradients epilogue of the Gram operator: out = A^T A p + shift p,
// one partial of p . out per tile, converged images skipped.
struct CgEpi {
  const float* p;
  double shift;
  double* partial;
  const CgState* skip;  // nullable
};

enum AdjMode { ADJ_PLAIN = 0, ADJ_XUPD = 1, ADJ_CG = 2 };

template <int MODE>
__global__ void __launch_bounds__(256)
sr_adjoint_kernel(const float* __restrict__ r, float* __restrict__ out, const SrWin win, int W,
                  int k, int rad, int sym, const Taps taps, const XUpd q, const CgEpi cg,
                  const RedEpi red = RedEpi{}) {
  pdl_begin();
  extern __shared__ float sm[];
  const int H = win.Hg, w = W / k, b = blockIdx.z;
  if (MODE == ADJ_CG && cg.skip && cg.skip[b].done) return;
  constexpr bool XU = MODE == ADJ_XUPD;
  const int S = kSrTA + 2 * rad;
  float* U = sm;             // [S][S]
  float* Hh = sm + S * S;    // [S][kSrTA]
  const int py0 = win.out_r0 + blockIdx.y * kSrTA, px0 = blockIdx.x * kSrTA;
  const float* rb = r + (size_t)b * win.in_rows * w;
  // The configs' operator (factor 2, 9x9 kernel) on tiles whose staged window
  // needs no boundary map: the zero-filled upsampled tile is never built.
  // Only even high-res rows / columns hold samples, so the horizontal pass
  // runs over the 20 x 20 low-res samples with the 5 (even output column) or
  // 4 (odd) taps that meet a sample, and the vertical pass over the 20
  // filtered sample rows with 5 or 4 taps.  The generic loops add exact
  // zeros for the skipped taps, in the same order -> the same bits.
  constexpr int FL = kSrTA / 2 + 4;  // low-res rows / columns staged
  const bool fast = k == 2 && rad == 4 && ((py0 | px0) & 1) == 0 && py0 - 4 >= 0 &&
                    py0 + kSrTA + 4 <= H && px0 - 4 >= 0 && px0 + kSrTA + 4 <= W &&
                    py0 / 2 - 2 - win.in_r0 >= 0 && py0 / 2 - 2 - win.in_r0 + FL <= win.in_rows;
  // per-thread tap sets: output column / row parity picks the even (5) or
  // odd (4) taps; a thread's column (lane) and row parity (warp) are fixed
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  if (fast) {
    const float* src = rb + (size_t)(py0 / 2 - 2 - win.in_r0 + wq) * w + px0 / 2 - 2 + lane;
    float v[3];
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const bool in = wq + 8 * m < FL && lane < FL;
      PNP_CHECK(!in || (py0 / 2 - 2 - win.in_r0 + wq + 8 * m < win.in_rows &&
                        px0 / 2 - 2 + lane < w && px0 / 2 - 2 + lane >= 0 && FL * FL <= S * S));
      v[m] = in ? src[(size_t)8 * m * w] : 0.f;
    }
#pragma unroll
    for (int m = 0; m < 3; ++m)
      if (wq + 8 * m < FL && lane < FL) U[(wq + 8 * m) * FL + lane] = v[m];
    __syncthreads();
    const int odd = lane & 1;
    float t5[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) t5[j] = odd ? (j < 4 ? taps.tx[2 * j + 1] : 0.f) : taps.tx[2 * j];
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const int i = wq + 8 * m;
      if (i < FL) {
        const float* row = U + i * FL + ((lane + 1) >> 1);
        PNP_CHECK(row + (odd ? 3 : 4) < U + FL * FL);
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) s = fmaf(t5[j], row[j], s);
        if (!odd) s = fmaf(t5[4], row[4], s);
        Hh[i * kSrTA + lane] = s;
      }
    }
  } else {
    // boundary tiles: the (separable) index maps once per staged row / column,
    // -1 where the mapped high-res row / column holds no low-res sample
    int* rmap = reinterpret_cast<int*>(Hh + S * kSrTA);
    int* cmap = rmap + S;
    for (int t = threadIdx.x; t < S; t += blockDim.x) {
      const int uy = map_index(min(py0 - rad + t, H - 1 + rad), H, sym);
      const int ux = map_index(min(px0 - rad + t, W - 1 + rad), W, sym);
      const int qy = uy / k, qx = ux / k;
      int ly = qy - win.in_r0;
      ly = ly < 0 ? 0 : (ly >= win.in_rows ? win.in_rows - 1 : ly);  // halo rows only: never hit
      rmap[t] = uy == qy * k ? ly : -1;
      cmap[t] = ux == qx * k ? qx : -1;
    }
    __syncthreads();
    for (int yy = threadIdx.x >> 5; yy < S; yy += blockDim.x >> 5) {
      const int ly = rmap[yy];
      for (int xx = threadIdx.x & 31; xx < S; xx += 32) {
        const int qx = cmap[xx];
        PNP_CHECK(ly < win.in_rows && qx < w);
        U[yy * S + xx] = (ly >= 0 && qx >= 0) ? rb[(size_t)ly * w + qx] : 0.f;
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < S * kSrTA; i += blockDim.x) {
      const int yy = i / kSrTA, xx = i - yy * kSrTA;
      const float* row = U + yy * S + xx;
      float s = 0.f;
      if (rad == 4) {
#pragma unroll
        for (int c = 0; c <= 8; ++c) s = fmaf(taps.tx[c], row[c], s);
      } else {
        for (int c = 0; c <= 2 * rad; ++c) s = fmaf(taps.tx[c], row[c], s);
      }
      Hh[i] = s;
    }
  }
  __syncthreads();
  int f = 0;
  double dot = 0.0;
  auto emit = [&](int py, int px, float acc) {
    const size_t o = (size_t)b * win.out_rows * W + (size_t)(py - win.out_r0) * W + px;
    if (XU) {
      f |= xupdate_pixel(q, o, acc);
    } else if (MODE == ADJ_CG) {
      const float pv = cg.p[o];
      const float ap = (float)((double)acc + cg.shift * (double)pv);
      out[o] = ap;
      dot += (double)pv * (double)ap;
    } else {
      out[o] = acc;
    }
  };
  if (fast && MODE != ADJ_CG) {
    // thread (warp wq, lane): output rows 4 wq .. 4 wq + 3 of column lane from
    // filtered sample rows 2 wq .. 2 wq + 5 (even rows: 5 taps, odd rows: 4)
    const float* col = Hh + 2 * wq * kSrTA + lane;
    PNP_CHECK(col + 5 * kSrTA < Hh + FL * kSrTA);
    float h6[6];
#pragma unroll
    for (int j6 = 0; j6 < 6; ++j6) h6[j6] = col[j6 * kSrTA];
    const int px = px0 + lane, py = py0 + 4 * wq;
    const size_t o0 = (size_t)b * win.out_rows * W + (size_t)(py - win.out_r0) * W + px;
#pragma unroll
    for (int r4 = 0; r4 < 4; ++r4) {
      const int base = (r4 + 1) >> 1, odd = r4 & 1;
      float acc = 0.f;
#pragma unroll
      for (int j5 = 0; j5 < 4; ++j5) acc = fmaf(taps.ty[2 * j5 + odd], h6[base + j5], acc);
      if (!odd) acc = fmaf(taps.ty[8], h6[base + 4], acc);
      if (py + r4 < win.out_r0 + win.out_rows) {
        const size_t o = o0 + (size_t)r4 * W;
        if (XU) f |= xupdate_pixel(q, o, acc);
        else out[o] = acc;
      }
    }
  } else if (fast) {
    // (conjugate gradients: the generic loop's thread / output order, so the
    // per-thread dot partials sum in the same order) thread (warp wq, lane):
    // output rows wq + 8 m, column lane; the rows' parity is the warp's
    float ty5[5];
#pragma unroll
    for (int j5 = 0; j5 < 5; ++j5)
      ty5[j5] = (wq & 1) ? (j5 < 4 ? taps.ty[2 * j5 + 1] : 0.f) : taps.ty[2 * j5];
    const int px = px0 + lane;
#pragma unroll
    for (int m = 0; m < kSrTA * kSrTA / 256; ++m) {
      const int yy = wq + 8 * m, py = py0 + yy;
      if (py >= win.out_r0 + win.out_rows || px >= W) continue;
      const float* col = Hh + ((yy + 1) >> 1) * kSrTA + lane;
      float acc = 0.f;
#pragma unroll
      for (int j5 = 0; j5 < 4; ++j5) acc = fmaf(ty5[j5], col[j5 * kSrTA], acc);
      if (!(wq & 1)) acc = fmaf(ty5[4], col[4 * kSrTA], acc);
      emit(py, px, acc);
    }
  } else {
    for (int i = threadIdx.x; i < kSrTA * kSrTA; i += blockDim.x) {
      const int yy = i / kSrTA, xx = i - yy * kSrTA;
      const int py = py0 + yy, px = px0 + xx;
      if (py >= win.out_r0 + win.out_rows || px >= W) continue;
      float acc = 0.f;
      if (rad == 4) {
#pragma unroll
        for (int a = 0; a <= 8; ++a) acc = fmaf(taps.ty[a], Hh[(yy + a) * kSrTA + xx], acc);
      } else {
        for (int a = 0; a <= 2 * rad; ++a) acc = fmaf(taps.ty[a], Hh[(yy + a) * kSrTA + xx], acc);
      }
      emit(py, px, acc);
    }
  }
  if (XU) flags_or(q.flags, f);
  if (MODE == ADJ_CG) {
    __shared__ double red8[8];
    for (int off = 16; off; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
    if ((threadIdx.x & 31) == 0) red8[threadIdx.x >> 5] = dot;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w8 = 0; w8 < (int)(blockDim.x >> 5); ++w8) t += red8[w8];
      cg.partial[((size_t)b * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
    }
  }
  if (MODE != ADJ_CG) red_epilogue(red);  // data term of the residual kernel
}

static size_t sr_res_smem(int k, int rad) {  // + the row / column index maps
  const int S = k * (kSrT - 1) + 1 + 2 * rad;
  return (size_t)(S * S + S * kSrT + 2 * S) * sizeof(float);
}
static size_t sr_adj_smem(int rad) {
  const int S = kSrTA + 2 * rad;
  return (size_t)(S * S + S * kSrTA + 2 * S) * sizeof(float);
}
static dim3 sr_res_grid(int H, int W, int k, int batch) {  // H: output HR rows of the window
  return dim3((W / k + kSrT - 1) / kSrT, (H / k + kSrT - 1) / kSrT, batch);
}
static dim3 sr_adj_grid(int H, int W, int batch) {
  return dim3((W + kSrTA - 1) / kSrTA, (H + kSrTA - 1) / kSrTA, batch);
}
static SrWin res_full(int H, int k) { return SrWin{H, 0, H, 0, H / k}; }
static SrWin adj_full(int H, int k) { return SrWin{H, 0, H / k, 0, H}; }
static cudaError_t sr_smem_attr(size_t res, size_t adj) {
  // opt-in shared-memory sizes are per-device function attributes: remember
  // the largest set per device (raised under a lock; reads are racy-benign
  // because a stale value only repeats an idempotent call)
  static std::mutex mu;
  static size_t set_res[64], set_adj[64];
  int dev = 0;
  cudaGetDevice(&dev);
  dev &= 63;
  if (res <= std::max<size_t>(set_res[dev], 48 * 1024) &&
      adj <= std::max<size_t>(set_adj[dev], 48 * 1024))
    return cudaSuccess;
  std::lock_guard<std::mutex> lock(mu);
  cudaError_t e = cudaSuccess;
  if (res > std::max<size_t>(set_res[dev], 48 * 1024)) {
    e = cudaFuncSetAttribute(sr_residual_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)res);
    if (e == cudaSuccess) set_res[dev] = res;
  }
  if (e == cudaSuccess && adj > std::max<size_t>(set_adj[dev], 48 * 1024)) {
    e = cudaFuncSetAttribute(sr_adjoint_kernel<ADJ_PLAIN>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)adj);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(sr_adjoint_kernel<ADJ_XUPD>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)adj);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(sr_adjoint_kernel<ADJ_CG>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)adj);
    if (e == cudaSuccess) set_adj[dev] = adj;
  }
  return e;
}

template <bool XU>
__global__ void __launch_bounds__(256)
qis_grad_kernel(const float* __restrict__ x, const float* __restrict__ ones,
                const float* __restrict__ zeros, float* __restrict__ grad, size_t n,
                double gk, double floor_, double* partial, const XUpd q) {
  pdl_begin();
  const int b = blockIdx.y;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  double term = 0.0;
  int f = 0;
  if (i < n) {
    const size_t o = (size_t)b * n + i;
    const double z = gk * fmax((double)x[o], floor_);
    const double k1 = ones[o], k0 = zeros[o];
    if (partial) term = k0 * z - k1 * log(-expm1(-z));
    const float gv = (float)(gk * (k0 - k1 / expm1(z)));
    if (XU)
      f = xupdate_pixel(q, o, gv);
    else if (grad)
      grad[o] = gv;
  }
  if (XU) flags_or(q.flags, f);
  if (partial) block_sum_store(term, partial);
}

__global__ void __launch_bounds__(256)
admm_xupdate_kernel(float* __restrict__ x, const float* __restrict__ v, const float* __restrict__ u,
                    const float* __restrict__ grad, float* __restrict__ z, size_t n, double mu,
                    double alpha, double rho, float lo, float hi, int* flags) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  int f = 0;
  if (i < n) {
    float xf, zf;
    f = admm_xupdate(mu, alpha, rho, lo, hi, x[i], v[i], u[i], grad[i], xf, zf);
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
  if (sr_res_smem(factor, radius) > 227 * 1024 || sr_adj_smem(radius) > 227 * 1024)
    return fail(PNP_EINVAL, "blur radius / factor too large for the tiled SR kernels");
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

// Input validation (image.py:35-40 "non-finite" ValueError) in one pass:
// flag |= 1 if any element is NaN/Inf (16 B vector loads, warp ballot).
__global__ void __launch_bounds__(256) nonfinite_kernel(const float* __restrict__ x, size_t n,
                                                        int* flag) {
  const size_t n4 = n / 4;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  bool bad = false;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 v = __ldcs(x4 + i);
    bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
  }
  for (size_t i = n4 * 4 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    bad |= !isfinite(x[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// ---- SplitMix64 streams on the device (reference forward.py:36-79) ----
// Output k (k = 1, 2, ...) of a stream with state s is mix(s + k*GOLDEN), so
// every element is independent of the others and the device reproduces the
// host stream bit for bit (uniforms) -- no sequential state to carry.
__device__ __forceinline__ double splitmix_uniform(unsigned long long state,
                                                   unsigned long long k) {
  unsigned long long z = state + 0x9E3779B97F4A7C15ull * k;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * 0x1.0p-53;
}

__global__ void __launch_bounds__(256) splitmix_uniform_kernel(unsigned long long state,
                                                               size_t n, double* out) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = splitmix_uniform(state, i + 1);
}

// Observation noise of sr_simulate (forward.py:205-212): Box-Muller on the
// uniform pairs (u1, u2) = outputs (2j+1, 2j+2): r = sqrt(-2 log1p(-u1)),
// n_2j = r cos(2 pi u2), n_2j+1 = r sin(2 pi u2) (forward.py:70-79), then
// y + sigma * n in float64, written as float32 and/or float64.  The libm
// calls are float64 (CUDA's are within 2 ulp of numpy's).
__global__ void __launch_bounds__(256) sr_noise_kernel(const float* __restrict__ y, size_t n,
                                                       unsigned long long state, double sigma,
                                                       float* out32, double* out64) {
  const size_t pairs = (n + 1) / 2;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < pairs; j += stride) {
    const double u1 = splitmix_uniform(state, 2 * j + 1);
    const double u2 = splitmix_uniform(state, 2 * j + 2);
    const double r = sqrt(-2.0 * log1p(-u1));
    const double th = 6.283185307179586 * u2;  // 2.0 * math.pi, then * u2
    const size_t i0 = 2 * j;
    const double v0 = (double)y[i0] + sigma * (r * cos(th));
    if (out32) out32[i0] = (float)v0;
    if (out64) out64[i0] = v0;
    if (i0 + 1 < n) {
      const double v1 = (double)y[i0 + 1] + sigma * (r * sin(th));
      if (out32) out32[i0 + 1] = (float)v1;
      if (out64) out64[i0 + 1] = v1;
    }
  }
}

// ---- conjugate gradients on (A^T A + shift I) x = rhs, device resident ----
// Reference cg_solve (solver.py:244-282), per image of a batch: the scalars
// (rs, p.Ap, ||rhs||, beta, iteration count, flags) live on the device, every
// kernel skips images that are done, and the host only polls the done flags
// every few iterations -- no per-iteration round trip.

__device__ __forceinline__ double block_sum256(double v) {
  __shared__ double red[8];
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
  return t;  // valid in thread 0
}

// r = rhs - ap (warm start) or rhs (x zeroed); p = r; partials r.r, rhs.rhs
__global__ void __launch_bounds__(256)
cg_init_kernel(const float* __restrict__ rhs, const float* __restrict__ ap, float* __restrict__ x,
               float* __restrict__ r, float* __restrict__ p, size_t n, double* partial) {
  const int b = blockIdx.y;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  double rr = 0.0, bb = 0.0;
  if (i < n) {
    const size_t o = (size_t)b * n + i;
    const float bv = rhs[o];
    float rv = bv;
    if (ap) rv = (float)((double)bv - (double)ap[o]);
    else x[o] = 0.f;
    r[o] = rv;
    p[o] = rv;
    rr = (double)rv * rv;
    bb = (double)bv * bv;
  }
  rr = block_sum256(rr);
  bb = block_sum256(bb);
  if (threadIdx.x == 0) {
    double* pp = partial + ((size_t)b * gridDim.x + blockIdx.x) * 2;
    pp[0] = rr;
    pp[1] = bb;
  }
}

__global__ void __launch_bounds__(256)
cg_start_kernel(const double* partial, int nblk, CgState* st, double tol, int max_iters) {
  const int b = blockIdx.x;
  double rr = 0.0, bb = 0.0;
  for (int j = threadIdx.x; j < nblk; j += blockDim.x) {
    rr += partial[((size_t)b * nblk + j) * 2];
    bb += partial[((size_t)b * nblk + j) * 2 + 1];
  }
  rr = block_sum256(rr);
  bb = block_sum256(bb);
  if (threadIdx.x == 0) {
    CgState s{};
    s.rs = rr;
    s.bnorm = sqrt(bb);
    s.done = (s.bnorm == 0.0 || sqrt(s.rs) / s.bnorm <= tol || max_iters < 1) ? 1 : 0;
    st[b] = s;
  }
}

// p.Ap -> curvature checks (the reference raises on non-finite / <= 0)
__global__ void __launch_bounds__(256) cg_curv_kernel(const double* partial, int nblk, CgState* st) {
  const int b = blockIdx.x;
  if (st[b].done) return;
  double v = 0.0;
  for (int j = threadIdx.x; j < nblk; j += blockDim.x) v += partial[(size_t)b * nblk + j];
  v = block_sum256(v);
  if (threadIdx.x == 0) {
    st[b].pap = v;
    if (!isfinite(v)) {
      st[b].status = 3;
      st[b].done = 1;
    } else if (v <= 0.0) {
      st[b].status = 2;
      st[b].done = 1;
    }
  }
}

// x += a p; r -= a Ap (a = rs / p.Ap); partials of r.r
__global__ void __launch_bounds__(256)
cg_update_kernel(float* __restrict__ x, float* __restrict__ r, const float* __restrict__ p,
                 const float* __restrict__ ap, size_t n, const CgState* st, double* partial) {
  const int b = blockIdx.y;
  if (st[b].done) return;
  const double a = st[b].rs / st[b].pap;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  double rr = 0.0;
  if (i < n) {
    const size_t o = (size_t)b * n + i;
    x[o] = (float)((double)x[o] + a * (double)p[o]);
    const float rv = (float)((double)r[o] - a * (double)ap[o]);
    r[o] = rv;
    rr = (double)rv * rv;
  }
  rr = block_sum256(rr);
  if (threadIdx.x == 0) partial[(size_t)b * gridDim.x + blockIdx.x] = rr;
}

__global__ void __launch_bounds__(256)
cg_step_kernel(const double* partial, int nblk, CgState* st, double tol, int max_iters) {
  const int b = blockIdx.x;
  if (st[b].done) {
    if (threadIdx.x == 0) st[b].stepped = 0;
    return;
  }
  double v = 0.0;
  for (int j = threadIdx.x; j < nblk; j += blockDim.x) v += partial[(size_t)b * nblk + j];
  v = block_sum256(v);
  if (threadIdx.x == 0) {
    CgState s = st[b];
    s.beta = v / s.rs;
    s.rs = v;
    s.iters += 1;
    s.stepped = 1;
    s.done = (sqrt(s.rs) / s.bnorm <= tol || s.iters >= max_iters) ? 1 : 0;
    st[b] = s;
  }
}

// p = r + beta p for the images that stepped
__global__ void __launch_bounds__(256)
cg_dir_kernel(float* __restrict__ p, const float* __restrict__ r, size_t n, const CgState* st) {
  const int b = blockIdx.y;
  if (!st[b].stepped) return;
  const double beta = st[b].beta;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const size_t o = (size_t)b * n + i;
    p[o] = (float)((double)r[o] + beta * (double)p[o]);
  }
}

// standard PnP-ADMM elementwise steps (solver.py:313-321)
__global__ void __launch_bounds__(256)
admm_std_rhs_kernel(float* __restrict__ rhs, const float* __restrict__ atb,
                    const float* __restrict__ v, const float* __restrict__ u, size_t n,
                    double rho) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) rhs[i] = (float)((double)atb[i] + rho * ((double)v[i] - (double)u[i]));
}

__global__ void __launch_bounds__(256)
admm_std_z_kernel(float* __restrict__ z, const float* __restrict__ x, const float* __restrict__ u,
                  size_t n, int* flags) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  int f = 0;
  if (i < n) {
    const float xv = x[i];
    const float zv = (float)((double)xv + (double)u[i]);
    if (!isfinite(xv)) f |= 1;
    if (!isfinite(zv)) f |= 2;
    z[i] = zv;
  }
  flags_or(flags, f);
}

// stats[b*4 + k] = sum_j part[b][j][k], k < 3 (fixed order)
int reduce_stats3(pnp_ctx* ctx, const double* part, int nblk, int batch, double* stats) {
  {
    ProfScope prof_(ctx, PROF_ADMM);
    reduce_partials_kernel<<<dim3(batch, 3), 256, 0, ctx->stream>>>(part, nblk, 3, 1.0, stats, 4);
  }
  PNP_LAUNCH_CHECK("reduce_partials_kernel");
  return PNP_OK;
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
  const size_t rs = sr_res_smem(factor, radius);
  PNP_CUDA(sr_smem_attr(rs, 0));
  {
    ProfScope prof_(ctx, PROF_FORWARD);
    sr_residual_kernel<<<sr_res_grid(H, W, factor, batch), 256, rs, ctx->stream>>>(
        x, nullptr, y, res_full(H, factor), W, factor, radius, boundary, t, nullptr);
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
  const size_t as = sr_adj_smem(radius);
  PNP_CUDA(sr_smem_attr(0, as));
  {
    ProfScope prof_(ctx, PROF_FORWARD);
    sr_adjoint_kernel<ADJ_PLAIN><<<sr_adj_grid(H, W, batch), 256, as, ctx->stream>>>(
        y, x, adj_full(H, factor), W, factor, radius, boundary, t, XUpd{}, CgEpi{});
  }
  PNP_LAUNCH_CHECK("sr_adjoint_kernel");
  return PNP_OK;
}

static int sr_grad_impl(pnp_ctx* ctx, const float* x, const float* yobs, float* grad, int batch,
                        int H, int W, const float* taps, int radius, int factor, int boundary,
                        double* data_out, const XUpd* xu) {
  if (!ctx || !x || !yobs || (!grad && !xu)) return fail(PNP_EINVAL, "null argument");
  Taps t;
  int rc = sr_check(batch, H, W, taps, radius, factor, boundary, t);
  if (rc) return rc;
  const int nl = (H / factor) * (W / factor);
  const dim3 rg = sr_res_grid(H, W, factor, batch);
  const int nblk = rg.x * rg.y;
  if ((rc = ctx->kx.ensure((size_t)batch * nl * sizeof(float)))) return rc;
  if (data_out && (rc = ensure_partials(ctx, (size_t)batch * nblk))) return rc;
  float* r = ctx->kx.as<float>();
  double* part = data_out ? ctx->stats.as<double>() : nullptr;
  const size_t rs = sr_res_smem(factor, radius), as = sr_adj_smem(radius);
  PNP_CUDA(sr_smem_attr(rs, as));
  {
    ProfScope prof_(ctx, PROF_FORWARD);
    PNP_CUDA(launch_pdl(sr_residual_kernel, rg, dim3(256), rs, ctx->stream, x, yobs, r,
                        res_full(H, factor), W, factor, radius, boundary, t, part,
                        (const CgState*)nullptr));
  }
  PNP_LAUNCH_CHECK("sr_residual_kernel");
  // the data term 0.5 ||r||^2 is reduced by the adjoint kernel's first CTA
  const RedEpi red{part, data_out, 0.5, nblk, batch};
  {
    ProfScope prof_(ctx, PROF_FORWARD);
    if (xu)
      PNP_CUDA(launch_pdl(sr_adjoint_kernel<ADJ_XUPD>, sr_adj_grid(H, W, batch), dim3(256), as,
                          ctx->stream, (const float*)r, (float*)nullptr, adj_full(H, factor), W,
                          factor, radius, boundary, t, *xu, CgEpi{}, red));
    else
      PNP_CUDA(launch_pdl(sr_adjoint_kernel<ADJ_PLAIN>, sr_adj_grid(H, W, batch), dim3(256), as,
                          ctx->stream, (const float*)r, grad, adj_full(H, factor), W, factor,
                          radius, boundary, t, XUpd{}, CgEpi{}, red));
  }
  PNP_LAUNCH_CHECK("sr_adjoint_kernel");
  return PNP_OK;
}

static int qis_grad_impl(pnp_ctx* ctx, const float* x, const float* ones, const float* zeros,
                         float* grad, int batch, int n, double gain_over_K, double floor_,
                         double* data_out, const XUpd* xu) {
  if (!ctx || !x || !ones || !zeros || (!grad && !data_out && !xu))
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
    if (xu)
      PNP_CUDA(launch_pdl(qis_grad_kernel<true>, dim3(nblk, batch), dim3(256), 0, ctx->stream, x,
                          ones, zeros, (float*)nullptr, (size_t)n, gain_over_K, floor_, part,
                          *xu));
    else
      PNP_CUDA(launch_pdl(qis_grad_kernel<false>, dim3(nblk, batch), dim3(256), 0, ctx->stream,
                          x, ones, zeros, grad, (size_t)n, gain_over_K, floor_, part, XUpd{}));
  }
  PNP_LAUNCH_CHECK("qis_grad_kernel");
  if (data_out) {
    {
      ProfScope prof_(ctx, PROF_ADMM);
      reduce_partials_kernel<<<dim3(batch, 1), 256, 0, ctx->stream>>>(part, nblk, 1, 1.0, data_out, 1);
    }
    PNP_LAUNCH_CHECK("reduce_partials_kernel");
  }
  return PNP_OK;
}

int pnp_sr_grad(pnp_ctx* ctx, const float* x, const float* yobs, float* grad, int batch, int H,
                int W, const float* taps, int radius, int factor, int boundary, double* data_out) {
  return sr_grad_impl(ctx, x, yobs, grad, batch, H, W, taps, radius, factor, boundary, data_out,
                      nullptr);
}

static XUpd make_xupd(float* x, const float* v, const float* u, float* z, double mu, double alpha,
                      double rho, double lo, double hi, int* flags) {
  XUpd q;
  q.x = x;
  q.v = v;
  q.u = u;
  q.z = z;
  q.mu = mu;
  q.alpha = alpha;
  q.rho = rho;
  q.lo = isinf(lo) ? -INFINITY : (float)lo;
  q.hi = isinf(hi) ? INFINITY : (float)hi;
  q.flags = flags;
  return q;
}

int pnp_sr_grad_xupdate(pnp_ctx* ctx, float* x, const float* yobs, int batch, int H, int W,
                        const float* taps, int radius, int factor, int boundary, double* data_out,
                        const float* v, const float* u, float* z, double mu, double alpha,
                        double rho, double lo, double hi, int* flags) {
  if (!v || !u || !z || !flags) return fail(PNP_EINVAL, "null argument");
  const XUpd q = make_xupd(x, v, u, z, mu, alpha, rho, lo, hi, flags);
  return sr_grad_impl(ctx, x, yobs, nullptr, batch, H, W, taps, radius, factor, boundary,
                      data_out, &q);
}

int pnp_qis_grad(pnp_ctx* ctx, const float* x, const float* ones, const float* zeros, float* grad,
                 int batch, int n, double gain_over_K, double floor_, double* data_out) {
  return qis_grad_impl(ctx, x, ones, zeros, grad, batch, n, gain_over_K, floor_, data_out,
                       nullptr);
}

int pnp_qis_grad_xupdate(pnp_ctx* ctx, float* x, const float* ones, const float* zeros, int batch,
                         int n, double gain_over_K, double floor_, double* data_out,
                         const float* v, const float* u, float* z, double mu, double alpha,
                         double rho, double lo, double hi, int* flags) {
  if (!v || !u || !z || !flags) return fail(PNP_EINVAL, "null argument");
  const XUpd q = make_xupd(x, v, u, z, mu, alpha, rho, lo, hi, flags);
  return qis_grad_impl(ctx, x, ones, zeros, nullptr, batch, n, gain_over_K, floor_, data_out,
                       &q);
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
    qis_grad_kernel<false><<<dim3(nblk, batch), 256, 0, ctx->stream>>>(
        x, ones, zeros, nullptr, (size_t)n, gain_over_K, floor_, part, XUpd{});
  }
  PNP_LAUNCH_CHECK("qis_grad_kernel");
  reduce_partials_kernel<<<dim3(batch, 1), 256, 0, ctx->stream>>>(part, nblk, 1, 1.0, data_out, 1);
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
  return reduce_stats3(ctx, part, nblk, batch, stats);
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


int pnp_flag_nonfinite(pnp_ctx* ctx, const float* x, int64_t n, int* flag) {
  if (!ctx || !x || !flag || n < 0) return fail(PNP_EINVAL, "null argument");
  if (((uintptr_t)x & 15) != 0) return fail(PNP_EINVAL, "x must be 16-byte aligned");
  {
    ProfScope prof_(ctx, PROF_CHECK);
    nonfinite_kernel<<<ctx->sms * 8, 256, 0, ctx->stream>>>(x, (size_t)n, flag);
  }
  PNP_LAUNCH_CHECK("nonfinite_kernel");
  return PNP_OK;
}

int pnp_check_finite(pnp_ctx* ctx, const float* x, int64_t n, int* all_finite) {
  if (!ctx || !x || !all_finite || n < 0) return fail(PNP_EINVAL, "null argument");
  if (((uintptr_t)x & 15) != 0) return fail(PNP_EINVAL, "x must be 16-byte aligned");
  int rc;
  if ((rc = ctx->flags.ensure(sizeof(int)))) return rc;
  int* f = ctx->flags.as<int>();
  PNP_CUDA(cudaMemsetAsync(f, 0, sizeof(int), ctx->stream));
  const int blocks = ctx->sms * 8;
  {
    ProfScope prof_(ctx, PROF_CHECK);
    nonfinite_kernel<<<blocks, 256, 0, ctx->stream>>>(x, (size_t)n, f);
  }
  PNP_LAUNCH_CHECK("nonfinite_kernel");
  int h = 0;
  PNP_CUDA(cudaMemcpyAsync(&h, f, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  PNP_CUDA(cudaStreamSynchronize(ctx->stream));
  *all_finite = h ? 0 : 1;
  return PNP_OK;
}


int pnp_splitmix_uniforms(pnp_ctx* ctx, uint64_t state, int64_t n, double* out) {
  if (!ctx || (!out && n > 0) || n < 0) return fail(PNP_EINVAL, "null argument");
  if (n == 0) return PNP_OK;
  const size_t need = ((size_t)n + 255) / 256;
  const int blocks = (int)std::min<size_t>(need, (size_t)ctx->sms * 16);
  {
    ProfScope prof_(ctx, PROF_FORWARD);
    splitmix_uniform_kernel<<<blocks, 256, 0, ctx->stream>>>(state, (size_t)n, out);
  }
  PNP_LAUNCH_CHECK("splitmix_uniform_kernel");
  return PNP_OK;
}

int pnp_sr_add_noise(pnp_ctx* ctx, const float* y, int64_t n, uint64_t seed, double sigma,
                     float* out32, double* out64) {
  if (!ctx || n < 0 || (n > 0 && (!y || (!out32 && !out64))))
    return fail(PNP_EINVAL, "null argument");
  if (!(sigma >= 0.0)) return fail(PNP_EINVAL, "noise_sigma must be >= 0");
  if (n == 0) return PNP_OK;
  const size_t need = ((size_t)n + 511) / 512;
  const int blocks = (int)std::min<size_t>(need, (size_t)ctx->sms * 16);
  {
    ProfScope prof_(ctx, PROF_FORWARD);
    sr_noise_kernel<<<blocks, 256, 0, ctx->stream>>>(y, (size_t)n, seed, sigma, out32, out64);
  }
  PNP_LAUNCH_CHECK("sr_noise_kernel");
  return PNP_OK;
}


int pnp_sr_gram(pnp_ctx* ctx, const float* x, float* out, int batch, int H, int W,
                const float* taps, int radius, int factor, int boundary, double shift) {
  if (!ctx || !x || !out) return fail(PNP_EINVAL, "null argument");
  Taps t;
  int rc = sr_check(batch, H, W, taps, radius, factor, boundary, t);
  if (rc) return rc;
  const dim3 rg = sr_res_grid(H, W, factor, batch), ag = sr_adj_grid(H, W, batch);
  const size_t nl = (size_t)batch * (H / factor) * (W / factor);
  if ((rc = ctx->kx.ensure(nl * sizeof(float)))) return rc;
  if ((rc = ensure_partials(ctx, (size_t)batch * ag.x * ag.y))) return rc;
  const size_t rs = sr_res_smem(factor, radius), as = sr_adj_smem(radius);
  PNP_CUDA(sr_smem_attr(rs, as));
  float* lr = ctx->kx.as<float>();
  {
    ProfScope prof_(ctx, PROF_FORWARD);
    sr_residual_kernel<<<rg, 256, rs, ctx->stream>>>(x, nullptr, lr, res_full(H, factor), W,
                                                     factor, radius, boundary, t, nullptr);
    sr_adjoint_kernel<ADJ_CG><<<ag, 256, as, ctx->stream>>>(
        lr, out, adj_full(H, factor), W, factor, radius, boundary, t, XUpd{},
        CgEpi{x, shift, ctx->stats.as<double>(), nullptr});
  }
  PNP_LAUNCH_CHECK("sr_gram");
  return PNP_OK;
}

int pnp_sr_cg(pnp_ctx* ctx, const float* rhs, float* x, int batch, int H, int W,
              const float* taps, int radius, int factor, int boundary, double shift, double tol,
              int max_iters, int warm, int* iters_out, double* resid_out, int* status_out) {
  if (!ctx || !rhs || !x || !iters_out || !resid_out || !status_out)
    return fail(PNP_EINVAL, "null argument");
  if (!(tol > 0)) return fail(PNP_EINVAL, "tol must be > 0");
  if (max_iters < 1) return fail(PNP_EINVAL, "max_iters must be >= 1");
  Taps t;
  int rc = sr_check(batch, H, W, taps, radius, factor, boundary, t);
  if (rc) return rc;
  const size_t n = (size_t)H * W, nl = (size_t)(H / factor) * (W / factor);
  const dim3 rg = sr_res_grid(H, W, factor, batch), ag = sr_adj_grid(H, W, batch);
  const int nblk_a = ag.x * ag.y, nblk_e = (int)((n + 255) / 256);
  // scratch: r, p, Ap (hi-res), A p (lo-res), partials, per-image state
  if ((rc = ctx->cg.ensure((3 * n * batch + nl * batch) * sizeof(float) +
                           (size_t)batch * sizeof(CgState) + 256)))
    return rc;
  const int np = (nblk_a > nblk_e ? nblk_a : nblk_e) * 2;
  if ((rc = ensure_partials(ctx, (size_t)batch * np))) return rc;
  float* r = ctx->cg.as<float>();
  float* p = r + n * batch;
  float* ap = p + n * batch;
  float* lr = ap + n * batch;
  CgState* st = reinterpret_cast<CgState*>(
      (reinterpret_cast<uintptr_t>(lr + nl * batch) + 255) & ~(uintptr_t)255);
  double* part = ctx->stats.as<double>();
  const size_t rsm = sr_res_smem(factor, radius), asm_ = sr_adj_smem(radius);
  PNP_CUDA(sr_smem_attr(rsm, asm_));
  ProfScope prof_(ctx, PROF_ADMM);
  if (warm) {
    if ((rc = pnp_sr_gram(ctx, x, ap, batch, H, W, taps, radius, factor, boundary, shift)))
      return rc;
  }
  cg_init_kernel<<<dim3(nblk_e, batch), 256, 0, ctx->stream>>>(rhs, warm ? ap : nullptr, x, r,
                                                                p, n, part);
  cg_start_kernel<<<batch, 256, 0, ctx->stream>>>(part, nblk_e, st, tol, max_iters);
  PNP_LAUNCH_CHECK("cg_start");
  std::vector<CgState> host(batch);
  int it = 0;
  int chunk = 4;
  while (it < max_iters) {
    const int m = (max_iters - it) < chunk ? (max_iters - it) : chunk;
    for (int k = 0; k < m; ++k) {
      sr_residual_kernel<<<rg, 256, rsm, ctx->stream>>>(p, nullptr, lr, res_full(H, factor), W,
                                                        factor, radius, boundary, t, nullptr, st);
      sr_adjoint_kernel<ADJ_CG><<<ag, 256, asm_, ctx->stream>>>(
          lr, ap, adj_full(H, factor), W, factor, radius, boundary, t, XUpd{},
          CgEpi{p, shift, part, st});
      cg_curv_kernel<<<batch, 256, 0, ctx->stream>>>(part, nblk_a, st);
      cg_update_kernel<<<dim3(nblk_e, batch), 256, 0, ctx->stream>>>(x, r, p, ap, n, st, part);
      cg_step_kernel<<<batch, 256, 0, ctx->stream>>>(part, nblk_e, st, tol, max_iters);
      cg_dir_kernel<<<dim3(nblk_e, batch), 256, 0, ctx->stream>>>(p, r, n, st);
    }
    PNP_LAUNCH_CHECK("cg iteration");
    it += m;
    PNP_CUDA(cudaMemcpyAsync(host.data(), st, batch * sizeof(CgState), cudaMemcpyDeviceToHost,
                             ctx->stream));
    PNP_CUDA(cudaStreamSynchronize(ctx->stream));
    bool all = true;
    for (int b = 0; b < batch; ++b) all = all && host[b].done;
    if (all) break;
    if (chunk < 16) chunk *= 2;
  }
  for (int b = 0; b < batch; ++b) {
    const CgState& s = host[b];
    iters_out[b] = s.iters;
    status_out[b] = s.status;
    if (s.bnorm == 0.0) {
      resid_out[b] = 0.0;
      PNP_CUDA(cudaMemsetAsync(x + (size_t)b * n, 0, n * sizeof(float), ctx->stream));
    } else {
      resid_out[b] = sqrt(s.rs) / s.bnorm;
    }
  }
  return PNP_OK;
}


int pnp_admm_std_rhs(pnp_ctx* ctx, float* rhs, const float* atb, const float* v, const float* u,
                     int64_t n, double rho) {
  if (!ctx || !rhs || !atb || !v || !u) return fail(PNP_EINVAL, "null argument");
  ProfScope prof_(ctx, PROF_ADMM);
  admm_std_rhs_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(rhs, atb, v, u,
                                                                            (size_t)n, rho);
  PNP_LAUNCH_CHECK("admm_std_rhs_kernel");
  return PNP_OK;
}

int pnp_admm_std_z(pnp_ctx* ctx, float* z, const float* x, const float* u, int64_t n,
                   int* flags) {
  if (!ctx || !z || !x || !u || !flags) return fail(PNP_EINVAL, "null argument");
  ProfScope prof_(ctx, PROF_ADMM);
  admm_std_z_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(z, x, u, (size_t)n,
                                                                          flags);
  PNP_LAUNCH_CHECK("admm_std_z_kernel");
  return PNP_OK;
}


// ---- row-strip SR operators for sharded ADMM (batch 1, one window) ----
int pnp_sr_strip_residual(pnp_ctx* ctx, const float* x, const float* y, float* r, int Hg, int W,
                          int in_r0, int in_rows, int out_r0, int out_rows, const float* taps,
                          int radius, int factor, int boundary, double* data_out) {
  if (!ctx || !x || !r) return fail(PNP_EINVAL, "null argument");
  Taps t;
  int rc = sr_check(1, Hg, W, taps, radius, factor, boundary, t);
  if (rc) return rc;
  if (out_rows < 1 || out_r0 < 0 || (out_r0 + out_rows) * factor > Hg || in_r0 < 0 ||
      in_r0 + in_rows > Hg)
    return fail(PNP_EINVAL, "bad strip window");
  const dim3 rg = sr_res_grid(out_rows * factor, W, factor, 1);
  const int nblk = rg.x * rg.y;
  double* part = nullptr;
  if (data_out) {
    if ((rc = ensure_partials(ctx, nblk))) return rc;
    part = ctx->stats.as<double>();
  }
  const size_t rs = sr_res_smem(factor, radius);
  PNP_CUDA(sr_smem_attr(rs, 0));
  {
    ProfScope prof_(ctx, PROF_FORWARD);
    sr_residual_kernel<<<rg, 256, rs, ctx->stream>>>(
        x, y, r, SrWin{Hg, in_r0, in_rows, out_r0, out_rows}, W, factor, radius, boundary, t,
        part);
    if (data_out)
      reduce_partials_kernel<<<dim3(1, 1), 256, 0, ctx->stream>>>(part, nblk, 1, 0.5, data_out, 1);
  }
  PNP_LAUNCH_CHECK("sr_strip_residual");
  return PNP_OK;
}

int pnp_sr_strip_adjoint(pnp_ctx* ctx, const float* r, float* out, int Hg, int W, int in_r0,
                         int in_rows, int out_r0, int out_rows, const float* taps, int radius,
                         int factor, int boundary) {
  if (!ctx || !r || !out) return fail(PNP_EINVAL, "null argument");
  Taps t;
  int rc = sr_check(1, Hg, W, taps, radius, factor, boundary, t);
  if (rc) return rc;
  if (out_rows < 1 || out_r0 < 0 || out_r0 + out_rows > Hg || in_r0 < 0 ||
      (in_r0 + in_rows) * factor > Hg)
    return fail(PNP_EINVAL, "bad strip window");
  const size_t as = sr_adj_smem(radius);
  PNP_CUDA(sr_smem_attr(0, as));
  {
    ProfScope prof_(ctx, PROF_FORWARD);
    sr_adjoint_kernel<ADJ_PLAIN><<<sr_adj_grid(out_rows, W, 1), 256, as, ctx->stream>>>(
        r, out, SrWin{Hg, in_r0, in_rows, out_r0, out_rows}, W, factor, radius, boundary, t,
        XUpd{}, CgEpi{});
  }
  PNP_LAUNCH_CHECK("sr_strip_adjoint");
  return PNP_OK;
}

}  // extern "C"

namespace pnp {

// pnp_admm_run for the SR model, pipelined: iteration k+1's residual
// r = A x_k - y needs only x_k, so it runs on a side stream while iteration
// k's denoiser (frozen apply + u-update) runs on the main stream; the adjoint
// + x-update of k+1 waits for it.  Same kernels with the same arguments as
// pnp_sr_grad_xupdate + pnp_dsg_apply_admm per iteration (bitwise equal);
// the residual uses its own r / partial buffers (the apply's statistics
// partials live in ctx->stats).
int sr_admm_pipelined(pnp_ctx* ctx, const float* y, int batch, int H, int W, const float* taps,
                      int radius, int factor, int boundary, const pnp_frozen* fz, int k0, int k1,
                      float* x, float* v0, float* v1, float* u, float* z, const float* gt,
                      double mu, double alpha, double rho, double lo, double hi, double* stats,
                      double* objv, int* flags, std::vector<cudaEvent_t>* timing, int* v_last) {
  Taps t;
  int rc = sr_check(batch, H, W, taps, radius, factor, boundary, t);
  if (rc) return rc;
  if (!ctx->side) {
    PNP_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
    PNP_CUDA(cudaEventCreateWithFlags(&ctx->ev_x, cudaEventDisableTiming));
    PNP_CUDA(cudaEventCreateWithFlags(&ctx->ev_g, cudaEventDisableTiming));
  }
  const int nl = (H / factor) * (W / factor);
  const dim3 rg = sr_res_grid(H, W, factor, batch), ag = sr_adj_grid(H, W, batch);
  const int nblk = rg.x * rg.y;
  if ((rc = ctx->admm_r.ensure((size_t)batch * nl * sizeof(float)))) return rc;
  if ((rc = ctx->admm_part.ensure((size_t)batch * nblk * sizeof(double)))) return rc;
  float* r = ctx->admm_r.as<float>();
  double* part = objv ? ctx->admm_part.as<double>() : nullptr;
  const size_t rsm = sr_res_smem(factor, radius), asm_ = sr_adj_smem(radius);
  PNP_CUDA(sr_smem_attr(rsm, asm_));
  const cudaStream_t main = ctx->stream, side = ctx->side;
  auto residual = [&](cudaStream_t st) {
    return launch_pdl(sr_residual_kernel, rg, dim3(256), rsm, st, x, y, r, res_full(H, factor), W,
                      factor, radius, boundary, t, part, (const CgState*)nullptr);
  };
  // iteration k0's gradient + x-update on the main stream (x is x_{k0-1})
  if ((rc = ctx->admm_g.ensure((size_t)batch * H * W * sizeof(float)))) return rc;
  float* grad = ctx->admm_g.as<float>();
  PNP_CUDA(residual(main));
  float* vcur = v0;
  float* vnext = v1;
  {
    double* obj = (objv && k0 >= 2) ? objv + (size_t)(k0 - 2) * batch : nullptr;
    const XUpd q = make_xupd(x, vcur, u, z, mu, alpha, rho, lo, hi, flags + (k0 - 1));
    const RedEpi red{part, obj, 0.5, nblk, batch};
    PNP_CUDA(launch_pdl(sr_adjoint_kernel<ADJ_XUPD>, ag, dim3(256), asm_, main, (const float*)r,
                        (float*)nullptr, adj_full(H, factor), W, factor, radius, boundary, t, q,
                        CgEpi{}, red));
  }
  int cur = 0;
  for (int k = k0; k <= k1; ++k) {
    Nvtx iter("admm_iteration");
    int* fk = flags + (k - 1);
    if (k < k1) {
      // the gradient of x_k (residual + adjoint, and the data term f(x_k)) on
      // the side stream while the main stream denoises; the apply's fixup
      // then performs iteration k+1's x-update
      PNP_CUDA(cudaEventRecord(ctx->ev_x, main));
      PNP_CUDA(cudaStreamWaitEvent(side, ctx->ev_x, 0));
      PNP_CUDA(residual(side));
      double* obj = objv ? objv + (size_t)(k - 1) * batch : nullptr;
      const RedEpi red{part, obj, 0.5, nblk, batch};
      PNP_CUDA(launch_pdl(sr_adjoint_kernel<ADJ_PLAIN>, ag, dim3(256), asm_, side,
                          (const float*)r, grad, adj_full(H, factor), W, factor, radius, boundary,
                          t, XUpd{}, CgEpi{}, red));
      PNP_CUDA(cudaEventRecord(ctx->ev_g, side));
      const AdmmXNext xn{grad, mu, alpha, lo, hi, flags + k, ctx->ev_g};
      if ((rc = dsg_apply_admm_x(ctx, fz, z, vnext, u, x, vcur, gt, rho,
                                 stats + (size_t)(k - 1) * batch * 4, fk, &xn)))
        return rc;
    } else if ((rc = pnp_dsg_apply_admm(ctx, fz, z, vnext, u, x, vcur, gt, rho,
                                        stats + (size_t)(k - 1) * batch * 4, fk))) {
      return rc;
    }
    float* tmp = vcur;
    vcur = vnext;
    vnext = tmp;
    cur ^= 1;
    if (timing) PNP_CUDA(cudaEventRecord((*timing)[k - k0 + 1], main));
  }
  if (v_last) *v_last = cur;
  return PNP_OK;
}

}  // namespace pnp
