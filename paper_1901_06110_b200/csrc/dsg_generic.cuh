// DSG-NLM offset sweep for any patch side and search radius (sm_100a).
//
// The P-templated sweep (dsg_sweep.cuh) covers Gaussian patch weights with
// P <= 15 (box weights with P <= 9), R <= 32.  This kernel is the general one,
// and the one used for the reference's own box patch weights from P = 11 on
// (its Table-1 range, P = 11..29, in one kernel): the box patch distance
//   SSD_t(s) = sum_{a,b < P} (G(s+ab) - G(s+t+ab))^2       (denoise.py:131-158)
// is computed with running sums (a horizontal then a vertical running box
// sum over the squared-difference rows), so the cost per pixel-offset does
// not grow with P -- the property the reference gets from its summed-area
// table ("cost independent of patch_side", denoise.py:11-15; Table 1 of the
// paper).  The running sums restart every 32 columns / TH/2 rows, so fp32
// rounding never accumulates over the image (the reference itself
// mean-centres its float64 table for the same reason, denoise.py:143-157).
// Gaussian taps (patch_sigma) use the direct separable filter instead (cost
// 2P per pair).
//
// Work decomposition: one CTA per output tile (TH x 64) and offset group;
// offsets are walked dy-major.  Per dy (and per chunk of at most kGenDXC dx
// values) the partner guide rows and partner channel rows are staged into
// shared memory (reflected guide, zero channel planes outside the image), then
// per offset: phase H (thread = map row x 32-column segment: running / direct
// horizontal filter of the squared differences into an H map), phase V
// (thread = column x half of the tile rows: vertical filter, ex2 with the
// hat folded into the exponent, near-end accumulation in registers).
//
// SYM (the default): the half window only; each unordered pair credited to
// both ends, the far end into a shared-memory plane over the tile + its
// R-wide band that is written as the tile's partial block (exactly the
// P-templated kernel's block format, summed by the same fixups).  Within one
// offset every far cell has one writer; offsets are separated by barriers and
// walked in a fixed order -> no atomics, bit-reproducible.
// !SYM (search radii whose far plane does not fit in shared memory): the full
// window from each end, near sums only, a TH x 64 block per tile.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "dsg_sweep.cuh"

namespace pnp {

constexpr int kGenThreads = 128;  // 64 columns x 2 row halves in phase V
constexpr int kGenDXC = 32;       // dx values per staged chunk
constexpr int kGenMaxP = 63;      // largest patch side (shared memory)
constexpr int kGenSeg = 32;       // phase-H segment (running-sum restart)
constexpr int kGenNmax = 16;      // rows per phase-V thread (TH <= 32)

struct GenArgs {
  const float* guide;  // [B][buf_rows][W]
  ChanSpec ch[2];
  float* partial;
  const float* ltab;   // log2 hat per offset, [(dy+R)*(2R+1) + dx+R]; null: 0 (NLM)
  int Hg, W, R, P, TH;
  int buf_r0, buf_rows;
  int tr0, tiles_x;
  int part_off, part_ntr;
  float cv;                 // box: -log2(e) / (2 P^2 bw^2)
  float taps_h[kGenMaxP];   // Gaussian: normalized taps w_b
  float taps_v[kGenMaxP];   // Gaussian: -log2(e)/(2 bw^2) * w_a
  int grp[kMaxGroups + 1];  // offset groups: dy-index ranges (dy = dyi + dy_min)
  long long partial_floats;  // buffer size (PNP_CHECKS)
  // k cache (SYM, MODE STORE / CACHED): one TH x 64 plane per tile and
  // half-window offset, offsets in the sweep's walk order, tiles
  // (b, tile row of the launch, tile col) in raster order
  float* kcache;
  long long kcache_floats;  // buffer size (PNP_CHECKS)
};

// Shared-memory geometry of one CTA (floats); also used by the host to pick
// the tile height TH and the batch size KG.
struct GenSmem {
  int M, GOS, GPR, GPS, HS, YR, YS, AR, AC;
  int off_gp, off_h, off_y, off_a, total;
};

// cached: the k-cache sweep stages no guide and keeps no H map
__host__ __device__ inline GenSmem gen_smem(int TH, int P, int R, int C, bool sym, int KG,
                                            bool cached = false) {
  GenSmem s;
  const int p = (P - 1) / 2;
  s.M = TH + 2 * p;
  s.GOS = (kTW + 2 * p) | 1;
  s.GPR = s.M + KG - 1;
  s.GPS = (kTW + 2 * p + kGenDXC) | 1;
  s.HS = kTW + 1;
  s.YR = TH + KG - 1;
  s.YS = kTW + kGenDXC;
  s.AR = sym ? TH + R + KG - 1 : 0;
  s.AC = sym ? kTW + 2 * R : 0;
  s.off_gp = cached ? 0 : s.M * s.GOS;
  s.off_h = s.off_gp + (cached ? 0 : s.GPR * s.GPS);
  s.off_y = s.off_h + (cached ? 0 : KG * s.M * s.HS);
  s.off_a = s.off_y + C * s.YR * s.YS;
  s.total = s.off_a + C * s.AR * s.AC;
  return s;
}

__device__ __forceinline__ float sqd(float a, float b) {
  const float t = __fsub_rn(a, b);
  return __fmul_rn(t, t);
}

// NM: rows per phase-V thread the register arrays hold (>= TH / 2); the
// k-cache sweep is instantiated per tile height (fewer registers -> more
// resident CTAs for the stream), the others with the maximum
template <int C, bool BOX, bool SYM, int KG, int MODE, int NM = kGenNmax>
__global__ void __launch_bounds__(kGenThreads, MODE == MODE_CACHED && NM <= 8 ? 4 : 1)
    dsg_generic_kernel(const GenArgs a) {
  constexpr bool STORE = MODE == MODE_STORE, CACHED = MODE == MODE_CACHED;
  static_assert(SYM || MODE == MODE_RECOMPUTE, "the k cache covers the half window");
  pdl_begin();
  extern __shared__ float smem[];
  const int R = a.R, P = a.P, TH = a.TH, p = (P - 1) / 2;
  const GenSmem L = gen_smem(TH, P, R, C, SYM, KG, CACHED);
  float* Gown = smem;
  float* Gpart = smem + L.off_gp;
  float* Hs = smem + L.off_h;
  float* Ys = smem + L.off_y;
  float* As = smem + L.off_a;

  const int Hg = a.Hg, W = a.W, br0 = a.buf_r0, brows = a.buf_rows;
  const int tile = blockIdx.x;
  const int tyl = tile / a.tiles_x, tx = tile - tyl * a.tiles_x;
  const int r0g = (a.tr0 + tyl) * TH, c0g = tx * kTW;
  const size_t plane = (size_t)brows * W;
  const int b = blockIdx.z;
  const float* Gimg = a.guide + (size_t)b * plane;
  const int tid = threadIdx.x;
  const int M = L.M;

  auto grow = [&](int gr) {  // reflected guide row -> buffer row
    int lr = reflect_index(gr, Hg) - br0;
    return lr < 0 ? 0 : (lr >= brows ? brows - 1 : lr);
  };
  const float* pa[C];
  const float* pb[C];
#pragma unroll
  for (int c_ = 0; c_ < C; ++c_) {
    pa[c_] = a.ch[c_].a ? a.ch[c_].a + (size_t)b * plane : nullptr;
    pb[c_] = a.ch[c_].b ? a.ch[c_].b + (size_t)b * plane : nullptr;
  }
  // channel value y = a*b at global (gr, gc); +0 outside the image / buffer
  auto yval = [&](int c_, int gr, int gc) {
    const int lr = gr - br0;
    if (gr < 0 || gr >= Hg || lr < 0 || lr >= brows || gc < 0 || gc >= W) return 0.f;
    const size_t o = (size_t)lr * W + gc;
    float v = 1.f;
    if (pa[c_]) v = __ldg(pa[c_] + o);
    if (pb[c_]) v = __fmul_rn(v, __ldg(pb[c_] + o));
    return v;
  };

  // ---- own guide rows (map rows q <-> image row r0g - p + q, map col j <->
  // image col c0g - p + j), far plane cleared ----
  if (!CACHED)
    for (int q = tid / 32; q < M; q += kGenThreads / 32) {
      const float* src = Gimg + (size_t)grow(r0g - p + q) * W;
      for (int j = tid & 31; j < kTW + 2 * p; j += 32)
        Gown[q * L.GOS + j] = __ldg(src + reflect_index(c0g - p + j, W));
    }
  if (SYM)
    for (int i = tid; i < C * L.AR * L.AC; i += kGenThreads) As[i] = 0.f;

  const int x = tid & (kTW - 1), g = tid / kTW;
  const int N = TH / 2, rA = g * N;  // phase-V rows [rA, rA + N)
  float near[C][NM], yown[C][NM];
#pragma unroll
  for (int c_ = 0; c_ < C; ++c_)
#pragma unroll
    for (int i = 0; i < NM; ++i) {
      const float v = i < N ? yval(c_, r0g + rA + i, c0g + x) : 0.f;
      yown[c_][i] = v;
      near[c_][i] = blockIdx.y == 0 ? v : 0.f;  // self pair: k = hat = 1
    }

  // Far end (SYM), per batch of KG offsets (dy0 + j, dx): thread (x, g)
  // credits tile rows rA + i + dy0 + j of column x + dx; they sit in a
  // register window pf[w], w = i + j < N + KG - 1, flushed once per dx.  The
  // two row halves' windows overlap in KG - 1 rows: half 0 flushes its whole
  // window before the barrier that ends the dx step, half 1 its private rows;
  // half 1's shared rows go in after that barrier (top of the next step,
  // before the next phase-H barrier): one writer per cell between barriers,
  // a fixed order (half 0, half 1) -> bit-reproducible.
  constexpr int WIN = NM + KG - 1;
  float pf[C][SYM ? WIN : 1];
  float pendv[C][KG > 1 ? KG - 1 : 1];
  float* pend = nullptr;
  auto flush_pending = [&]() {
    if (SYM && pend) {
#pragma unroll
      for (int c_ = 0; c_ < C; ++c_)
#pragma unroll
        for (int w = 0; w < KG - 1; ++w) {
          float* q = pend + (c_ * L.AR + w) * L.AC;
          PNP_CHECK(q >= As && q < As + C * L.AR * L.AC);
          *q = __fadd_rn(*q, pendv[c_][w]);
        }
      pend = nullptr;
    }
  };

  const int dy_min = SYM ? 0 : -R;
  const int n_dx = 2 * R + 1;
  const int gend = a.grp[blockIdx.y + 1];
  // k cache: this tile's planes; kplane = planes of the offsets walked before
  // (dy = 0 has R offsets in the half window, every dy > 0 has 2R + 1)
  float* ktile = nullptr;
  int kplane = 0;
  if (STORE || CACHED) {
    const int hw = 2 * R * R + 2 * R;
    ktile = a.kcache + ((((size_t)b * (gridDim.x / a.tiles_x) + tyl) * a.tiles_x + tx) * hw) *
                           (size_t)(TH * kTW);
    const int dyf = a.grp[blockIdx.y];
    kplane = dyf == 0 ? 0 : R + (dyf - 1) * n_dx;
  }
  for (int b0 = a.grp[blockIdx.y]; b0 < gend; b0 += KG) {
    const int nb = min(KG, gend - b0);
    const int dy0 = b0 + dy_min;
    for (int dxa = -R; dxa <= R; dxa += kGenDXC) {
      const int dxb = min(dxa + kGenDXC, R + 1);
      jitter_sync();  // previous users of Gpart / Ys are done
      // partner guide rows: row q <-> image row r0g - p + q + dy0 (offset j
      // reads rows q + j), col jj <-> image col c0g - p + dxa + jj
      const int gpw = kTW + 2 * p + (dxb - dxa) - 1;
      if (!CACHED)
        for (int q = tid / 32; q < L.GPR; q += kGenThreads / 32) {
          const float* src = Gimg + (size_t)grow(r0g - p + q + dy0) * W;
          for (int jj = tid & 31; jj < gpw; jj += 32)
            Gpart[q * L.GPS + jj] = __ldg(src + reflect_index(c0g - p + dxa + jj, W));
        }
      // partner channel rows: row r <-> image row r0g + r + dy0, col jj <->
      // image col c0g + dxa + jj
      const int yw = kTW + (dxb - dxa) - 1;
#pragma unroll
      for (int c_ = 0; c_ < C; ++c_)
        for (int r = tid / 32; r < L.YR; r += kGenThreads / 32)
          for (int jj = tid & 31; jj < yw; jj += 32)
            Ys[(c_ * L.YR + r) * L.YS + jj] = yval(c_, r0g + r + dy0, c0g + dxa + jj);
      jitter_sync();

      for (int dx = dxa; dx < dxb; ++dx) {
        const int cdx = dx - dxa;
        // offsets of the batch that exist: j < nb, minus the half window's
        // (0, dx <= 0) / the full window's self pair (uniform over the CTA)
        unsigned valid = 0;
#pragma unroll
        for (int j = 0; j < KG; ++j) {
          const int dy = dy0 + j;
          const bool ok = j < nb && !(dy == 0 && (SYM ? dx <= 0 : dx == 0));
          valid |= (ok ? 1u : 0u) << j;
        }
        if (!valid) continue;
        flush_pending();
        // this step's k planes (valid offsets in order): kplane, kplane + 1, ...
        float kv[CACHED ? KG : 1][CACHED ? NM : 1];
        if (CACHED) {  // all the step's loads in flight before the sums
#pragma unroll
          for (int j = 0; j < KG; ++j) {
            const bool vj = (valid >> j) & 1u;
            const float* kq = ktile +
                              (size_t)(kplane + __popc(valid & ((1u << j) - 1u))) * (TH * kTW) +
                              rA * kTW + x;
#pragma unroll
            for (int i = 0; i < NM; ++i) {
              const bool ok = vj && i < N;
              PNP_CHECK(!ok || (long long)(kq + i * kTW - a.kcache) < a.kcache_floats);
              kv[j][i] = ok ? __ldcs(kq + i * kTW) : 0.f;
            }
          }
        }
        // ---- phase H: offset j, map row q, columns [x0, x0 + 32) ----
        for (int it = tid; it < (CACHED ? 0 : KG * 2 * M); it += kGenThreads) {
          const int j = it / (2 * M), rem = it - j * 2 * M;
          if (!((valid >> j) & 1u)) continue;
          const int x0 = (rem / M) * kGenSeg, q = rem % M;
          const float* own = Gown + q * L.GOS + x0;
          const float* part = Gpart + (q + j) * L.GPS + x0 + cdx;
          float* h = Hs + (j * M + q) * L.HS + x0;
          if (BOX) {
            float s = sqd(part[0], own[0]);
            for (int bb = 1; bb < P; ++bb) s = __fadd_rn(s, sqd(part[bb], own[bb]));
            h[0] = s;
#pragma unroll 4
            for (int i = 1; i < kGenSeg; ++i) {
              s = __fsub_rn(__fadd_rn(s, sqd(part[i + P - 1], own[i + P - 1])),
                            sqd(part[i - 1], own[i - 1]));
              h[i] = s;
            }
          } else {
#pragma unroll 2
            for (int i = 0; i < kGenSeg; ++i) {
              float s = __fmul_rn(a.taps_h[0], sqd(part[i], own[i]));
              for (int bb = 1; bb < P; ++bb)
                s = __fmaf_rn(a.taps_h[bb], sqd(part[i + bb], own[i + bb]), s);
              h[i] = s;
            }
          }
        }
        jitter_sync();
        // ---- phase V: column x, rows [rA, rA + N), the batch's offsets as
        // independent chains ----
        float Lt[KG], sv[KG];
        const float* hc[KG];
#pragma unroll
        for (int j = 0; j < KG; ++j) {
          const int dy = dy0 + j;
          Lt[j] = ((valid >> j) & 1u) ? (a.ltab ? a.ltab[(dy + R) * n_dx + dx + R] : 0.f)
                                      : -INFINITY;
          hc[j] = Hs + (j * M + rA) * L.HS + x;
          sv[j] = 0.f;
          if (BOX && !CACHED && ((valid >> j) & 1u)) {
            float s = hc[j][0];
            for (int aa = 1; aa < P; ++aa) s = __fadd_rn(s, hc[j][aa * L.HS]);
            sv[j] = s;
          }
        }
        if (SYM) {
#pragma unroll
          for (int c_ = 0; c_ < C; ++c_)
#pragma unroll
            for (int w = 0; w < WIN; ++w) pf[c_][w] = 0.f;
        }
        const float* yp = Ys + rA * L.YS + x + cdx;
#pragma unroll
        for (int i = 0; i < NM; ++i) {
          if (i >= N) break;
#pragma unroll
          for (int j = 0; j < KG; ++j) {
            if (!((valid >> j) & 1u)) continue;
            float k;
            if (CACHED) {
              k = kv[j][i];
            } else {
              float e;
              if (BOX) {
                e = __fmaf_rn(sv[j], a.cv, Lt[j]);
                if (i + 1 < N)
                  sv[j] = __fsub_rn(__fadd_rn(sv[j], hc[j][(i + P) * L.HS]), hc[j][i * L.HS]);
              } else {
                e = Lt[j];
                for (int aa = 0; aa < P; ++aa)
                  e = __fmaf_rn(a.taps_v[aa], hc[j][(i + aa) * L.HS], e);
              }
              k = ex2_approx(e);
              if (STORE) {
                float* kq = ktile +
                            (size_t)(kplane + __popc(valid & ((1u << j) - 1u))) * (TH * kTW) +
                            (rA + i) * kTW + x;
                PNP_CHECK((long long)(kq - a.kcache) < a.kcache_floats);
                __stcs(kq, k);
              }
            }
#pragma unroll
            for (int c_ = 0; c_ < C; ++c_) {
              near[c_][i] = __fmaf_rn(k, yp[(c_ * L.YR + i + j) * L.YS], near[c_][i]);
              if (SYM) pf[c_][i + j] = __fmaf_rn(k, yown[c_][i], pf[c_][i + j]);
            }
          }
        }
        if (SYM) {  // flush the window (half 1 defers its first KG - 1 rows)
          float* base = As + (rA + dy0) * L.AC + x + dx + R;
#pragma unroll
          for (int c_ = 0; c_ < C; ++c_)
#pragma unroll
            for (int w = 0; w < WIN; ++w) {
              if (w >= N + KG - 1) break;
              if (g == 1 && w < KG - 1) {
                pendv[c_][w] = pf[c_][w];
                continue;
              }
              float* q = base + (c_ * L.AR + w) * L.AC;
              PNP_CHECK(q >= As && q < As + C * L.AR * L.AC);
              *q = __fadd_rn(*q, pf[c_][w]);
            }
          if (g == 1 && KG > 1) pend = base;
        }
        if (STORE || CACHED) kplane += __popc(valid);
        jitter_sync();
      }
    }
  }
  flush_pending();
  jitter_sync();

  // ---- emit: own pixels get near + far; the block is tile + band (SYM) or
  // the tile alone ----
  const int BR = SYM ? TH + R : TH, BC = SYM ? kTW + 2 * R : kTW;
  const size_t slot =
      (((size_t)b * a.part_ntr + a.part_off + tyl) * gridDim.y + blockIdx.y) * a.tiles_x + tx;
  float* out = a.partial + slot * (size_t)(C * BR * BC);
  PNP_CHECK((long long)((slot + 1) * (size_t)(C * BR * BC)) <= a.partial_floats);
  if (SYM) {
#pragma unroll
    for (int c_ = 0; c_ < C; ++c_)
#pragma unroll
      for (int i = 0; i < NM; ++i) {
        if (i >= N) break;
        float* q = As + (c_ * L.AR + rA + i) * L.AC + x + R;
        *q = __fadd_rn(near[c_][i], *q);
      }
    __syncthreads();
    for (int c_ = 0; c_ < C; ++c_)
      for (int i = tid; i < BR * BC; i += kGenThreads)
        out[(size_t)c_ * BR * BC + i] = As[c_ * L.AR * L.AC + i];
  } else {
#pragma unroll
    for (int c_ = 0; c_ < C; ++c_)
#pragma unroll
      for (int i = 0; i < NM; ++i) {
        if (i >= N) break;
        out[((size_t)c_ * BR + rA + i) * BC + x] = near[c_][i];
      }
  }
}

// pnp_generic.cu
cudaError_t launch_generic(const GenArgs& a, int C, bool box, bool sym, int KG, int mode,
                           dim3 grid, cudaStream_t st);

}  // namespace pnp
