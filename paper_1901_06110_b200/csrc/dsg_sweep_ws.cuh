// Warp-specialized variant of the recomputing sweep (sweep A: mass, C = 1;
// modes RECOMPUTE / STORE) for sm_100a.
//
// dsg_sweep_kernel runs phase 1 (squared differences + horizontal filter) and
// phase 2 (vertical filter, ex2, near / far accumulation) back to back with
// all four warps and a CTA barrier between them.  Here a CTA has eight warps:
//   warps 4-7 (producers)  phase 1 of chunk i into H buffer i & 1
//   warps 0-3 (consumers)  phase 2 of chunk i from H buffer i & 1
// handing buffers over with named barriers (FULL: producers arrive, consumers
// wait; EMPTY: consumers arrive, producers wait), so phase 1 of chunk i+1
// overlaps phase 2 of chunk i inside the CTA.  setmaxnreg moves registers
// from the producers (few live values) to the consumers (the accumulators).
// Every float is computed by the same expression in the same order as in
// dsg_sweep_kernel (same per-thread mappings, same flush protocol: the FULL
// wait plays the old mid-chunk barrier, a consumer-only barrier the old
// chunk-end one), so results are bitwise identical.
#pragma once

#include "dsg_sweep.cuh"

namespace pnp {

constexpr int kWsThreads = 256;

template <int P, int RB, int MODE>
struct CfgWs {
  using K = Cfg<P, RB, 1, MODE>;
  static constexpr int HB = kKY * 32 * K::HS;              // floats of one H buffer
  static constexpr int OFF_H2 = (K::TOTAL + 3) & ~3;       // second H buffer
  static constexpr int TOTAL = OFF_H2 + HB;
};

// named barriers with immediate ids (1, 2: FULL of buffer 0 / 1; 3, 4: EMPTY;
// 5: consumers only)
template <int ID, int NT>
__device__ __forceinline__ void named_sync() {
  asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(NT) : "memory");
}
template <int ID, int NT>
__device__ __forceinline__ void named_arrive() {
  asm volatile("bar.arrive %0, %1;" ::"n"(ID), "n"(NT) : "memory");
}

template <int P, int RB, int MODE>
__global__ void __launch_bounds__(kWsThreads, 2)
dsg_sweep_ws_kernel(const SweepArgs a, const ChunkTab<RB> tab) {
  constexpr int C = 1;
  using K = Cfg<P, RB, C, MODE>;
  using KW = CfgWs<P, RB, MODE>;
  constexpr bool STORE = MODE == MODE_STORE;
  constexpr int p = K::p, TH = K::TH, N = K::N, SEG = K::SEG, SEGW = K::SEGW, KY = K::KY;
  constexpr int WIN = K::WIN, GS = K::GS, GC = K::GC, GR = K::GR, HS = K::HS;
  constexpr int YC = K::YC, YR = K::YR, AR = K::AR;
  static_assert(MODE != MODE_CACHED, "the warp-specialized sweep recomputes the filter");
  static_assert(kTW / SEG == 4, "four producer warps, one phase-1 segment each");
  extern __shared__ float smem[];
  float* Gs = smem;
  float* Ys = smem + K::OFF_Y;
  float* As = smem + K::OFF_A;

  const int R = a.R;
  const int Hg = a.Hg, W = a.W, br0 = a.buf_r0, brows = a.buf_rows;
  const int tile = blockIdx.x;
  const int tyl = tile / a.tiles_x, tx = tile - tyl * a.tiles_x;
  const int r0g = (a.tr0 + tyl) * TH, c0g = tx * kTW;
  const size_t plane = (size_t)brows * W;
  const int b = blockIdx.z;
  const float* Gimg = a.guide + (size_t)b * plane;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  constexpr int kW = kWsThreads / 32;

  // ---- prologue (all eight warps): stage guide, channel plane, clear A ----
  {
    constexpr int NJ = (GC + 31) / 32;
    int gcol[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int cc = lane + 32 * j;
      gcol[j] = cc < GC ? reflect_index(c0g - RB - p + cc, W) : -1;
    }
#pragma unroll 2
    for (int q = warp; q < GR; q += kW) {
      int lr = reflect_index(r0g - p + q, Hg) - br0;
      lr = lr < 0 ? 0 : (lr >= brows ? brows - 1 : lr);
      const float* src = Gimg + (size_t)lr * W;
      float* dst = Gs + q * GS + lane;
#pragma unroll
      for (int j = 0; j < NJ; ++j)
        if (gcol[j] >= 0) dst[32 * j] = __ldg(src + gcol[j]);
    }
  }
  {
    constexpr int NJ = (YC + 31) / 32;
    int ycol[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int cc = lane + 32 * j, gc = c0g - RB + cc;
      ycol[j] = (cc < YC) ? ((gc >= 0 && gc < W) ? gc : -1) : -2;
    }
    const float* pa = a.ch[0].a ? a.ch[0].a + (size_t)b * plane : nullptr;
    const float* pb = a.ch[0].b ? a.ch[0].b + (size_t)b * plane : nullptr;
#pragma unroll 2
    for (int r = warp; r < YR; r += kW) {
      const int gr = r0g + r, lr = gr - br0;
      const bool rv = gr < Hg && lr >= 0 && lr < brows;
      const size_t ro = (size_t)(rv ? lr : 0) * W;
      float* dst = Ys + r * YC + lane;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        if (ycol[j] == -2) continue;
        float v = 0.f;
        if (rv && ycol[j] >= 0) {
          v = 1.f;
          if (pa) v = __ldg(pa + ro + ycol[j]);
          if (pb) v = __fmul_rn(v, __ldg(pb + ro + ycol[j]));
        }
        dst[32 * j] = v;
      }
    }
  }
  for (int i = tid; i < C * AR * YC; i += kWsThreads) As[i] = 0.f;
  const int cbeg = tab.grp[blockIdx.y], cend = tab.grp[blockIdx.y + 1];
  constexpr int HPF = TH * kTW;
  const float* kimg = STORE ? a.kcache + (long long)b * a.kc_img + (long long)tile * a.kc_tile
                            : nullptr;
  __syncthreads();

  // near accumulators (consumers) live across the role split; declared here
  // so the epilogue after the final barrier can read them
  float near[N];
  const int c = tid & (kTW - 1);  // consumer column
  const int g = (tid >> 6) & 1;   // consumer row group
  const int r0 = g * N;

  if (warp >= 4) {
    // ======================= producers: phase 1 =========================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 96;");
    const int c0 = SEG * (warp - 4);
    float ngown[SEGW];
    {
      const float* grow = Gs + lane * GS + c0 + RB;
#pragma unroll
      for (int x = 0; x < SEGW; ++x) ngown[x] = -grow[x];
    }
    for (int ci = cbeg; ci < cend; ++ci) {
      const int buf = (ci - cbeg) & 1;
      if (ci - cbeg >= 2) {  // consumers done with it
        if (buf) named_sync<4, kWsThreads>();
        else named_sync<3, kWsThreads>();
      }
      const Chunk& chk = tab.c[ci];
      const int dx = chk.dx, dy0 = chk.dy0, kc = chk.kc;
      float2* hrow0 =
          reinterpret_cast<float2*>(smem + (buf ? KW::OFF_H2 : K::OFF_H)) + lane * HS + c0;
      const int poff = (lane + dy0) * GS + c0 + RB + dx;
#pragma unroll
      for (int kp = 0; kp < KY / 2; ++kp) {
        if (kp == 0 || 2 * kp < kc) {
          float2 dd[SEGW];
#pragma unroll
          for (int x = 0; x < SEGW; ++x) {
            const float* pa = Gs + poff + 2 * kp * GS;
            const float2 t = __fadd2_rn(make_float2(pa[x], pa[GS + x]),
                                        make_float2(ngown[x], ngown[x]));
            dd[x] = __fmul2_rn(t, t);
          }
#pragma unroll
          for (int i = 0; i < SEG; ++i) {
            float2 h = __fmul2_rn(make_float2(a.taps_h[0], a.taps_h[0]), dd[i]);
#pragma unroll
            for (int bb = 1; bb < P; ++bb)
              h = __ffma2_rn(make_float2(a.taps_h[bb], a.taps_h[bb]), dd[i + bb], h);
            hrow0[kp * 32 * HS + i] = h;
          }
        }
      }
      if (buf) named_arrive<2, kWsThreads>();  // H[buf] filled
      else named_arrive<1, kWsThreads>();
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 128;");
  } else {
    // ======================= consumers: phase 2 =========================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 160;");
    float yown[N];
#pragma unroll
    for (int r = 0; r < N; ++r) {
      yown[r] = Ys[(r0 + r) * YC + c + RB];
      near[r] = (blockIdx.y == 0) ? yown[r] : 0.f;  // self pair, k = hat = 1
    }
    float2 pf[WIN - 1];
    float* pend = nullptr;
    float pendv[KY - 1];
    for (int ci = cbeg; ci < cend; ++ci) {
      const int buf = (ci - cbeg) & 1;
      const Chunk& chk = tab.c[ci];
      const int dx = chk.dx, dy0 = chk.dy0, kc = chk.kc;
      if (g == 1 && pend) {  // shared rows of the previous chunk (see dsg_sweep_kernel)
#pragma unroll
        for (int j = 0; j < KY - 1; ++j) {
          float* pA = pend + j * YC;
          *pA = __fadd_rn(*pA, pendv[j]);
        }
      }
      if (buf) named_sync<2, kWsThreads>();  // H[buf] ready (and the old mid barrier)
      else named_sync<1, kWsThreads>();
      const float2* hcol0 =
          reinterpret_cast<const float2*>(smem + (buf ? KW::OFF_H2 : K::OFF_H)) + r0 * HS + c;
      const float* ybase = Ys + (r0 + dy0) * YC + c + dx + RB;
      float* abase = As + (r0 + dy0) * YC + c + dx + RB;
      float yw[WIN];
#pragma unroll
      for (int j = 0; j < WIN; ++j) yw[j] = ybase[j * YC];
#pragma unroll
      for (int j = 0; j < WIN - 1; ++j) pf[j] = make_float2(0.f, 0.f);
      const float* kq = STORE ? kimg + (long long)chk.koff * HPF : nullptr;
#pragma unroll
      for (int kp = 0; kp < KY / 2; ++kp) {
        if (kp == 0 || 2 * kp < kc) {
          const bool pairp = 2 * kp + 1 < kc;
          float2 kk[N];
          const float2 L = make_float2(chk.L[2 * kp], chk.L[2 * kp + 1]);
          float2 hcol[N + 2 * p];
#pragma unroll
          for (int i = 0; i < N + 2 * p; ++i) hcol[i] = hcol0[(kp * 32 + i) * HS];
#pragma unroll
          for (int r = 0; r < N; ++r) {
            float2 v = L;
#pragma unroll
            for (int aa = 0; aa < P; ++aa)
              v = __ffma2_rn(make_float2(a.taps_v[aa], a.taps_v[aa]), hcol[r + aa], v);
            kk[r] = make_float2(ex2_approx(v.x), ex2_approx(v.y));
            if (STORE) {
              float* kpl = const_cast<float*>(kq) + 2 * kp * HPF;
              if (pairp) {
                float2* dst = reinterpret_cast<float2*>(kpl) + r0 * kTW + kpos<N>(c, r & ~1);
                if (r & 1)
                  __stcs(reinterpret_cast<float4*>(dst),
                         make_float4(kk[r - 1].x, kk[r - 1].y, kk[r].x, kk[r].y));
                else if (r == N - 1)
                  __stcs(dst, kk[r]);
              } else {
                float* dst = kpl + r0 * kTW + kpos<N>(c, r & ~1);
                if (r & 1)
                  __stcs(reinterpret_cast<float2*>(dst), make_float2(kk[r - 1].x, kk[r].x));
                else if (r == N - 1)
                  __stcs(dst, kk[r].x);
              }
            }
          }
#pragma unroll
          for (int r = 0; r < N; ++r) {
            near[r] = __fmaf_rn(kk[r].x, yw[r + 2 * kp], near[r]);
            near[r] = __fmaf_rn(kk[r].y, yw[r + 2 * kp + 1], near[r]);
            pf[r + 2 * kp] = __ffma2_rn(kk[r], make_float2(yown[r], yown[r]), pf[r + 2 * kp]);
          }
        }
      }
      // H[buf] fully read: the producers may refill it (chunk ci + 2)
      if (ci + 2 < cend) {
        if (buf) named_arrive<4, kWsThreads>();
        else named_arrive<3, kWsThreads>();
      }
      if (g == 0) {
#pragma unroll
        for (int j = 0; j < WIN; ++j) {
          float v;
          if (j == 0) v = pf[0].x;
          else if (j == WIN - 1) v = pf[WIN - 2].y;
          else v = __fadd_rn(pf[j].x, pf[j - 1].y);
          float* pA = abase + j * YC;
          *pA = __fadd_rn(*pA, v);
        }
      } else {
#pragma unroll
        for (int j = KY - 1; j < WIN; ++j) {
          float v;
          if (j == WIN - 1) v = pf[WIN - 2].y;
          else v = __fadd_rn(pf[j].x, pf[j - 1].y);
          float* pA = abase + j * YC;
          *pA = __fadd_rn(*pA, v);
        }
#pragma unroll
        for (int j = 0; j < KY - 1; ++j)
          pendv[j] = j == 0 ? pf[0].x : __fadd_rn(pf[j].x, pf[j - 1].y);
        pend = abase;
      }
      named_sync<5, 128>();  // the old chunk-end barrier (consumers only)
    }
    if (g == 1 && pend) {
#pragma unroll
      for (int j = 0; j < KY - 1; ++j) {
        float* pA = pend + j * YC;
        *pA = __fadd_rn(*pA, pendv[j]);
      }
    }
    asm volatile("setmaxnreg.dec.sync.aligned.u32 128;");
  }
  __syncthreads();

  // ---- own pixels: near + far; then emit tile + band block ----
  if (warp < 4) {
#pragma unroll
    for (int r = 0; r < N; ++r) {
      float* pA = As + (r0 + r) * YC + c + RB;
      *pA = __fadd_rn(near[r], *pA);
    }
  }
  __syncthreads();
  const int BR = TH + R, BC = kTW + 2 * R;
  const size_t slot =
      (((size_t)b * a.part_ntr + a.part_off + tyl) * gridDim.y + blockIdx.y) * a.tiles_x + tx;
  float* out = a.partial + slot * (size_t)(C * BR * BC);
  const float* A0 = As + (RB - R);
  for (int br = warp; br < BR; br += kW)
    for (int bc = lane; bc < BC; bc += 32) out[br * BC + bc] = A0[br * YC + bc];
}

}  // namespace pnp
