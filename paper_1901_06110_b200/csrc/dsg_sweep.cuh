// DSG-NLM offset sweep for sm_100a.
//
// Replaces the reference's per-offset numpy sweeps (pnprestore/denoise.py:
// _mass_sweep 207-212, _scale_sweep 215-224, _filter_sweep 227-241, and the
// distance engine 131-158 / kernel maps 191-197).  One CTA owns an output tile
// of TH x TW pixels and walks the half window of search offsets t (dy > 0, or
// dy == 0 and dx > 0).  Each unordered pair (s, s+t) is evaluated once and
// credited to both ends (K is symmetric), the self pair analytically:
//
//   near end (s in tile, register accumulator):   acc[s]   += k * y[s+t]
//   far end  (s+t in tile or its R-wide band):    A[s+t]   += k * y[s]
//
// where y is a per-channel input plane (mask / rs / rs*x) and
// k = hat(t) * exp(-sum_ab w_a w_b (G(s+ab) - G(s+t+ab))^2 / (2 bw^2)).
// Everything is ordered: near sums run over offsets in table order; far sums
// are staged per chunk in registers and flushed by exactly one thread per
// SMEM cell between __syncthreads.  No atomics -> bit-reproducible, and the
// same code computes freeze/apply/adaptive so FrozenGuide.apply is
// bit-identical to dsg_nlm_denoise (reference tests/test_denoise.py:256-268).
//
// Patch filter, per chunk of KY offsets sharing dx (consecutive dy), in
// packed f32x2 over offset pairs (k, k+1) (sm_100 FFMA2 / FADD2 / FMUL2):
//   phase 1  lane = map row q (32 rows = TH + 2p), warp = 16-column segment;
//            the own guide row segment (16+2p, negated) lives in registers for
//            the whole kernel as the broadcast operand, the two partner rows
//            are read from SMEM; (D_k, D_k+1) = (G_partner - G_own)^2, then the
//            horizontal P-tap filter -> one float2 H map per offset pair
//            (odd row stride: conflict-free 64-bit stores).
//   phase 2  thread = (column c, row group g of N rows): vertical P-tap filter
//            of the H column with the exponent scale folded into the taps and
//            (log2 hat_k, log2 hat_k+1) as the initial pair, two MUFU ex2,
//            near FFMA into registers, far FFMA2 (both offsets at once) into a
//            register window, one flush per chunk (group 0 before the chunk
//            barrier, group 1 after it: one shared far plane, no race).
// The offset table rides in the kernel parameters (constant bank); all SMEM
// strides are compile-time (R bucket RB >= R).
//
// Modes: RECOMPUTE (the fused offset loop), STORE (also writes every pair
// weight to the HBM k cache), CACHED (streams the weights back: no guide, no
// filter; C = 2 through SMEM with bulk async copies + mbarriers).  Same
// floats, same add order -> bitwise identical results in all three.
//
// The tile writes its accumulators over rows [0, TH+R) x cols [-R, TW+R)
// (tile + far band) to a partial block; the fixup kernels sum the covering
// blocks of every pixel in a fixed order.
#pragma once

#include <cuda.h>  // CUtensorMap (the driver entry point is resolved at run time)
#include <cuda_runtime.h>
#include <stdint.h>

#include "pnp_pdl.cuh"

namespace pnp {

constexpr int kTW = 64;        // tile width (output columns)
constexpr int kThreads = 128;  // 64 columns x 2 row groups in phase 2
#ifndef PNP_KY
#define PNP_KY 4
#endif
constexpr int kKY = PNP_KY;
#ifndef PNP_SB
#define PNP_SB 6  // rows per warp per batch of prologue loads (k-cache sweeps)
#endif

#ifndef PNP_KPF
#define PNP_KPF 3  // k-cache stream: chunks of L2 prefetch lead (TMA path)
#endif    // offsets per chunk (same dx, consecutive dy)
constexpr int kMaxP = 15;      // largest patch side with a fast kernel
constexpr int kMaxR = 32;      // largest search radius (R bucket)

// Sweep modes.  The pair weights k = hat*exp(.) are identical floats in all
// three, and the accumulation order is the same, so results are bitwise equal:
//   RECOMPUTE  patch filter + ex2 per pair (the fused offset-loop kernel)
//   STORE      same, and also writes every pair weight to a HBM "k cache"
//              (the reference memoizes kernel maps the same way when they fit,
//              denoise.py:27-29, 187-197)
//   CACHED     reads the pair weights from the k cache (no guide staging, no
//              filter): an HBM-streaming pass used for sweep B and frozen applies
enum SweepMode { MODE_RECOMPUTE = 0, MODE_STORE = 1, MODE_CACHED = 2 };

struct ChanSpec {
  const float* a;  // y = a * b, null factor = 1; inside the image only
  const float* b;
};

// One chunk of the half-window offset table: KY offsets (dx, dy0 + k),
// k < kc, with their log2(hat) (0 for plain NLM; -inf for k >= kc)
// precomputed on the host, and the chunk's place in a tile's k-cache run
// (koff planes of TH x 64 floats: one plane per offset).
struct Chunk {
  int dx, dy0, kc, koff;
  float L[kKY];
};

// Chunks of the half window at R = RB (the largest R of a bucket):
// dx > 0 has RB+1 dy values (0..RB), dx <= 0 has RB (1..RB).
__host__ __device__ constexpr int max_chunks(int RB) {
  return RB * ((RB + 1 + kKY - 1) / kKY) + (RB + 1) * ((RB + kKY - 1) / kKY);
}
constexpr int kMaxGroups = 64;

// The offset table travels in the kernel parameters (constant bank): every
// chunk read is a uniform constant-cache hit, never a global-memory round trip
// at the top of the chunk loop.
template <int RB>
struct ChunkTab {
  Chunk c[max_chunks(RB)];
  int grp[kMaxGroups + 1];  // NG+1 chunk starts
};

// Host view of a table (built once per (R, NG) and kept in the context).
struct HostTab {
  const Chunk* ch;
  int nch;
  const int* grp;
  int ng;
};

// Per-pixel planes are windows of the global image: rows [buf_r0, buf_r0 +
// buf_rows) of a Hg x W image (single GPU: buf_r0 = 0, buf_rows = Hg; a row
// strip on one rank of a sharded run: its rows plus halos).  The launch
// covers global tile rows [tr0, tr0 + gridDim.x / tiles_x).  Partial blocks
// go to slot (part_off + local tile row) of a [B][part_ntr][NG][tiles_x]
// array of C*(TH+R)*(TW+2R) floats; tile rows are outermost so a
// neighbour's rows can be received into a contiguous prefix.
struct SweepArgs {
  const float* guide;  // [B][buf_rows][W]
  ChanSpec ch[2];
  float* partial;
  int Hg, W, R;
  int buf_r0, buf_rows;
  int tr0, tiles_x;
  int part_off, part_ntr;
  // k cache, tile-major, exactly one float per pixel and half-window offset:
  // a tile's run is kc_tile floats; chunk ci starts koff planes (TH*64
  // floats) into it.  Offsets (2kp, 2kp+1) of a chunk share one float2 "pair
  // plane" (2 planes); an odd last offset of a chunk (kc = 1 or 3) has a
  // float "single plane".  Within either, a row group's N rows are stored
  // row-pair interleaved per column (kpos) -> 128-bit (pair) / 64-bit
  // (single) accesses, and a chunk is one contiguous kc*TH*64*4 B run.
  float* kcache;
  long long kc_img, kc_tile;
  long long partial_floats, kcache_floats;  // buffer sizes (PNP_CHECKS)
  // the launch's guide tensor map (3-D: W x buf_rows x B fp32, box GCB x GR x
  // 1) is valid: interior tiles stage their guide tile with one TMA load
  int tma;
  float taps_h[kMaxP];  // normalized patch taps w_b (phase 1)
  float taps_v[kMaxP];  // -log2(e)/(2 bw^2) * w_a (phase 2)
};

__host__ __device__ constexpr int tile_height(int P) { return 32 - (P - 1); }

__host__ __device__ constexpr int r_bucket(int R) {
  return R <= 5 ? 5 : (R <= 10 ? 10 : (R <= 16 ? 16 : 32));
}

template <int P, int RB, int C, int MODE = MODE_RECOMPUTE>
struct Cfg {
  static constexpr int p = (P - 1) / 2;
  static constexpr int TH = 32 - 2 * p;  // tile height
  static constexpr int N = TH / 2;       // rows per phase-2 thread
  static constexpr int SEG = 16;         // phase-1 segment width
  static constexpr int SEGW = SEG + 2 * p;
  static constexpr int KY = kKY;
  static constexpr int WIN = N + KY - 1;
  static constexpr int GC = kTW + 2 * (RB + p), GS = GC | 1, GR = 33 + RB;  // partner rows <= 31 + R + 1
  static constexpr int HS = kTW + 1;  // float2 units (odd: conflict-free STS.64 by row)
  static constexpr int YC = kTW + 2 * RB, YR = TH + RB + KY - 1, AR = YR;  // rows < r0 + R + WIN
  static constexpr bool CACHED = MODE == MODE_CACHED;  // no guide tile, no H maps
  static constexpr int OFF_H = CACHED ? 0 : (GR * GS + 3) & ~3;  // 16 B aligned
  static constexpr int OFF_Y = CACHED ? 0 : OFF_H + KY * 32 * HS;  // KY/2 float2 maps
  static constexpr int OFF_A = OFF_Y + C * YR * YC;
  // CACHED with C = 2 streams the k cache through SMEM: two chunk buffers
  // filled by bulk async copies (TMA engine) one chunk ahead + 2 mbarriers
  static constexpr bool TMAK = CACHED && C == 2;
  static constexpr int KCH = KY * TH * kTW;  // floats per chunk (KY offset planes)
  static constexpr int OFF_K = (OFF_A + C * AR * YC + 3) & ~3;
  static constexpr int OFF_MB = OFF_K + (TMAK ? 2 * KCH : 0);
  // guide staging by TMA (recompute / store sweeps): a dense GCB-pitch box
  // landed in the H-map / channel / far area (128-byte aligned; all staged
  // after it), then re-laid out with the odd pitch GS; one mbarrier
  // box width: the tile's GC columns from a 16-byte-aligned start column (the
  // TMA box's inner start must be 16-byte aligned: up to 3 leading columns)
  static constexpr int GCB = (GC + 3 + 3) & ~3;
  static constexpr int OFF_TB = (OFF_MB + (TMAK ? 4 : 0) + 1) & ~1;
  static constexpr int TOTAL = OFF_TB + (CACHED ? 0 : 2);  // floats
  static_assert(CACHED || OFF_TB - OFF_H >= GCB * GR + 32,
                "TMA box fits the H-map / channel / far area");
};

__device__ __forceinline__ int reflect_index(int i, int n) {
  // half-sample symmetric (np.pad mode="symmetric"; image.py:97-113),
  // clamped so out-of-range tile padding stays in bounds (never used).
  if (i < 0) i = -i - 1;
  if (i >= n) i = 2 * n - 1 - i;
  return i < 0 ? 0 : (i >= n ? n - 1 : i);
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
// one elected thread: arm the barrier with the byte count, then start the
// bulk global -> shared copy that completes it
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes,
                                          uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}

// Offset (in elements: float2 in a pair plane, float in a single plane) of row
// r, column c inside one row group of a k-cache plane: rows (2i, 2i+1)
// interleaved per column, an odd last row stored plainly after them.
template <int N>
__device__ __forceinline__ int kpos(int c, int r) {
  return (r < (N & ~1)) ? ((r >> 1) * kTW + c) * 2 + (r & 1) : (N & ~1) * kTW + c;
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// One TMA load of a 3-D box (fp32) into shared memory, completing on `bar`.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            unsigned bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

template <int P, int RB, int C, int MODE>
__global__ void __launch_bounds__(kThreads)
dsg_sweep_kernel(const SweepArgs a, const ChunkTab<RB> tab, const __grid_constant__ CUtensorMap gmap) {
  using K = Cfg<P, RB, C, MODE>;
  constexpr bool CACHED = K::CACHED, STORE = MODE == MODE_STORE;
  constexpr int p = K::p, TH = K::TH, N = K::N, SEG = K::SEG, SEGW = K::SEGW, KY = K::KY;
  constexpr int WIN = K::WIN, GS = K::GS, GC = K::GC, GR = K::GR, HS = K::HS;
  constexpr int YC = K::YC, YR = K::YR, AR = K::AR;
  static_assert(kTW / SEG == kThreads / 32, "one phase-1 segment per warp");
  static_assert(KY % 2 == 0, "offsets are processed in packed pairs");
  pdl_begin();
  extern __shared__ float smem[];
  float* Gs = smem;
  float* Hs = smem + K::OFF_H;
  float* Ys = smem + K::OFF_Y;
  float* As = smem + K::OFF_A;  // [C][AR][YC] far-end accumulators (tile + band)

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

  // ---- stage guide (reflected), channel planes (zero outside), clear A ----
  // warps walk rows, lanes walk columns: index math once per row / column.
  // G col cc <-> image col c0g - RB - p + cc ; row q <-> r0g - p + q
  if (!CACHED) {
    // interior tiles (no reflection anywhere in the guide tile, all its rows
    // in the buffer): one TMA load of the tile, then re-laid out with the odd
    // pitch GS (conflict-free phase-1 loads); border tiles gather with the
    // half-sample reflection (image.py:97-113).  Same floats either way.
    const int gx0 = c0g - RB - p, gy0 = r0g - p, ly0 = gy0 - br0;
    const int gxa = gx0 & ~3, sx = gx0 - gxa;  // 16-byte-aligned box start
    const bool tma = a.tma && gx0 >= 0 && gxa + K::GCB <= W && gy0 >= 0 && gy0 + GR <= Hg &&
                     ly0 >= 0 && ly0 + GR <= brows;
    if (tma) {
      float* tbuf = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(Hs) + 127) & ~uintptr_t(127));
      uint64_t* tbar = reinterpret_cast<uint64_t*>(smem + K::OFF_TB);
      if (tid == 0) {
        mbar_init(tbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        tma_load_3d(tbuf, &gmap, gxa, ly0, b, (unsigned)(K::GCB * GR * 4), tbar);
      }
      __syncthreads();
      mbar_wait(tbar, 0);
      for (int q = warp; q < GR; q += kThreads / 32)
        for (int j = lane; j < GC; j += 32) Gs[q * GS + j] = tbuf[q * K::GCB + sx + j];
      __syncthreads();  // tbuf (the H-map / channel / far area) is free again
    } else {
      constexpr int NJ = (GC + 31) / 32;
      int gcol[NJ];
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int cc = lane + 32 * j;
        gcol[j] = cc < GC ? reflect_index(c0g - RB - p + cc, W) : -1;
      }
#pragma unroll 2
      for (int q = warp; q < GR; q += kThreads / 32) {
        int lr = reflect_index(r0g - p + q, Hg) - br0;
        lr = lr < 0 ? 0 : (lr >= brows ? brows - 1 : lr);
        const float* src = Gimg + (size_t)lr * W;
        float* dst = Gs + q * GS + lane;
#pragma unroll
        for (int j = 0; j < NJ; ++j)
          if (gcol[j] >= 0) {
            PNP_CHECK(dst + 32 * j < Hs);
            dst[32 * j] = __ldg(src + gcol[j]);
          }
      }
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
#pragma unroll
    for (int c_ = 0; c_ < C; ++c_) {
      const float* pa = a.ch[c_].a ? a.ch[c_].a + (size_t)b * plane : nullptr;
      const float* pb = a.ch[c_].b ? a.ch[c_].b + (size_t)b * plane : nullptr;
      if constexpr (CACHED) {
        // k-cache sweeps run few chunks per CTA on small images, so the
        // prologue's latency shows: rows go in batches of kSB per warp with
        // every load of a batch issued before its first shared store
        constexpr int kSB = PNP_SB, kWarps = kThreads / 32;
        for (int r0_ = 0; r0_ < YR; r0_ += kSB * kWarps) {
          float va[kSB][NJ], vb[kSB][NJ];
          bool ok[kSB][NJ];
#pragma unroll
          for (int i = 0; i < kSB; ++i) {
            const int r = r0_ + warp + kWarps * i;
            const int gr = r0g + r, lr = gr - br0;
            const bool rv = r < YR && gr < Hg && lr >= 0 && lr < brows;
            const size_t ro = (size_t)(rv ? lr : 0) * W;
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
              ok[i][j] = rv && ycol[j] >= 0;
              va[i][j] = (pa && ok[i][j]) ? __ldg(pa + ro + ycol[j]) : 1.f;
              vb[i][j] = (pb && ok[i][j]) ? __ldg(pb + ro + ycol[j]) : 1.f;
            }
          }
#pragma unroll
          for (int i = 0; i < kSB; ++i) {
            const int r = r0_ + warp + kWarps * i;
            float* dst = Ys + (c_ * YR + r) * YC + lane;
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
              if (r >= YR || ycol[j] == -2) continue;
              // same floats as 1 -> *a -> *b: a*b, a, b or 1
              const float v = pa ? (pb ? __fmul_rn(va[i][j], vb[i][j]) : va[i][j]) : vb[i][j];
              dst[32 * j] = ok[i][j] ? v : 0.f;
            }
          }
        }
      } else {
#pragma unroll 2
        for (int r = warp; r < YR; r += kThreads / 32) {
          const int gr = r0g + r, lr = gr - br0;
          const bool rv = gr < Hg && lr >= 0 && lr < brows;
          const size_t ro = (size_t)(rv ? lr : 0) * W;
          float* dst = Ys + (c_ * YR + r) * YC + lane;
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
    }
  }
  for (int i = tid; i < C * AR * YC; i += kThreads) As[i] = 0.f;

  constexpr bool TMAK = K::TMAK;
  constexpr int HPF = TH * kTW;              // floats of one offset plane
  constexpr unsigned HPB = HPF * 4;           // its bytes
  float* Ks = smem + K::OFF_K;                // [2][KY planes] (TMAK)
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + K::OFF_MB);
  const int cbeg = tab.grp[blockIdx.y], cend = tab.grp[blockIdx.y + 1];
  const float* kimg =
      CACHED || STORE ? a.kcache + (long long)b * a.kc_img + (long long)tile * a.kc_tile : nullptr;
  auto issue_chunk = [&](int ci) {  // TMAK: chunk ci -> buffer ci & 1
    bulk_load(Ks + (ci & 1) * K::KCH, kimg + (long long)tab.c[ci].koff * HPF,
              (unsigned)tab.c[ci].kc * HPB, mbar + (ci & 1));
  };
  if (TMAK && tid == 0) {
    mbar_init(mbar, 1);
    mbar_init(mbar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (cbeg < cend) issue_chunk(cbeg);
  }
  unsigned kphase = 0;  // TMAK: bit i = parity to wait for on buffer i
  __syncthreads();

  const int c0 = SEG * warp;         // phase-1 segment
  const int c = tid & (kTW - 1);     // phase-2 column
  const int g = tid / kTW;           // phase-2 row group
  const int r0 = g * N;

  // own guide row segment (negated), resident for the whole kernel: it is the
  // broadcast operand of every packed subtraction in phase 1
  float ngown[SEGW];
  if (!CACHED) {
    const float* grow = Gs + lane * GS + c0 + RB;
#pragma unroll
    for (int x = 0; x < SEGW; ++x) ngown[x] = -grow[x];
  }
  float yown[C][N], near[C][N];
#pragma unroll
  for (int c_ = 0; c_ < C; ++c_)
#pragma unroll
    for (int r = 0; r < N; ++r) {
      yown[c_][r] = Ys[(c_ * YR + r0 + r) * YC + c + RB];
      near[c_][r] = (blockIdx.y == 0) ? yown[c_][r] : 0.f;  // self pair, k = hat = 1
    }

  const float2* hcol0 = reinterpret_cast<const float2*>(Hs) + r0 * HS + c;
  float2* hrow0 = reinterpret_cast<float2*>(Hs) + lane * HS + c0;

  // Far accumulators of an offset pair (k, k+1) = (2kp, 2kp+1) live in packed
  // registers: pf[i].x collects even-k terms of window row i, pf[i].y odd-k
  // terms of window row i+1, so one FFMA2 credits both offsets.  Window row j
  // = pf[j].x + pf[j-1].y at flush.  The two row groups' windows overlap in
  // KY-1 rows (group 1's first = group 0's last): group 0 flushes its whole
  // window and group 1 its private rows before the chunk's closing barrier;
  // group 1's shared rows go after it (top of the next chunk, before the
  // phase-1 barrier).  Every SMEM cell sees one writer between barriers and a
  // fixed order (group 0, then group 1) -> bit-reproducible.
  float2 pf[C][WIN - 1];
  float* pend = nullptr;  // group 1's pending (shared-row) flush target
  auto flush = [&](float* base, int j0, int j1) {
#pragma unroll
    for (int c_ = 0; c_ < C; ++c_)
#pragma unroll
      for (int j = 0; j < WIN; ++j) {
        if (j < j0 || j >= j1) continue;  // compile-time after unrolling
        // window rows past the chunk's last offset hold +0: adding them is exact
        float v;
        if (j == 0) v = pf[c_][0].x;
        else if (j == WIN - 1) v = pf[c_][WIN - 2].y;
        else v = __fadd_rn(pf[c_][j].x, pf[c_][j - 1].y);
        float* pA = base + c_ * AR * YC + j * YC;
        PNP_CHECK(pA >= As && pA < As + C * AR * YC);
        *pA = __fadd_rn(*pA, v);
      }
  };
  // the pending flush reads pf after the next chunk cleared it: keep a copy of
  // the KY-1 shared rows (group 1 only)
  float pendv[C][KY - 1];

  for (int ci = cbeg; ci < cend; ++ci) {
    const Chunk& chk = tab.c[ci];
    const int dx = chk.dx, dy0 = chk.dy0, kc = chk.kc;
    if (g == 1 && pend) {
#pragma unroll
      for (int c_ = 0; c_ < C; ++c_)
#pragma unroll
        for (int j = 0; j < KY - 1; ++j) {
          float* pA = pend + c_ * AR * YC + j * YC;
          PNP_CHECK(pA >= As && pA < As + C * AR * YC);
          *pA = __fadd_rn(*pA, pendv[c_][j]);
        }
    }

    // ---------------- phase 1: squared differences + horizontal filter ----
    // packed over the offset pair: (D_k, D_k+1) = (G_partner - G_own)^2
    if (!CACHED) {
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
            PNP_CHECK((const float*)(hrow0 + kp * 32 * HS + i) >= Hs &&
                      (const float*)(hrow0 + kp * 32 * HS + i) < Ys);
            hrow0[kp * 32 * HS + i] = h;
          }
        }
      }
    }
    jitter_sync();

    // ---------------- phase 2: vertical filter, exp, near/far -------------
    const float* ybase = Ys + (r0 + dy0) * YC + c + dx + RB;
    float* abase = As + (r0 + dy0) * YC + c + dx + RB;
    float yw[C][WIN];
#pragma unroll
    for (int c_ = 0; c_ < C; ++c_) {
#pragma unroll
      for (int j = 0; j < WIN; ++j) yw[c_][j] = ybase[c_ * YR * YC + j * YC];
#pragma unroll
      for (int j = 0; j < WIN - 1; ++j) pf[c_][j] = make_float2(0.f, 0.f);
    }
    // this chunk's planes; thread (c, g) owns rows r0.. of column c, stored
    // row-pair interleaved (kpos): pair planes as 16 B (rows 2i, 2i+1 of both
    // offsets), single planes as 8 B (rows 2i, 2i+1); N odd: last row plain.
    // Plane of kp: 2kp planes into the chunk, a pair plane iff 2kp+1 < kc.
    const float* kq = CACHED || STORE ? kimg + (long long)chk.koff * HPF : nullptr;
    float2 kcl[CACHED && !TMAK ? KY / 2 : 1][N];
    if (CACHED && !TMAK) {
      // register path (C = 1): all the chunk's loads in flight together
      // (predicated, not branched)
#pragma unroll
      for (int kp = 0; kp < KY / 2; ++kp) {
        const bool pairp = 2 * kp + 1 < kc;
        const float* plane = kq + 2 * kp * HPF;
        if (pairp) {
          const float2* q2 = reinterpret_cast<const float2*>(plane) + r0 * kTW;
#pragma unroll
          for (int r = 0; r + 1 < N; r += 2) {
            const float4 v = __ldcs(reinterpret_cast<const float4*>(q2 + kpos<N>(c, r)));
            kcl[kp][r] = make_float2(v.x, v.y);
            kcl[kp][r + 1] = make_float2(v.z, v.w);
          }
          if (N & 1) kcl[kp][N - 1] = __ldcs(q2 + kpos<N>(c, N - 1));
        } else {
          const float* q1 = plane + r0 * kTW;
#pragma unroll
          for (int r = 0; r + 1 < N; r += 2) {
            float2 v = make_float2(0.f, 0.f);
            asm volatile(
                "{\n\t.reg .pred q;\n\tsetp.lt.s32 q, %3, %4;\n\t"
                "@q ld.global.cs.v2.f32 {%0, %1}, [%2];\n\t}"
                : "+f"(v.x), "+f"(v.y)
                : "l"(q1 + kpos<N>(c, r)), "r"(2 * kp), "r"(kc));
            kcl[kp][r] = make_float2(v.x, 0.f);
            kcl[kp][r + 1] = make_float2(v.y, 0.f);
          }
          if (N & 1) {
            float v = 0.f;
            asm volatile(
                "{\n\t.reg .pred q;\n\tsetp.lt.s32 q, %2, %3;\n\t"
                "@q ld.global.cs.f32 %0, [%1];\n\t}"
                : "+f"(v)
                : "l"(q1 + kpos<N>(c, N - 1)), "r"(2 * kp), "r"(kc));
            kcl[kp][N - 1] = make_float2(v, 0.f);
          }
        }
      }
    }
    const float* kb = nullptr;  // TMAK: SMEM copy of this chunk
    if (TMAK) {
      if (tid == 0 && ci + 1 < cend) {
        issue_chunk(ci + 1);  // buffer freed by the last barrier
        if (ci + PNP_KPF < cend) {  // and warm L2 further ahead
          const Chunk& cj = tab.c[ci + PNP_KPF];
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                           kimg + (long long)cj.koff * HPF),
                       "r"((unsigned)cj.kc * HPB)
                       : "memory");
        }
      }
      mbar_wait(mbar + (ci & 1), (kphase >> (ci & 1)) & 1u);
      kphase ^= 1u << (ci & 1);
      kb = Ks + (ci & 1) * K::KCH;
    }
#pragma unroll
    for (int kp = 0; kp < KY / 2; ++kp) {
      if (kp == 0 || 2 * kp < kc) {
        const bool pairp = 2 * kp + 1 < kc;
        float2 kk[N];
        if (TMAK) {
          if (pairp) {
            const float2* q2 = reinterpret_cast<const float2*>(kb + 2 * kp * HPF) + r0 * kTW;
#pragma unroll
            for (int r = 0; r + 1 < N; r += 2) {
              const float4 v = *reinterpret_cast<const float4*>(q2 + kpos<N>(c, r));
              kk[r] = make_float2(v.x, v.y);
              kk[r + 1] = make_float2(v.z, v.w);
            }
            if (N & 1) kk[N - 1] = q2[kpos<N>(c, N - 1)];
          } else {
            const float* q1 = kb + 2 * kp * HPF + r0 * kTW;
#pragma unroll
            for (int r = 0; r + 1 < N; r += 2) {
              const float2 v = *reinterpret_cast<const float2*>(q1 + kpos<N>(c, r));
              kk[r] = make_float2(v.x, 0.f);
              kk[r + 1] = make_float2(v.y, 0.f);
            }
            if (N & 1) kk[N - 1] = make_float2(q1[kpos<N>(c, N - 1)], 0.f);
          }
        } else if (CACHED) {
#pragma unroll
          for (int r = 0; r < N; ++r) kk[r] = kcl[CACHED && !TMAK ? kp : 0][r];
        } else {
          // invalid odd slot: L = -inf on the host -> its weight is exactly +0
          const float2 L = make_float2(chk.L[2 * kp], chk.L[2 * kp + 1]);
          float2 hcol[N + 2 * p];
#pragma unroll
          for (int i = 0; i < N + 2 * p; ++i) hcol[i] = hcol0[(kp * 32 + i) * HS];
          // rows in pairs: the four weights of rows (r, r+1) are produced in
          // one 128-bit register quad, which is also the k-cache store operand
          // (the pair plane interleaves rows 2i, 2i+1; kpos)
#pragma unroll
          for (int r = 0; r < N; r += 2) {
            float* plane = STORE ? const_cast<float*>(kq) + 2 * kp * HPF : nullptr;
            if (r + 1 < N) {
              float2 v0 = L, v1 = L;
#pragma unroll
              for (int aa = 0; aa < P; ++aa) {
                const float2 t = make_float2(a.taps_v[aa], a.taps_v[aa]);
                v0 = __ffma2_rn(t, hcol[r + aa], v0);
                v1 = __ffma2_rn(t, hcol[r + 1 + aa], v1);
              }
              const float4 q4 = make_float4(ex2_approx(v0.x), ex2_approx(v0.y),
                                            ex2_approx(v1.x), ex2_approx(v1.y));
              kk[r] = make_float2(q4.x, q4.y);
              kk[r + 1] = make_float2(q4.z, q4.w);
              if (STORE) {
                if (pairp) {
                  float2* dst = reinterpret_cast<float2*>(plane) + r0 * kTW + kpos<N>(c, r);
                  PNP_CHECK(((const float*)(dst + 2) - a.kcache) <= a.kcache_floats);
                  __stcs(reinterpret_cast<float4*>(dst), q4);
                } else {  // single plane: the even offset only
                  float* dst = plane + r0 * kTW + kpos<N>(c, r);
                  PNP_CHECK((dst + 2 - a.kcache) <= a.kcache_floats);
                  __stcs(reinterpret_cast<float2*>(dst), make_float2(q4.x, q4.z));
                }
              }
            } else {  // N odd: the last row alone
              float2 v = L;
#pragma unroll
              for (int aa = 0; aa < P; ++aa)
                v = __ffma2_rn(make_float2(a.taps_v[aa], a.taps_v[aa]), hcol[r + aa], v);
              kk[r] = make_float2(ex2_approx(v.x), ex2_approx(v.y));
              if (STORE) {
                if (pairp) {
                  float2* dst = reinterpret_cast<float2*>(plane) + r0 * kTW + kpos<N>(c, r);
                  PNP_CHECK(((const float*)(dst + 1) - a.kcache) <= a.kcache_floats);
                  __stcs(dst, kk[r]);
                } else {
                  float* dst = plane + r0 * kTW + kpos<N>(c, r);
                  PNP_CHECK((dst + 1 - a.kcache) <= a.kcache_floats);
                  __stcs(dst, kk[r].x);
                }
              }
            }
          }
        }
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int c_ = 0; c_ < C; ++c_) {
            near[c_][r] = __fmaf_rn(kk[r].x, yw[c_][r + 2 * kp], near[c_][r]);
            near[c_][r] = __fmaf_rn(kk[r].y, yw[c_][r + 2 * kp + 1], near[c_][r]);
            pf[c_][r + 2 * kp] =
                __ffma2_rn(kk[r], make_float2(yown[c_][r], yown[c_][r]), pf[c_][r + 2 * kp]);
          }
      }
    }
    if (g == 0) {
      flush(abase, 0, WIN);
    } else {
      flush(abase, KY - 1, WIN);
#pragma unroll
      for (int c_ = 0; c_ < C; ++c_)
#pragma unroll
        for (int j = 0; j < KY - 1; ++j)
          pendv[c_][j] = j == 0 ? pf[c_][0].x : __fadd_rn(pf[c_][j].x, pf[c_][j - 1].y);
      pend = abase;
    }
    jitter_sync();
  }
  if (g == 1 && pend) {
#pragma unroll
    for (int c_ = 0; c_ < C; ++c_)
#pragma unroll
      for (int j = 0; j < KY - 1; ++j) {
        float* pA = pend + c_ * AR * YC + j * YC;
        *pA = __fadd_rn(*pA, pendv[c_][j]);
      }
  }
  __syncthreads();

  // ---- own pixels: near + far; then emit tile + band block ----
#pragma unroll
  for (int c_ = 0; c_ < C; ++c_)
#pragma unroll
    for (int r = 0; r < N; ++r) {
      float* pA = As + (c_ * AR + r0 + r) * YC + c + RB;
      *pA = __fadd_rn(near[c_][r], *pA);
    }
  __syncthreads();
  const int BR = TH + R, BC = kTW + 2 * R;
  const size_t slot =
      (((size_t)b * a.part_ntr + a.part_off + tyl) * gridDim.y + blockIdx.y) * a.tiles_x + tx;
  float* out = a.partial + slot * (size_t)(C * BR * BC);
  PNP_CHECK((long long)((slot + 1) * (size_t)(C * BR * BC)) <= a.partial_floats);
#pragma unroll
  for (int c_ = 0; c_ < C; ++c_) {
    const float* A0 = As + c_ * AR * YC + (RB - R);
    float* o = out + (size_t)c_ * BR * BC;
    for (int br = warp; br < BR; br += kThreads / 32)
      for (int bc = lane; bc < BC; bc += 32) o[br * BC + bc] = A0[br * YC + bc];
  }
}

// Fixup geometry: the partial blocks covering global pixel (y, x) are summed
// in a fixed order (group, tile row, tile col) by the fixup kernels
// (pnp_dsg.cu).  Slot 0 of the partial array holds global tile row part_tr0.
struct FixGeo {
  const float* partial;
  int Hg, W, R, TH, tiles_x, NP, C;  // R: block band (0: tile-only blocks); NP = offset groups
  int part_tr0, part_ntr;
  int y0, nrows;          // output rows [y0, y0 + nrows) (global)
  int buf_r0, buf_rows;   // per-pixel buffers' window
};

}  // namespace pnp
