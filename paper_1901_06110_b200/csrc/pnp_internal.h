// Internal host-side helpers shared by the pnp_b200 translation units.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <map>
#include <tuple>
#include <string>
#include <utility>
#include <vector>

#include "../../include/pnp_b200.h"

namespace pnp {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define PNP_CUDA(call)                                 \
  do {                                                 \
    cudaError_t e__ = (call);                          \
    if (e__ != cudaSuccess) return cuda_fail(e__, #call); \
  } while (0)

#define PNP_LAUNCH_CHECK(what)                         \
  do {                                                 \
    cudaError_t e__ = cudaGetLastError();              \
    if (e__ != cudaSuccess) return cuda_fail(e__, what); \
  } while (0)

// Grow-only device buffer.
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  int ensure(size_t want);
  void release();
  template <class T>
  T* as() const { return static_cast<T*>(ptr); }
};

}  // namespace pnp

namespace pnp {
enum ProfCat {
  PROF_SWEEP = 0,         // fused recompute sweep (incl. k-cache store)
  PROF_FIXUP = 1,
  PROF_FORWARD = 2,
  PROF_ADMM = 3,
  PROF_SWEEP_CACHED = 4,  // HBM-streaming sweep over the k cache
  PROF_CHECK = 5,         // input validation (non-finite scan)
  PROF_NCAT = 6
};
struct ProfSlot {
  cudaEvent_t a = nullptr, b = nullptr;
  int cat = 0;
};
}  // namespace pnp

struct pnp_ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t stream = 0;
  // orders a call on a new stream after the context's work on the previous
  // one (the scratch buffers below are shared by every call on the context)
  cudaEvent_t ev_switch = nullptr;
  pnp::DevBuf partial, rs, kx, d, mbits, stats, flags;
  // adaptive-denoise k cache: a caller-bound buffer (pnp_ctx_bind_kcache; the
  // Python layer binds torch-allocated memory per call), else allocated from
  // the stream-ordered pool at the start of the call and freed at its end
  void* kc_ext = nullptr;
  size_t kc_ext_bytes = 0;
  float* kc_call = nullptr;        // the current call's cache (banded calls)
  bool kc_call_pooled = false;
  pnp::DevBuf cg;                  // conjugate-gradients work vectors + state
  pnp::DevBuf counter;             // last-CTA reduction counter (kept at zero)
  size_t cache_limit = (size_t)-1;  // bytes; 0 disables the k cache
  // offset tables keyed by (R, NG, sweep path): host blobs of Chunk (hat,
  // no-hat) + NG+1 group starts, which reach the kernels through the launch
  // parameters; the general kernel's dy-group starts + a device table of
  // log2 hat per offset
  struct Tables {
    std::vector<char> hat, nohat;
    std::vector<int> grp;
    pnp::DevBuf ltab;
  };
  std::map<std::tuple<int, int, int>, Tables> tables;
  // per-iteration timing events of the native ADMM loop (pnp_admm_run)
  std::vector<cudaEvent_t> iter_events;
  // its side stream (the next iteration's SR gradient overlaps the denoiser),
  // two ordering events (x ready, gradient ready), and the residual /
  // partial / gradient buffers it owns
  cudaStream_t side = nullptr;
  cudaEvent_t ev_x = nullptr, ev_g = nullptr;
  pnp::DevBuf admm_r, admm_part, admm_g;
  // incremental banded denoise (pnp_dsg_band_sweep / _finish): the next band
  // expected (-1: none in progress), the call's band count and cached tile rows
  int band_next = -1, band_count = 0, band_kc_rows = 0;
  // optional per-launch CUDA-event timing (pnp_ctx_profile)
  bool prof = false;
  std::vector<pnp::ProfSlot> slots;
  size_t nslots = 0;
};

namespace pnp {
// NVTX range for timelines (nsys): API calls, launches, ADMM iterations.
// Header-only NVTX v3: a no-op unless a tool is attached.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};
inline const char* prof_name(int cat) {
  static const char* names[] = {"sweep", "fixup", "forward", "admm", "sweep_cached", "check"};
  return cat >= 0 && cat < 6 ? names[cat] : "pnp";
}
// Brackets one kernel launch with an NVTX range and, when profiling is on,
// with events on the context stream (bench.py's live roofline numbers).
struct ProfScope {
  pnp_ctx* c;
  size_t idx;
  Nvtx range;
  ProfScope(pnp_ctx* ctx, int cat) : c(ctx), idx((size_t)-1), range(prof_name(cat)) {
    if (!c->prof) return;
    if (c->nslots == c->slots.size()) {
      ProfSlot s;
      if (cudaEventCreate(&s.a) != cudaSuccess || cudaEventCreate(&s.b) != cudaSuccess) return;
      c->slots.push_back(s);
    }
    idx = c->nslots++;
    c->slots[idx].cat = cat;
    cudaEventRecord(c->slots[idx].a, c->stream);
  }
  ~ProfScope() {
    if (idx != (size_t)-1) cudaEventRecord(c->slots[idx].b, c->stream);
  }
};
}  // namespace pnp

namespace pnp {
// stats[b*4 + k] = sum_j part[b][j][k] for k < 3 (pnp_forward.cu)
int reduce_stats3(pnp_ctx* ctx, const double* part, int nblk, int batch, double* stats);
// The next iteration's x-update fused into a frozen apply's u-update fixup
// (pnp_dsg_apply_admm + pnp_sr_grad_xupdate in one pass over the pixels): x
// (the apply's `x`) and z (its input) are rewritten in place once `ready`
// (the gradient's event, nullable) has fired.
struct AdmmXNext {
  const float* grad;
  double mu, alpha, lo, hi;
  int* flags;
  cudaEvent_t ready;
};
int dsg_apply_admm_x(pnp_ctx* ctx, const pnp_frozen* fz, const float* z, float* v, float* u,
                     const float* x, const float* v_prev, const float* gt, double rho,
                     double* stats, int* flags, const AdmmXNext* xn);
// pnp_admm_run's SR loop with the gradient of the next iteration (residual +
// adjoint) on a side stream during the frozen apply, and the x-update fused
// into the apply's fixup (pnp_forward.cu): bitwise the sequential loop.
int sr_admm_pipelined(pnp_ctx* ctx, const float* y, int batch, int H, int W, const float* taps,
                      int radius, int factor, int boundary, const pnp_frozen* fz, int k0, int k1,
                      float* x, float* v0, float* v1, float* u, float* z, const float* gt,
                      double mu, double alpha, double rho, double lo, double hi, double* stats,
                      double* objv, int* flags, std::vector<cudaEvent_t>* timing, int* v_last);
}  // namespace pnp

struct pnp_frozen {
  int device = 0;
  int B = 0, H = 0, W = 0, R = 0, P = 0;
  float taps[64] = {0};
  double bw = 0;
  float* guide = nullptr;  // B*H*W
  float* rs = nullptr;     // B*H*W
  float* d = nullptr;      // B*H*W
  float* mv = nullptr;     // B floats: m; then B floats: 1/m
  float* kcache = nullptr; // pair weights (null: recompute on apply)
  int kc_rows = 0;
  int tiles_y = 0;         // tile rows per image (kc_rows == tiles_y: fully cached)
  size_t kc_bytes = 0;     // bytes of the k cache
  bool kc_ext = false;     // the k cache is a caller-bound buffer (not freed here)
  // the stream current at the freeze (a caller-bound k cache was handed out
  // on it): destroy orders it after the handle's last use
  cudaStream_t kc_stream = 0;
  // buffers come from the device's stream-ordered pool (cudaMallocAsync) and
  // go back to it on the stream of the handle's last use: no device-wide
  // synchronization and no page-mapping cost when ADMM runs re-freeze
  mutable cudaStream_t stream = 0;
};
