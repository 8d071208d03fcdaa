// Native iteration loop of the linearized PnP-ADMM with a frozen guide
// (reference solver.py:199-235, Algorithm 1) for the device forward models.
//
// The Python driver (solver.linearized_pnp_admm) issues two fused steps per
// iteration -- gradient + x-update (pnp_sr_grad_xupdate / pnp_qis_grad_xupdate)
// and frozen apply + u-update (pnp_dsg_apply_admm) -- through ctypes; at
// ~100 us of device time per 512^2 iteration the interpreter's ~110 us per
// iteration became the bound.  This loop issues exactly the same calls with
// exactly the same arguments from C++ (bitwise-identical iterates), ping-pongs
// the v buffers, and records one event per iteration for the log's time_ms.
#include <cuda_runtime.h>

#include <vector>

#include "pnp_b200.h"
#include "pnp_internal.h"

using namespace pnp;

extern "C" {

int pnp_admm_run(pnp_ctx* ctx, int kind, const float* obs, const float* obs2, int batch, int H,
                 int W, const float* taps, int radius, int factor, int boundary,
                 double gain_over_K, double floor_, const pnp_frozen* fz, int k0, int k1, float* x,
                 float* v0, float* v1, float* u, float* z, const float* gt, double mu,
                 double alpha, double rho, double lo, double hi, double* stats, double* objv,
                 int* flags, float* ms_out, int* v_last) {
  if (!ctx || !fz || !obs || !x || !v0 || !v1 || !u || !z || !stats || !flags)
    return fail(PNP_EINVAL, "null argument");
  if (kind != 0 && kind != 1) return fail(PNP_EINVAL, "kind must be 0 (SR) or 1 (QIS)");
  if (kind == 1 && !obs2) return fail(PNP_EINVAL, "QIS needs ones and zeros");
  if (k0 < 1 || k1 < k0 - 1) return fail(PNP_EINVAL, "bad iteration range");
  const int n_it = k1 - k0 + 1;
  std::vector<cudaEvent_t>& ev = ctx->iter_events;
  if (ms_out) {
    while ((int)ev.size() < n_it + 1) {
      cudaEvent_t e;
      PNP_CUDA(cudaEventCreate(&e));
      ev.push_back(e);
    }
    PNP_CUDA(cudaEventRecord(ev[0], ctx->stream));
  }
  int cur = 0;
  if (kind == 0 && n_it > 0) {  // SR: next residual pipelined on a side stream
    int rc = sr_admm_pipelined(ctx, obs, batch, H, W, taps, radius, factor, boundary, fz, k0, k1,
                               x, v0, v1, u, z, gt, mu, alpha, rho, lo, hi, stats, objv, flags,
                               ms_out ? &ev : nullptr, &cur);
    if (rc) return rc;
  } else {
    float* vcur = v0;
    float* vnext = v1;
    for (int k = k0; k <= k1; ++k) {
      Nvtx iter("admm_iteration");
      int* fk = flags + (k - 1);
      double* obj = (objv && k >= 2) ? objv + (size_t)(k - 2) * batch : nullptr;
      int rc = kind == 0
                   ? pnp_sr_grad_xupdate(ctx, x, obs, batch, H, W, taps, radius, factor, boundary,
                                         obj, vcur, u, z, mu, alpha, rho, lo, hi, fk)
                   : pnp_qis_grad_xupdate(ctx, x, obs, obs2, batch, H * W, gain_over_K, floor_,
                                          obj, vcur, u, z, mu, alpha, rho, lo, hi, fk);
      if (rc) return rc;
      rc = pnp_dsg_apply_admm(ctx, fz, z, vnext, u, x, vcur, gt, rho,
                              stats + (size_t)(k - 1) * batch * 4, fk);
      if (rc) return rc;
      float* t = vcur;
      vcur = vnext;
      vnext = t;
      cur ^= 1;
      if (ms_out) PNP_CUDA(cudaEventRecord(ev[k - k0 + 1], ctx->stream));
    }
  }
  if (v_last) *v_last = cur;
  if (ms_out && n_it > 0) {
    PNP_CUDA(cudaEventSynchronize(ev[n_it]));
    for (int i = 1; i <= n_it; ++i) PNP_CUDA(cudaEventElapsedTime(ms_out + i - 1, ev[0], ev[i]));
  }
  return PNP_OK;
}

}  // extern "C"
