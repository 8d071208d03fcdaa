// Per-pixel arithmetic of the linearized-ADMM x-update (solver.py:219-221),
// shared by every kernel that performs it (the SR adjoint / QIS gradient
// epilogues and the frozen-apply fixup of the pipelined SR loop), so the
// fused and unfused paths round identically: explicit _rn operations, no
// contraction left to the compiler.
#pragma once

#include <math.h>

namespace pnp {

// x' = clamp(mu (alpha x + rho (v - u) - grad), lo, hi), z = x' + u;
// returns flags (1: x' non-finite before the clamp, 2: z non-finite)
__device__ __forceinline__ int admm_xupdate(double mu, double alpha, double rho, float lo,
                                            float hi, float x, float v, float u, float grad,
                                            float& xo, float& zo) {
  const double a = __dmul_rn(alpha, (double)x);
  const double b = __dmul_rn(rho, __dsub_rn((double)v, (double)u));
  const double xn = __dmul_rn(mu, __dsub_rn(__dadd_rn(a, b), (double)grad));
  float xf = __double2float_rn(xn);
  int f = isfinite(xf) ? 0 : 1;
  xf = fminf(fmaxf(xf, lo), hi);
  const float zf = __double2float_rn(__dadd_rn((double)xf, (double)u));
  if (!isfinite(zf)) f |= 2;
  xo = xf;
  zo = zf;
  return f;
}

}  // namespace pnp
