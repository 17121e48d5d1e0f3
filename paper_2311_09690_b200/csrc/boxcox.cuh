// Box-Cox decode on the device (dataset.py:97-115, costmodel.py:358-373),
// float64, shared by the training kernels' original-space relative term.
#pragma once

#include "common.cuh"

namespace tpcb {

// y = decode(e) and dy/de with the reference's clamp at the domain edge
// (base clamped to 1e-12, zero derivative beyond: _decode_with_grad)
__device__ __forceinline__ void boxcox_decode_with_grad(double e, const tpcb_boxcox& n, double* y,
                                                        double* dy) {
  const double t = e * n.t_std + n.t_mean;
  if (fabs(n.lambda_bc) < 1e-9) {
    *y = exp(t) - n.shift;
    *dy = n.t_std * exp(t);
    return;
  }
  double base = n.lambda_bc * t + 1.0;
  const bool ok = base > 1e-12;
  if (!ok) base = 1e-12;
  *y = pow(base, 1.0 / n.lambda_bc) - n.shift;
  *dy = ok ? n.t_std * pow(base, 1.0 / n.lambda_bc - 1.0) : 0.0;
}

// decode of a model-space training label (inside the domain by construction)
__device__ __forceinline__ double boxcox_decode_plain(double e, const tpcb_boxcox& n) {
  const double t = e * n.t_std + n.t_mean;
  if (fabs(n.lambda_bc) < 1e-9) return exp(t) - n.shift;
  return pow(n.lambda_bc * t + 1.0, 1.0 / n.lambda_bc) - n.shift;
}

__device__ __forceinline__ double sign_d(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

}  // namespace tpcb
