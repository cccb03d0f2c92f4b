// givens.cuh -- Givens update of one Hessenberg column (Alg.1 l.19-32), shared by the
// reduction epilogues of krylov.cu and fused.cu.  Device code only.
#pragma once
#include <math.h>

#include "internal.h"

namespace psp {

// ------------------------------------------------------------------------------------------
// Givens update of column k (Alg.1 l.19-32; R4, R10).  One thread.  Also sets the
// lagged normalisation alpha_{k+1} = 1/H(k+1,k) of V(:,k+1) (l.18; 0 on breakdown).
// ------------------------------------------------------------------------------------------
static __device__ __forceinline__ void givens_update(DevState ds, int k, int nA) {
  const int ld = nA + 1;
  double* Hc = ds.H + (int64_t)(k - 1) * ld;
  double colsq = 0.0;
  for (int j = 0; j <= k; ++j) {
    ds.Hraw[(int64_t)(k - 1) * ld + j] = Hc[j];
    colsq += Hc[j] * Hc[j];
  }
  const double hk1 = Hc[k];
  bool breakdown = !(hk1 > 1e-14 * sqrt(colsq));   // R4, before rotation
  const bool nonfinite = !isfinite(hk1);
  ds.alpha[k] = (breakdown || nonfinite) ? 0.0 : 1.0 / hk1;
  ds.G[k] = 0.0;                                    // l.9: G(k+1) <- 0
  for (int j = 1; j <= k - 1; ++j) {                // l.19-23
    const double delta = Hc[j - 1];
    Hc[j - 1] = delta * ds.C[j - 1] + ds.S[j - 1] * Hc[j];
    Hc[j] = -delta * ds.S[j - 1] + ds.C[j - 1] * Hc[j];
  }
  const double a = Hc[k - 1], b = Hc[k];            // l.24-28, R10
  const double gamma = sqrt(a * a + b * b);
  if (gamma == 0.0) {
    ds.C[k - 1] = 1.0;
    ds.S[k - 1] = 0.0;
    breakdown = true;
  } else {
    ds.C[k - 1] = a / gamma;
    ds.S[k - 1] = b / gamma;
  }
  Hc[k - 1] = gamma;
  Hc[k] = 0.0;
  const double delta = ds.G[k - 1];                 // l.29-31
  ds.G[k - 1] = ds.C[k - 1] * delta + ds.S[k - 1] * ds.G[k];
  ds.G[k] = -ds.S[k - 1] * delta + ds.C[k - 1] * ds.G[k];
  const double R = fabs(ds.G[k]);                   // l.32
  ds.resid[k - 1] = R;
  ds.scal[SC_RK] = R;
  int flags = 0;
  if (R <= ds.scal[SC_EPS]) flags |= PSP_FLAG_CONVERGED;  // l.33
  if (breakdown) flags |= PSP_FLAG_BREAKDOWN;
  if (nonfinite || !isfinite(R)) flags |= PSP_FLAG_NONFINITE;
  ds.scal[SC_FLAGS] = (double)flags;
}

// ------------------------------------------------------------------------------------------
// Scalar tail of a ring-resident step k (the fused pass of fused.cu, or EPI_FUSED after the
// multi-rank all-reduce): from tot = [t_0..t_{k-1}, l_0..l_{k-1}, t_u, nu] (t_j = V_j' w~,
// l_j = V_j' u, t_u = u' w~, nu = u'u of u = V(:,k+1) unnormalised) -- H(k+1,k) = ||U_k||, the
// Givens update of column k (l.17-32), alpha_{k+1} -> slot_scale[dst_slot], and step k+1's MGS
// coefficients by (I + L) h = s (R11).  k = 0: the cycle-start pass (no column to finish).
// ------------------------------------------------------------------------------------------
static __device__ void fused_tail(DevState ds, int k, int nA, const double* tot, double* slot_scale, int dst_slot) {
  const int ld = nA + 1;
  const double t_u = tot[2 * k], s_nu = tot[2 * k + 1];
  double an;  // alpha of u = V_{k+1}
  if (k >= 1) {
    ds.H[(int64_t)(k - 1) * ld + k] = sqrt(s_nu);  // l.17: H(k+1,k) = ||U_k||
    givens_update(ds, k, nA);                      // l.19-32, sets alpha[k] (0 on breakdown)
    an = ds.alpha[k];
  } else {
    an = ds.alpha[0];                              // 1/beta from the residual kernel (l.6)
  }
  slot_scale[dst_slot] = an;
  if (k >= nA) return;
  // MGS coefficients of step k+1 (column index k): (I + L) h = s (R11)
  double* Lrow = ds.Lm + (int64_t)k * ld;
  for (int j = 0; j < k; ++j) Lrow[j] = ds.alpha[j] * an * tot[k + j];
  double* Hc = ds.H + (int64_t)k * ld;
  for (int j = 0; j <= k; ++j) {
    double h = (j < k) ? ds.alpha[j] * an * tot[j] : an * an * t_u;
    const double* Lr = ds.Lm + (int64_t)j * ld;
    for (int c = 0; c < j; ++c) h -= Lr[c] * Hc[c];
    Hc[j] = h;
  }
}

}  // namespace psp
