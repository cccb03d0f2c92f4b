// cg.cuh -- scalar epilogues of the PSP-CG reductions (f4; readings R27-R31), shared by
// krylov.cu (the generic passes) and stencil.cu (the fused direction pass).  One thread.
// The recurrences are textbook preconditioned CG (Hestenes-Stiefel), as oracle/oracle.c orc_pcg:
//   alpha = rho / p'q,  x += alpha p,  r -= alpha q,  R(k) = ||r||,  z = M^-1 r,
//   rho' = r'z,  beta = rho' / rho,  p = z + beta p.
#pragma once
#include <math.h>

#include "internal.h"

namespace psp {

static __device__ void cg_epilogue(int kind, DevState ds, int slot, int identity, const double* tot) {
  double* sc = ds.scal;
  switch (kind) {
    case EPI_CG_START: {                       // r0 = b - A x0: beta = ||r0|| (R3 test), rho = r'r (N = I)
      sc[SC_BETA] = sqrt(tot[0]);
      sc[SC_RHO] = tot[0];
      sc[SC_BETACG] = 0.0;
      break;
    }
    case EPI_CG_DIR: {                         // alpha = rho / p'q; the probe (p, A p) / ||p|| (R28)
      const double pq = tot[0], pp = tot[1];
      int flags = 0;
      if (!isfinite(pq) || !isfinite(pp)) flags |= PSP_FLAG_NONFINITE;
      else if (!(pq > 0.0)) flags |= PSP_FLAG_BREAKDOWN;   // R30: A (or M) not SPD
      sc[SC_ALPHA] = sc[SC_RHO] / pq;
      ds.slot_scale[slot] = pp > 0.0 ? 1.0 / sqrt(pp) : 0.0;
      sc[SC_FLAGS] = (double)flags;
      break;
    }
    case EPI_CG_UPD: {                         // R(k) = ||r|| (l.32's test, R1); N = I: z = r
      const double rr = tot[0], R = sqrt(rr);
      int flags = (int)sc[SC_FLAGS];
      sc[SC_RK] = R;
      if (R <= sc[SC_EPS]) flags |= PSP_FLAG_CONVERGED;
      if (!isfinite(R)) flags |= PSP_FLAG_NONFINITE;
      sc[SC_FLAGS] = (double)flags;
      if (identity) {
        sc[SC_BETACG] = rr / sc[SC_RHO];
        sc[SC_RHO] = rr;
      }
      break;
    }
    case EPI_CG_RHO: {                         // rho' = r'z, beta = rho' / rho
      sc[SC_BETACG] = tot[0] / sc[SC_RHO];
      sc[SC_RHO] = tot[0];
      break;
    }
  }
}

}  // namespace psp
