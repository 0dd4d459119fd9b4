// sm_100a fp64 device kernels of the DiffPD hot path.
//
// Layouts:
//   state   [n][3][B]      index (3*node + axis)*B + b       (sims fastest: coalesced over b)
//   solve   [nfree][R]     index pos*R + axis*B + b, R = 3B  (A = A_s (x) I_3: 3B RHS per row)
//   elemF   [m][8][3][B]   per-element nodal force contributions (deterministic gather input)
#pragma once
#include <cstdint>

namespace pdb {

struct Stencil {
  double m3[3];        // the three |dN_a/dX_j| magnitudes of the voxel stencil (see dNf)
  double fiber[3];
  double V;            // quadrature weight dx^3/8
  double w_m;          // muscle weight (0 = off)
  double clamp;        // eigenvalue floor factor of the polar derivative (1e-6)
  double kappa;        // volume-preserving weight per corotated weight, w_v / w = nu / (1 - 2 nu); 0 = no volume term
};

struct ElemArgs {
  const int32_t* hex8;
  int m, B;
  const double* w_sim;     // [B] corotated weight per sim
  const double* act;       // actuation base for this step: act[b*act_bstride + e], or null
  int64_t act_bstride;
  const double* fib;       // [m][3] per-element unit fiber directions, or null = Stencil::fiber
};

struct SweepDev {  // device copy of HostPlan::Sweep
  const double* A;
  const int64_t *a_off, *zidx;
  const int32_t *nk, *nkd, *zrow, *out, *nvalid, *chain;
  const int4* rec;  // packed per-item records, 2 x int4 per item (plan.h int4x2)
  const int32_t *red_row, *red_mode, *red_ptr, *red_src;
};

struct Sweep4Dev {  // device copy of HostPlan::Sweep4 (K3 v4)
  const double* A;
  const int32_t *krow, *pstart, *pkg, *pout, *pnv, *wg, *wpiece;
  const int32_t *red_row, *red_mode, *red_ptr, *red_src;
};

struct DotArgs {
  const double* u[3];
  const double* v[3];
  int npairs;
};

}  // namespace pdb
