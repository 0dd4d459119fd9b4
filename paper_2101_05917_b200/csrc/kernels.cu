// sm_100a fp64 kernels of the DiffPD hot path (see kernels.cuh for layouts).
//
//   K1  k_elem_residual   local step: per (element, sim) F_q = G_q x_e, R = polar(F_q)
//                         by scaled Newton iteration (SVD fallback), muscle p = r Fm/||Fm||,
//                         element force sum_q V G_q^T [w (F - R) + w_m (Fm - p) m^T] and energy
//   K2  k_gather          deterministic element->node gather (fixed incidence order, no atomics):
//                         grad g = M/h^2 (x - y) + sum_e ... (eq:time_integration / eq:gradient)
//   K3  k_fwdA/B, k_bwdA/B level-scheduled supernodal solves with L_s, 3B RHS per factor stream
//   K4  k_elem_AN         matrix-free A_N p = (M/h^2) p + sum w V G^T (dF - dR[dF]) G p
//   --  per-sim deterministic dot products, axpys, PCG scalars, parameter-gradient terms
#include <cuda_runtime.h>

#include <cmath>

#include "kernels.cuh"

namespace pdb {
// Programmatic dependent launch: every hot-loop kernel is launched with programmatic stream
// serialisation; it waits for its predecessor grid (complete, memory visible) before its first access and then lets
// the next launch be scheduled, so launch latency and ramp overlap the running kernel.  Without the launch attribute
// both instructions are no-ops.
#define PDL_ENTRY() asm volatile("griddepcontrol.wait;\n" "griddepcontrol.launch_dependents;\n" ::: "memory")

// ----------------------------------------------------------------- 3x3 helpers (row-major)
__device__ __forceinline__ double det3(const double* A) {
  return A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
         A[2] * (A[3] * A[7] - A[4] * A[6]);
}
// cofactor matrix C (C_ij = cofactor of A_ij); A^{-T} = C / det
__device__ __forceinline__ void cof3(const double* A, double* C) {
  C[0] = A[4] * A[8] - A[5] * A[7];
  C[1] = A[5] * A[6] - A[3] * A[8];
  C[2] = A[3] * A[7] - A[4] * A[6];
  C[3] = A[2] * A[7] - A[1] * A[8];
  C[4] = A[0] * A[8] - A[2] * A[6];
  C[5] = A[1] * A[6] - A[0] * A[7];
  C[6] = A[1] * A[5] - A[2] * A[4];
  C[7] = A[2] * A[3] - A[0] * A[5];
  C[8] = A[0] * A[4] - A[1] * A[3];
}

// Symmetric 3x3 eigen-decomposition by cyclic Jacobi: A (row-major, symmetric) ->
// eigenvalues lam[3] (descending), eigenvectors V[:,k] (columns, row-major V), det V = +1.
__device__ __noinline__ void jacobi_eig3(const double* Ain, double* lam, double* V) {
  double a[9];
  for (int i = 0; i < 9; ++i) a[i] = Ain[i];
  for (int i = 0; i < 9; ++i) V[i] = (i % 4 == 0) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 30; ++sweep) {
    const double off = a[1] * a[1] + a[2] * a[2] + a[5] * a[5];
    const double dia = a[0] * a[0] + a[4] * a[4] + a[8] * a[8];
    if (off <= 1e-34 * dia || off == 0.0) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        const double apq = a[3 * p + q];
        if (apq == 0.0) continue;
        const double app = a[3 * p + p], aqq = a[3 * q + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 3; ++k) {  // A <- J^T A J
          const double akp = a[3 * k + p], akq = a[3 * k + q];
          a[3 * k + p] = c * akp - s * akq;
          a[3 * k + q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          const double apk = a[3 * p + k], aqk = a[3 * q + k];
          a[3 * p + k] = c * apk - s * aqk;
          a[3 * q + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          const double vkp = V[3 * k + p], vkq = V[3 * k + q];
          V[3 * k + p] = c * vkp - s * vkq;
          V[3 * k + q] = s * vkp + c * vkq;
        }
      }
  }
  double l[3] = {a[0], a[4], a[8]};
  int idx[3] = {0, 1, 2};
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2 - i; ++j)
      if (l[idx[j]] < l[idx[j + 1]]) { int t = idx[j]; idx[j] = idx[j + 1]; idx[j + 1] = t; }
  double W[9];
  for (int k = 0; k < 3; ++k) {
    lam[k] = l[idx[k]];
    for (int r = 0; r < 3; ++r) W[3 * r + k] = V[3 * r + idx[k]];
  }
  if (det3(W) < 0)
    for (int r = 0; r < 3; ++r) W[3 * r + 2] = -W[3 * r + 2];
  for (int i = 0; i < 9; ++i) V[i] = W[i];
}

// Rotation closest to F via an SVD from the eigen-decomposition of F^T F; the
// smallest singular direction is flipped when det F < 0.
__device__ __noinline__ void polar_svd_fallback(const double* F, double* R) {
  double C[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) C[3 * i + j] = F[i] * F[j] + F[3 + i] * F[3 + j] + F[6 + i] * F[6 + j];
  double lam[3], V[9];
  jacobi_eig3(C, lam, V);
  double u[3][3];
  for (int k = 0; k < 2; ++k) {
    double fv[3];
    for (int i = 0; i < 3; ++i) fv[i] = F[3 * i] * V[k] + F[3 * i + 1] * V[3 + k] + F[3 * i + 2] * V[6 + k];
    if (k == 1) {  // Gram-Schmidt against u0
      const double d = fv[0] * u[0][0] + fv[1] * u[0][1] + fv[2] * u[0][2];
      for (int i = 0; i < 3; ++i) fv[i] -= d * u[0][i];
    }
    double nr = sqrt(fv[0] * fv[0] + fv[1] * fv[1] + fv[2] * fv[2]);
    if (!(nr > 1e-300)) {  // degenerate: any unit vector orthogonal to the previous ones
      if (k == 0) { fv[0] = 1; fv[1] = 0; fv[2] = 0; }
      else {
        const double* a = u[0];
        const double e[3] = {fabs(a[0]) < 0.9 ? 1.0 : 0.0, fabs(a[0]) < 0.9 ? 0.0 : 1.0, 0.0};
        fv[0] = a[1] * e[2] - a[2] * e[1];
        fv[1] = a[2] * e[0] - a[0] * e[2];
        fv[2] = a[0] * e[1] - a[1] * e[0];
      }
      nr = sqrt(fv[0] * fv[0] + fv[1] * fv[1] + fv[2] * fv[2]);
    }
    for (int i = 0; i < 3; ++i) u[k][i] = fv[i] / nr;
  }
  u[2][0] = u[0][1] * u[1][2] - u[0][2] * u[1][1];
  u[2][1] = u[0][2] * u[1][0] - u[0][0] * u[1][2];
  u[2][2] = u[0][0] * u[1][1] - u[0][1] * u[1][0];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R[3 * i + j] = u[0][i] * V[3 * j] + u[1][i] * V[3 * j + 1] + u[2][i] * V[3 * j + 2];
}

// R = rotation of the polar decomposition F = R S, det F > 0: Newton-Schulz iteration
// X <- X (3I - X^T X)/2 on X0 = F sqrt(3)/||F||_F (all singular values in (0, sqrt3), quadratic
// convergence, no divisions); stops after the step taken with ||X^T X - I||_F < 1e-8 (the next error is
// below fp64 resolution).  Falls back to the scaled Newton iteration X <- (g X + X^{-T}/g)/2 if it is
// slow (strongly anisotropic F), and to the SVD path for det F <= 1e-6 ||F||^3.
__device__ __noinline__ void polar_newton(const double* F, double* R) {
  double X[9];
  for (int i = 0; i < 9; ++i) X[i] = F[i];
  bool scaled = true, last = false;
  for (int it = 0; it < 40; ++it) {
    double C[9];
    cof3(X, C);
    const double det = X[0] * C[0] + X[1] * C[1] + X[2] * C[2];
    const double idet = 1.0 / det;
    double g = 1.0;
    if (scaled) {
      double xn = 0, cn = 0;
      for (int i = 0; i < 9; ++i) { xn += X[i] * X[i]; cn += C[i] * C[i]; }
      g = sqrt(sqrt(cn * idet * idet / xn));  // (||X^{-1}||_F / ||X||_F)^{1/2}
    }
    double diff = 0, nrm = 0;
    for (int i = 0; i < 9; ++i) {
      const double xn = 0.5 * (g * X[i] + C[i] * idet / g);
      diff += (xn - X[i]) * (xn - X[i]);
      nrm += xn * xn;
      X[i] = xn;
    }
    if (diff < 1e-4 * nrm) scaled = false;
    if (last) break;
    if (!scaled && diff < 1e-18 * nrm) last = true;
  }
  for (int i = 0; i < 9; ++i) R[i] = X[i];
}

__device__ void polar_rotation(const double* F, double* R) {
  const double d0 = det3(F);
  double fn2 = 0;
#pragma unroll
  for (int i = 0; i < 9; ++i) fn2 += F[i] * F[i];
  if (!(d0 > 1e-6 * fn2 * sqrt(fn2))) {
    polar_svd_fallback(F, R);
    return;
  }
  const double c = sqrt(3.0 / fn2);
  double X[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) X[i] = c * F[i];
  for (int it = 0; it < 14; ++it) {
    // C = X^T X (symmetric), delta = ||C - I||_F^2
    const double c00 = X[0] * X[0] + X[3] * X[3] + X[6] * X[6];
    const double c11 = X[1] * X[1] + X[4] * X[4] + X[7] * X[7];
    const double c22 = X[2] * X[2] + X[5] * X[5] + X[8] * X[8];
    const double c01 = X[0] * X[1] + X[3] * X[4] + X[6] * X[7];
    const double c02 = X[0] * X[2] + X[3] * X[5] + X[6] * X[8];
    const double c12 = X[1] * X[2] + X[4] * X[5] + X[7] * X[8];
    const double d = (c00 - 1) * (c00 - 1) + (c11 - 1) * (c11 - 1) + (c22 - 1) * (c22 - 1) +
                     2.0 * (c01 * c01 + c02 * c02 + c12 * c12);
    // Y = (3I - C)/2 ; X <- X Y
    const double y00 = 1.5 - 0.5 * c00, y11 = 1.5 - 0.5 * c11, y22 = 1.5 - 0.5 * c22;
    const double y01 = -0.5 * c01, y02 = -0.5 * c02, y12 = -0.5 * c12;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double a0 = X[3 * i], a1 = X[3 * i + 1], a2 = X[3 * i + 2];
      X[3 * i] = a0 * y00 + a1 * y01 + a2 * y02;
      X[3 * i + 1] = a0 * y01 + a1 * y11 + a2 * y12;
      X[3 * i + 2] = a0 * y02 + a1 * y12 + a2 * y22;
    }
    if (d < 1e-16) {
#pragma unroll
      for (int i = 0; i < 9; ++i) R[i] = X[i];
      return;
    }
  }
  polar_newton(F, R);
}

// 1/sqrt(x) for normal x > 0 without the libm slow-path call (whose register saves would put the caller's live
// values in local memory): hardware approximation + two Newton steps (relative error a few ulp of fp64).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double h = x * y;
  double r = fma(-h, y, 1.0);
  y = fma(0.5 * y, r, y);
  h = x * y;
  r = fma(-h, y, 1.0);
  return fma(0.5 * y, r, y);
}

// K1's polar without address-taken arrays on the common path: Newton-Schulz inline (as polar_rotation);
// returns false when F needs the SVD or scaled-Newton fallback (det F <= 1e-6 ||F||^3, or no convergence in 14
// iterations).  F and R stay in registers: no call frame, no local memory on the common path.
__device__ __forceinline__ bool polar_ns(const double (&F)[9], double (&R)[9], int* its = nullptr) {
  const double d0 = det3(F);
  double fn2 = 0;
#pragma unroll
  for (int i = 0; i < 9; ++i) fn2 += F[i] * F[i];
  if (!(fn2 > 1e-250)) return false;
  const double ifn = rsqrt_nr(fn2);  // 1/||F||_F
  if (!(d0 > 1e-6 * fn2 * fn2 * ifn)) return false;
  const double c = 1.7320508075688772 * ifn;  // sqrt(3)/||F||_F
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = c * F[i];
  for (int it = 0; it < 14; ++it) {
    const double c00 = R[0] * R[0] + R[3] * R[3] + R[6] * R[6];
    const double c11 = R[1] * R[1] + R[4] * R[4] + R[7] * R[7];
    const double c22 = R[2] * R[2] + R[5] * R[5] + R[8] * R[8];
    const double c01 = R[0] * R[1] + R[3] * R[4] + R[6] * R[7];
    const double c02 = R[0] * R[2] + R[3] * R[5] + R[6] * R[8];
    const double c12 = R[1] * R[2] + R[4] * R[5] + R[7] * R[8];
    const double d = (c00 - 1) * (c00 - 1) + (c11 - 1) * (c11 - 1) + (c22 - 1) * (c22 - 1) +
                     2.0 * (c01 * c01 + c02 * c02 + c12 * c12);
    const double y00 = 1.5 - 0.5 * c00, y11 = 1.5 - 0.5 * c11, y22 = 1.5 - 0.5 * c22;
    const double y01 = -0.5 * c01, y02 = -0.5 * c02, y12 = -0.5 * c12;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double a0 = R[3 * i], a1 = R[3 * i + 1], a2 = R[3 * i + 2];
      R[3 * i] = a0 * y00 + a1 * y01 + a2 * y02;
      R[3 * i + 1] = a0 * y01 + a1 * y11 + a2 * y12;
      R[3 * i + 2] = a0 * y02 + a1 * y12 + a2 * y22;
    }
    if (d < 1e-16) {
      if (its) *its = it + 1;  // (statistics hook only; K1 passes nothing and the count is compiled out)
      return true;
    }
  }
  return false;
}

// ----------------------------------------------------------------- layout kernels
__global__ void k_abi_to_state(const double* __restrict__ in, double* __restrict__ out, int n3, int B,
                               int64_t in_bstride = -1) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)n3 * B) return;
  const int64_t d = i / B;
  const int b = (int)(i - d * B);
  out[i] = in[(int64_t)b * (in_bstride < 0 ? n3 : in_bstride) + d];
}
// OUT[i] += in (ABI layout, batch stride in_bstride) on non-Dirichlet DoFs (per-step loss terms)
__global__ void k_add_abi(double* __restrict__ out, const double* __restrict__ in, int n3, int B, int64_t in_bstride,
                          const uint8_t* __restrict__ fixed) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)n3 * B) return;
  const int64_t d = i / B;
  const int b = (int)(i - d * B);
  if (fixed[d / 3]) return;
  out[i] += in[(int64_t)b * in_bstride + d];
}
__global__ void k_state_to_abi(const double* __restrict__ in, double* __restrict__ out, int n3, int B,
                               int64_t out_bstride) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)n3 * B) return;
  const int64_t d = i / B;
  const int b = (int)(i - d * B);
  out[(int64_t)b * out_bstride + d] = in[i];
}

// ---- general contact plane n . x = d: the library works in plane coordinates
// x' = Q x - d e_z (Q n = e_z); the PD energy is invariant under this rigid motion, so only the ABI boundary changes.
// One thread per (node, sim): the node's three components.
struct FrameQ {
  double q[9];  // row-major rotation, rows t1, t2, n
  double d;     // plane offset along the unit normal
};
// ABI [B][bstride] (world) -> state [n][3][B] (plane): point = positions (affine), else vectors
__global__ void k_abi_to_state_frame(const double* __restrict__ in, double* __restrict__ out, int n, int B,
                                     int64_t bstride, FrameQ f, int point) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * B) return;
  const int node = (int)(i / B), b = (int)(i - (int64_t)node * B);
  const double* v = in + (int64_t)b * bstride + 3 * (int64_t)node;
  const double v0 = v[0], v1 = v[1], v2 = v[2];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    double o = f.q[3 * r] * v0 + f.q[3 * r + 1] * v1 + f.q[3 * r + 2] * v2;
    if (point && r == 2) o -= f.d;
    out[((int64_t)node * 3 + r) * B + b] = o;
  }
}
// state [n][3][B] (plane) -> ABI [B][bstride] (world): x = Q^T (x' + d e_z)
__global__ void k_state_to_abi_frame(const double* __restrict__ in, double* __restrict__ out, int n, int B,
                                     int64_t bstride, FrameQ f, int point) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * B) return;
  const int node = (int)(i / B), b = (int)(i - (int64_t)node * B);
  const double* v = in + (int64_t)node * 3 * B + b;
  const double v0 = v[0], v1 = v[B], v2 = v[2 * B] + (point ? f.d : 0.0);
  double* o = out + (int64_t)b * bstride + 3 * (int64_t)node;
#pragma unroll
  for (int c = 0; c < 3; ++c) o[c] = f.q[c] * v0 + f.q[3 + c] * v1 + f.q[6 + c] * v2;
}
// OUT += Q in (vectors, ABI -> state) on non-Dirichlet nodes (per-step loss terms in plane coordinates)
__global__ void k_add_abi_frame(double* __restrict__ out, const double* __restrict__ in, int n, int B, int64_t bstride,
                                const uint8_t* __restrict__ fixed, FrameQ f) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * B) return;
  const int node = (int)(i / B), b = (int)(i - (int64_t)node * B);
  if (fixed[node]) return;
  const double* v = in + (int64_t)b * bstride + 3 * (int64_t)node;
  const double v0 = v[0], v1 = v[1], v2 = v[2];
#pragma unroll
  for (int r = 0; r < 3; ++r)
    out[((int64_t)node * 3 + r) * B + b] += f.q[3 * r] * v0 + f.q[3 * r + 1] * v1 + f.q[3 * r + 2] * v2;
}

// y = x + h v + h^2 (g + f_ext / m)
__global__ void k_y(const double* __restrict__ X, const double* __restrict__ V,
                    const double* __restrict__ Fext, const double* __restrict__ mass, double* __restrict__ Y,
                    int n, int B, double h, double g0, double g1, double g2) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)3 * n * B) return;
  const int64_t d = i / B;
  const int node = (int)(d / 3), ax = (int)(d - 3 * (int64_t)node);
  const double g = ax == 0 ? g0 : (ax == 1 ? g1 : g2);
  const double f = Fext ? Fext[i] / mass[node] : 0.0;
  Y[i] = X[i] + h * V[i] + h * h * (g + f);
}

// fiber direction of element e: the per-element field (material.fiber_dir) or the uniform Stencil fiber
__device__ __forceinline__ void fiber_of(const Stencil& st, const ElemArgs& ea, int e, double (&mf)[3]) {
  if (ea.fib) {
#pragma unroll
    for (int j = 0; j < 3; ++j) mf[j] = __ldg(ea.fib + 3 * (int64_t)e + j);
  } else {
#pragma unroll
    for (int j = 0; j < 3; ++j) mf[j] = st.fiber[j];
  }
}

// ----------------------------------------------------------------- K1: local step
#ifndef K1_MIN_BLOCKS
#define K1_MIN_BLOCKS 5  // resident 256-thread blocks per SM the register allocation targets
#endif
// One thread per (element, sim, quad point), q fastest: the 8 quadrature points of an
// (element, sim) pair are 8 consecutive lanes; their 24 nodal force contributions are summed by a
// 3-stage xor butterfly (identical bits in all 8 lanes: fixed pairing, commutative adds), then lane q
// stores components 3q..3q+2.  No atomics; deterministic.
__device__ __forceinline__ double qsum8(double v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  return v;
}

// Shape-function gradient of the voxel stencil at quad point q, corner a, axis j (reading §2.1):
// dN_a/dX_j = s_j(a)/(4 dx) prod_{k != j} (1 + s_k(a) xi_k(q)); each factor is (1 + 1/sqrt3) when bit k
// of a equals bit k of q, else (1 - 1/sqrt3) -> one of three magnitudes (st.m3), computed from bits so
// that lanes with different q never diverge on a constant-bank index.
__device__ __forceinline__ double dNf(const Stencil& st, int q, int a, int j) {
  const int n = __popc(~(a ^ q) & 7 & ~(1 << j));
  const double mag = n == 2 ? st.m3[2] : (n == 1 ? st.m3[1] : st.m3[0]);
  return ((a >> j) & 1) ? mag : -mag;
}

// Per-block tables of dN_a/dX_j (from dNf, so bit-identical): f[(a*3 + j)*8 + q] (load_F: lanes = q, one
// 64-byte row per (a, j)) and b[(q*3 + j)*8 + a] (store_force: lanes = a).  One shared-memory load replaces
// dNf's integer work per use.
struct DNTab {
  double f[192], b[192];
};
__device__ __forceinline__ void dn_fill(DNTab& t, const Stencil& st) {
  for (int i = threadIdx.x; i < 192; i += blockDim.x) {
    const int x = i / 24, j = (i / 8) % 3, y = i % 8;
    t.f[i] = dNf(st, y, x, j);
    t.b[i] = dNf(st, x, y, j);
  }
  __syncthreads();
}

// Deformation gradient F = G_q x_e at quad point q of element e, sim b (state layout [n][3][B]).
__device__ __forceinline__ void load_F(const double* __restrict__ X, const int32_t* __restrict__ hex8,
                                       const DNTab& dt, int e, int b, int q, int B, double* F) {
#pragma unroll
  for (int k = 0; k < 9; ++k) F[k] = 0.0;
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int node = __ldg(hex8 + 8 * (int64_t)e + a);
    const double d0 = dt.f[(a * 3) * 8 + q], d1 = dt.f[(a * 3 + 1) * 8 + q], d2 = dt.f[(a * 3 + 2) * 8 + q];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double xv = __ldg(X + (3 * (int64_t)node + i) * B + b);
      F[3 * i] = fma(xv, d0, F[3 * i]);
      F[3 * i + 1] = fma(xv, d1, F[3 * i + 1]);
      F[3 * i + 2] = fma(xv, d2, F[3 * i + 2]);
    }
  }
}

// Element force sum_q G_q^T P_q of the (e, b) group (8 consecutive lanes, lane q holds P_q): the 8 P_q
// go through shared memory (group-private, padded rows), then lane a forms the 3 components of corner
// a in a fixed q order: EF[e][a][i][b].  Ps = this group's kPsSlot-double slot: P_q at 10 q (16-byte
// aligned, read back with 128-bit loads); slots 82 doubles apart so the 4 groups of a warp hit distinct banks.
constexpr int kPsSlot = 82;
__device__ __forceinline__ void store_force(const double* Pm, const DNTab& dt, int e, int b, int q, int B,
                                            double* Ps, double* __restrict__ EF) {
#pragma unroll
  for (int k = 0; k < 9; ++k) Ps[10 * q + k] = Pm[k];
  __syncwarp();
  const int a = q;
  double o0 = 0, o1 = 0, o2 = 0;
#pragma unroll
  for (int qq = 0; qq < 8; ++qq) {
    const double d0 = dt.b[(qq * 3) * 8 + a], d1 = dt.b[(qq * 3 + 1) * 8 + a], d2 = dt.b[(qq * 3 + 2) * 8 + a];
    const double2* P2 = reinterpret_cast<const double2*>(Ps + 10 * qq);
    const double2 p01 = P2[0], p23 = P2[1], p45 = P2[2], p67 = P2[3];
    const double p8 = Ps[10 * qq + 8];
    o0 = fma(p01.x, d0, fma(p01.y, d1, fma(p23.x, d2, o0)));
    o1 = fma(p23.y, d0, fma(p45.x, d1, fma(p45.y, d2, o1)));
    o2 = fma(p67.x, d0, fma(p67.y, d1, fma(p8, d2, o2)));
  }
  __syncwarp();
  if (EF) {
    double* o = EF + ((8 * (int64_t)e + a) * 3) * B + b;
    o[0] = o0;
    o[B] = o1;
    o[2 * B] = o2;
  }
}

// K1's rare fallback (SVD / scaled Newton, polar_rotation): recomputes F from x itself so that the caller's F
// never needs an address; R goes to `out` (the thread's slot of the group's shared-memory area).
__device__ __noinline__ void k1_polar_fallback(const double* __restrict__ X, const int32_t* __restrict__ hex8,
                                               const DNTab* dt, int e, int b, int q, int B, double* out) {
  double F[9], R[9];
  load_F(X, hex8, *dt, e, b, q, B, F);
  polar_rotation(F, R);
  for (int k = 0; k < 9; ++k) out[k] = R[k];
}

// FIB: per-element fiber field (material.fiber_dir); the uniform-fiber instance reads the fiber from the kernel
// parameters (no registers held for it: the tuned corotated/muscle path keeps its allocation)
template <bool FIB>
__global__ void __launch_bounds__(256, K1_MIN_BLOCKS) k_elem_residual(const double* __restrict__ X, Stencil st,
                                                                    ElemArgs ea, double* __restrict__ EF,
                                                                    double* __restrict__ EE) {
  PDL_ENTRY();
  __shared__ DNTab dnt;
  __shared__ __align__(16) double Psm[32][kPsSlot];
  dn_fill(dnt, st);
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int B = ea.B;
  const int64_t pair = tid >> 3;
  const int q = (int)(tid & 7);
  // dead lanes (past the end) compute on pair 0 and store nothing: every shuffle sees a full warp
  const bool live = pair < (int64_t)ea.m * B;
  const int pr = live ? (int)pair : 0;  // (m B < 2^31: 32-bit division, no 64-bit division call)
  const int e = pr / B, b = pr - e * B;
  const double w = ea.w_sim[b];
  double F[9], R[9];
  load_F(X, ea.hex8, dnt, e, b, q, B, F);
  if (!polar_ns(F, R)) {  // rare: SVD (det F <= 1e-6 ||F||^3) or scaled Newton; R through this thread's slot
    double* slot = &Psm[threadIdx.x >> 3][10 * q];
    k1_polar_fallback(X, ea.hex8, &dnt, e, b, q, B, slot);
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = slot[k];
  }
  double Pm[9];
  double en = 0;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const double dk = F[k] - R[k];
    en += dk * dk;
    Pm[k] = w * st.V * dk;
  }
  double energy = 0.5 * w * st.V * en;
  if (st.w_m != 0.0) {
    const double r_act = ea.act ? ea.act[(int64_t)b * ea.act_bstride + e] : 0.0;
    double mf[3];
    if constexpr (FIB) {
      fiber_of(st, ea, e, mf);
    } else {
#pragma unroll
      for (int j = 0; j < 3; ++j) mf[j] = st.fiber[j];
    }
    double Fm[3], nr2 = 0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      Fm[i] = F[3 * i] * mf[0] + F[3 * i + 1] * mf[1] + F[3 * i + 2] * mf[2];
      nr2 += Fm[i] * Fm[i];
    }
    const bool pos = nr2 > 1e-250;
    const double s_act = pos ? r_act * rsqrt_nr(nr2) : 0.0;  // r / ||Fm||
    double dm[3], em = 0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double p = pos ? s_act * Fm[i] : r_act * mf[i];
      dm[i] = Fm[i] - p;
      em += dm[i] * dm[i];
    }
    energy += 0.5 * st.w_m * st.V * em;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) Pm[3 * i + j] += st.w_m * st.V * dm[i] * mf[j];
  }
  __syncwarp();  // (the slot may have carried a fallback R: every lane has read its own before it is reused)
  store_force(Pm, dnt, e, b, q, B, Psm[threadIdx.x >> 3], live ? EF : nullptr);
  energy = qsum8(energy);
  if (live && EE && q == 0) EE[(int64_t)e * B + b] = energy;
}

// Local-step statistics (diagnostic, pd_polar_stats): per quadrature point of x, the Newton-Schulz iterations K1's
// polar takes (or the fallback); acc[0] += iterations, acc[1] += points on the Newton-Schulz path, acc[2] +=
// fallback points.  Integer sums: exact and order-independent.
__global__ void k_polar_stats(const double* __restrict__ X, Stencil st, const int32_t* __restrict__ hex8, int m, int B,
                              unsigned long long* __restrict__ acc) {
  PDL_ENTRY();
  __shared__ DNTab dnt;
  dn_fill(dnt, st);
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t pair = tid >> 3;
  const int q = (int)(tid & 7);
  unsigned long long it_sum = 0, ns = 0, fb = 0;
  if (pair < (int64_t)m * B) {
    const int e = (int)(pair / B), b = (int)(pair - (int64_t)e * B);
    double F[9], R[9];
    load_F(X, hex8, dnt, e, b, q, B, F);
    int its = 0;
    if (polar_ns(F, R, &its)) {
      it_sum = (unsigned long long)its;
      ns = 1;
    } else {
      fb = 1;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    it_sum += __shfl_down_sync(0xffffffffu, it_sum, o);
    ns += __shfl_down_sync(0xffffffffu, ns, o);
    fb += __shfl_down_sync(0xffffffffu, fb, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(acc, it_sum);
    atomicAdd(acc + 1, ns);
    atomicAdd(acc + 2, fb);
  }
}

// Rotations of every quad point (diagnostic / parity hook).
__global__ void k_elem_rotations(const double* __restrict__ X, Stencil st, const int32_t* __restrict__ hex8,
                                 int m, int B, double* __restrict__ Rout) {
  PDL_ENTRY();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= (int64_t)m * B) return;
  const int e = (int)(tid / B), b = (int)(tid - (int64_t)e * B);
  double xe[8][3];
  for (int a = 0; a < 8; ++a) {
    const int node = hex8[8 * (int64_t)e + a];
    for (int i = 0; i < 3; ++i) xe[a][i] = X[(3 * (int64_t)node + i) * B + b];
  }
  for (int q = 0; q < 8; ++q) {
    double F[9], R[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double s = 0;
        for (int a = 0; a < 8; ++a) s += xe[a][i] * dNf(st, q, a, j);
        F[3 * i + j] = s;
      }
    polar_rotation(F, R);
    for (int k = 0; k < 9; ++k) Rout[(((int64_t)b * m + e) * 8 + q) * 9 + k] = R[k];
  }
}

// ----------------------------------------------------------------- K4: A_N p (matrix-free)
// dR[dF] = R [w]x with (tr S I - S) w = vee(R^T dF - dF^T R), eigenvalues floored at
// clamp * max|eig S|; muscle dp = (r/||Fm||)(I - n n^T) dFm.
// Mi = (tr S I - S)^{-1} (symmetric; stored xx, xy, xz, yy, yz, zz), eigenvalues floored at
// clamp * max|eig S|.  Fast path: Cholesky positivity test of (M - floor I), then the
// cofactor inverse; clamped path: Jacobi eigen-decomposition.
__device__ void rot_derivative_matrix(const double* S, double clamp, double* Mi) {
  double tr = S[0] + S[4] + S[8];
  double M[9];
  for (int i = 0; i < 9; ++i) M[i] = -S[i];
  M[0] += tr; M[4] += tr; M[8] += tr;
  double sn = 0;
  for (int i = 0; i < 9; ++i) sn += S[i] * S[i];
  const double fub = clamp * sqrt(sn);  // >= clamp * max|eig S|
  const double a00 = M[0] - fub, a11 = M[4] - fub, a22 = M[8] - fub;
  bool fast = a00 > 0;
  double l10 = 0, l20 = 0, l11 = 0, l21 = 0;
  if (fast) {
    const double l00 = sqrt(a00);
    l10 = M[3] / l00; l20 = M[6] / l00;
    const double t11 = a11 - l10 * l10;
    fast = t11 > 0;
    if (fast) {
      l11 = sqrt(t11);
      l21 = (M[7] - l20 * l10) / l11;
      fast = a22 - l20 * l20 - l21 * l21 > 0;
    }
  }
  if (fast) {
    double C[9];
    cof3(M, C);  // M symmetric: M^{-1} = C / det
    const double idet = 1.0 / (M[0] * C[0] + M[1] * C[1] + M[2] * C[2]);
    Mi[0] = C[0] * idet; Mi[1] = C[1] * idet; Mi[2] = C[2] * idet;
    Mi[3] = C[4] * idet; Mi[4] = C[5] * idet; Mi[5] = C[8] * idet;
    return;
  }
  double lam[3], V[9];
  jacobi_eig3(S, lam, V);
  const double mx = fmax(fabs(lam[0]), fmax(fabs(lam[1]), fabs(lam[2])));
  const double floor_ = clamp * mx;
  double iv[3];
  for (int k = 0; k < 3; ++k) iv[k] = 1.0 / fmax(tr - lam[k], floor_);
  const int pr[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
  for (int t = 0; t < 6; ++t) {
    const int i = pr[t][0], j = pr[t][1];
    Mi[t] = V[3 * i] * iv[0] * V[3 * j] + V[3 * i + 1] * iv[1] * V[3 * j + 1] + V[3 * i + 2] * iv[2] * V[3 * j + 2];
  }
}

// S = sym(R^T F)
__device__ __forceinline__ void sym_stretch(const double* R, const double* F, double* S) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) S[3 * i + j] = R[i] * F[j] + R[3 + i] * F[3 + j] + R[6 + i] * F[6 + j];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = i + 1; j < 3; ++j) {
      const double avg = 0.5 * (S[3 * i + j] + S[3 * j + i]);
      S[3 * i + j] = S[3 * j + i] = avg;
    }
}

// Pm = w V (dF - dR[dF]) (+ muscle w_m V (dFm - s (dFm - (n.dFm) n)) m^T): the projection-derivative
// term of A_N p, dR = R [om]x, om = Mi vee(R^T dF - dF^T R).
__device__ __forceinline__ void an_stress(const double* R, const double* Mi, const double* dF, double wv,
                                          const Stencil& st, bool mus, const double* nh, double sc, double* Pm,
                                          const double* mf) {
  double Wm[9];  // R^T dF
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) Wm[3 * i + j] = R[i] * dF[j] + R[3 + i] * dF[3 + j] + R[6 + i] * dF[6 + j];
  const double r0 = Wm[7] - Wm[5], r1 = Wm[2] - Wm[6], r2 = Wm[3] - Wm[1];
  const double om0 = Mi[0] * r0 + Mi[1] * r1 + Mi[2] * r2;
  const double om1 = Mi[1] * r0 + Mi[3] * r1 + Mi[4] * r2;
  const double om2 = Mi[2] * r0 + Mi[4] * r1 + Mi[5] * r2;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double a0 = R[3 * i], a1 = R[3 * i + 1], a2 = R[3 * i + 2];
    Pm[3 * i] = wv * (dF[3 * i] - (a1 * om2 - a2 * om1));
    Pm[3 * i + 1] = wv * (dF[3 * i + 1] - (-a0 * om2 + a2 * om0));
    Pm[3 * i + 2] = wv * (dF[3 * i + 2] - (a0 * om1 - a1 * om0));
  }
  if (mus) {
    double dFm[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) dFm[i] = dF[3 * i] * mf[0] + dF[3 * i + 1] * mf[1] + dF[3 * i + 2] * mf[2];
    const double nd = nh[0] * dFm[0] + nh[1] * dFm[1] + nh[2] * dFm[2];
    const double wm = st.w_m * st.V;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double jd = sc * (dFm[i] - nd * nh[i]);
#pragma unroll
      for (int j = 0; j < 3; ++j) Pm[3 * i + j] += wm * (dFm[i] - jd) * mf[j];
    }
  }
}

// muscle data at F: n = Fm/||Fm||, sc = r/||Fm|| (0 if ||Fm|| = 0)
__device__ __forceinline__ void muscle_dir(const double* F, const double* mf, double r_act, double* nh, double& sc) {
  double Fm[3], nr = 0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    Fm[i] = F[3 * i] * mf[0] + F[3 * i + 1] * mf[1] + F[3 * i + 2] * mf[2];
    nr += Fm[i] * Fm[i];
  }
  nr = sqrt(nr);
  if (nr > 0) {
#pragma unroll
    for (int i = 0; i < 3; ++i) nh[i] = Fm[i] / nr;
    sc = r_act / nr;
  } else {
#pragma unroll
    for (int i = 0; i < 3; ++i) nh[i] = mf[i];
    sc = 0.0;
  }
}

constexpr int kJC = 19;  // cached doubles per quad point: R (9), Mi (6), n (3), sc (1)

// Per-step Jacobian data at x_{i+1} ("needs to be done only once per time step"), SoA:
// JC[k * nq + tid], tid = (e*B + b)*8 + q.
__global__ void __launch_bounds__(256) k_elem_jac(const double* __restrict__ X, Stencil st, ElemArgs ea,
                                                  double* __restrict__ JC) {
  PDL_ENTRY();
  __shared__ DNTab dnt;
  dn_fill(dnt, st);
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nq = (int64_t)ea.m * ea.B * 8;
  if (tid >= nq) return;
  const int B = ea.B;
  const int64_t pair = tid >> 3;
  const int q = (int)(tid & 7);
  const int e = (int)(pair / B), b = (int)(pair - (int64_t)e * B);
  double F[9], R[9], S[9], Mi[6];
  load_F(X, ea.hex8, dnt, e, b, q, B, F);
  polar_rotation(F, R);
  sym_stretch(R, F, S);
  rot_derivative_matrix(S, st.clamp, Mi);
#pragma unroll
  for (int k = 0; k < 9; ++k) JC[k * nq + tid] = R[k];
#pragma unroll
  for (int k = 0; k < 6; ++k) JC[(9 + k) * nq + tid] = Mi[k];
  if (st.w_m != 0.0) {
    double nh[3], sc, mf[3];
    fiber_of(st, ea, e, mf);
    muscle_dir(F, mf, ea.act ? ea.act[(int64_t)b * ea.act_bstride + e] : 0.0, nh, sc);
#pragma unroll
    for (int k = 0; k < 3; ++k) JC[(15 + k) * nq + tid] = nh[k];
    JC[18 * nq + tid] = sc;
  }
}

// K4 with cached Jacobian data: A_N p element term from dF = G_q p_e only (no polar per product).
__global__ void __launch_bounds__(256) k_elem_AN_cached(const double* __restrict__ Pv, Stencil st, ElemArgs ea,
                                                        const double* __restrict__ JC, double* __restrict__ EF) {
  PDL_ENTRY();
  __shared__ DNTab dnt;
  dn_fill(dnt, st);
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int B = ea.B;
  const int64_t nq = (int64_t)ea.m * B * 8;
  const int64_t pair = tid >> 3;
  const int q = (int)(tid & 7);
  const bool live = pair < (int64_t)ea.m * B;
  const int64_t pr = live ? pair : 0;
  const int64_t t = live ? tid : q;
  const int e = (int)(pr / B), b = (int)(pr - (int64_t)e * B);
  double dF[9], R[9], Mi[6], nh[3] = {0, 0, 0}, sc = 0;
  load_F(Pv, ea.hex8, dnt, e, b, q, B, dF);
#pragma unroll
  for (int k = 0; k < 9; ++k) R[k] = __ldg(JC + k * nq + t);
#pragma unroll
  for (int k = 0; k < 6; ++k) Mi[k] = __ldg(JC + (9 + k) * nq + t);
  const bool mus = st.w_m != 0.0;
  double mf[3] = {0, 0, 0};
  if (mus) {
#pragma unroll
    for (int k = 0; k < 3; ++k) nh[k] = __ldg(JC + (15 + k) * nq + t);
    sc = __ldg(JC + 18 * nq + t);
    fiber_of(st, ea, e, mf);
  }
  double Pm[9];
  an_stress(R, Mi, dF, ea.w_sim[b] * st.V, st, mus, nh, sc, Pm, mf);
  __shared__ __align__(16) double Psm[32][kPsSlot];
  store_force(Pm, dnt, e, b, q, B, Psm[threadIdx.x >> 3], live ? EF : nullptr);
}

__global__ void __launch_bounds__(256) k_elem_AN(const double* __restrict__ X, const double* __restrict__ Pv,
                                                 Stencil st, ElemArgs ea, double* __restrict__ EF) {
  PDL_ENTRY();
  __shared__ DNTab dnt;
  dn_fill(dnt, st);
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int B = ea.B;
  const int64_t pair = tid >> 3;
  const int q = (int)(tid & 7);
  const bool live = pair < (int64_t)ea.m * B;
  const int64_t pr = live ? pair : 0;
  const int e = (int)(pr / B), b = (int)(pr - (int64_t)e * B);
  double F[9], dF[9], R[9], S[9], Mi[6], nh[3] = {0, 0, 0}, sc = 0;
  load_F(X, ea.hex8, dnt, e, b, q, B, F);
  load_F(Pv, ea.hex8, dnt, e, b, q, B, dF);
  polar_rotation(F, R);
  sym_stretch(R, F, S);
  rot_derivative_matrix(S, st.clamp, Mi);
  const bool mus = st.w_m != 0.0;
  double mf[3] = {0, 0, 0};
  if (mus) {
    fiber_of(st, ea, e, mf);
    muscle_dir(F, mf, ea.act ? ea.act[(int64_t)b * ea.act_bstride + e] : 0.0, nh, sc);
  }
  double Pm[9];
  an_stress(R, Mi, dF, ea.w_sim[b] * st.V, st, mus, nh, sc, Pm, mf);
  __shared__ __align__(16) double Psm[32][kPsSlot];
  store_force(Pm, dnt, e, b, q, B, Psm[threadIdx.x >> 3], live ? EF : nullptr);
}

// Parameter-gradient terms at x_{i+1} for adjoint u (chain rule):
//   DW[e][b] = -sum_q V <G_q u_e, F_q - R_q>,  DR[e][b] = w_m sum_q V n_hat^T (G_q u_e) m
__global__ void __launch_bounds__(256) k_elem_param(const double* __restrict__ X, const double* __restrict__ U,
                                                    Stencil st, ElemArgs ea, double* __restrict__ DW,
                                                    double* __restrict__ DR) {
  PDL_ENTRY();
  __shared__ DNTab dnt;
  dn_fill(dnt, st);
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int B = ea.B;
  const int64_t pair = tid >> 3;
  const int q = (int)(tid & 7);
  const bool live = pair < (int64_t)ea.m * B;
  const int64_t pr = live ? pair : 0;
  const int e = (int)(pr / B), b = (int)(pr - (int64_t)e * B);
  double F[9], dF[9];
  load_F(X, ea.hex8, dnt, e, b, q, B, F);
  load_F(U, ea.hex8, dnt, e, b, q, B, dF);
  double R[9];
  polar_rotation(F, R);
  double acc = 0;
#pragma unroll
  for (int k = 0; k < 9; ++k) acc += dF[k] * (F[k] - R[k]);
  double dw = -st.V * acc, dr = 0;
  if (st.w_m != 0.0 && DR) {
    double Fm[3], dFm[3], nr = 0, mf[3];
    fiber_of(st, ea, e, mf);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      Fm[i] = F[3 * i] * mf[0] + F[3 * i + 1] * mf[1] + F[3 * i + 2] * mf[2];
      dFm[i] = dF[3 * i] * mf[0] + dF[3 * i + 1] * mf[1] + dF[3 * i + 2] * mf[2];
      nr += Fm[i] * Fm[i];
    }
    nr = sqrt(nr);
    double nh[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) nh[i] = nr > 0 ? Fm[i] / nr : mf[i];
    dr = st.w_m * st.V * (nh[0] * dFm[0] + nh[1] * dFm[1] + nh[2] * dFm[2]);
  }
  dw = qsum8(dw);
  dr = qsum8(dr);
  if (live && q == 0) {
    DW[(int64_t)e * B + b] = dw;
    if (DR) DR[(int64_t)e * B + b] = dr;
  }
}

// ----------------------------------------------------------------- volume-preserving term
// (w_v/2)||F - D||^2, D the projection of F onto det D = 1: with R = polar(F) and the symmetric
// S = sym(R^T F) = V diag(s) V^T (s the signed singular values, U = R V), d* = argmin ||d||^2 s.t. prod(s + d) = 1
// by Newton on the KKT system from d = 0 (same iteration and stopping rule as the oracle), g = s + d*,
// D = R V diag(g) V^T.  Jacobian: J = dg/ds from the differentiated KKT system (eq:vol_kkt); dD[dF] =
// U M V^T with P = U^T dF V, M_ii = (J diag P)_i, M_ij = (g_i - g_j)/(s_i - s_j) sym(P)_ij + (g_i + g_j)/(s_i +
// s_j) skew(P)_ij (limit J_ii - J_ij for s_i = s_j; s_i + s_j floored at clamp max|s|).  These helpers run only
// when the term is enabled and are not inlined, so the corotated-only kernels keep their registers.

// x = K^{-1} rhs for a 4 x 4 K (row-major, overwritten) and nr right-hand sides rhs[4][nr]: Gaussian elimination
// with partial pivoting
__device__ void solve4(double* K, double* rhs, int nr) {
  for (int c = 0; c < 4; ++c) {
    int p = c;
    for (int r = c + 1; r < 4; ++r)
      if (fabs(K[4 * r + c]) > fabs(K[4 * p + c])) p = r;
    if (p != c) {
      for (int k = 0; k < 4; ++k) { const double t = K[4 * c + k]; K[4 * c + k] = K[4 * p + k]; K[4 * p + k] = t; }
      for (int k = 0; k < nr; ++k) { const double t = rhs[c * nr + k]; rhs[c * nr + k] = rhs[p * nr + k]; rhs[p * nr + k] = t; }
    }
    const double ip = 1.0 / K[4 * c + c];
    for (int r = c + 1; r < 4; ++r) {
      const double f = K[4 * r + c] * ip;
      for (int k = c; k < 4; ++k) K[4 * r + k] -= f * K[4 * c + k];
      for (int k = 0; k < nr; ++k) rhs[r * nr + k] -= f * rhs[c * nr + k];
    }
  }
  for (int c = 3; c >= 0; --c) {
    for (int k = 0; k < nr; ++k) {
      double v = rhs[c * nr + k];
      for (int j = c + 1; j < 4; ++j) v -= K[4 * c + j] * rhs[j * nr + k];
      rhs[c * nr + k] = v / K[4 * c + c];
    }
  }
}

// KKT matrix [I + lam Hc, gc; gc^T, 0] at z = s + d and the constraint gradient gc
__device__ void vol_kkt_matrix(const double* z, double lam, double* K, double* gc) {
  gc[0] = z[1] * z[2];
  gc[1] = z[0] * z[2];
  gc[2] = z[0] * z[1];
  const double H01 = z[2], H02 = z[1], H12 = z[0];
  K[0] = 1.0; K[1] = lam * H01; K[2] = lam * H02; K[3] = gc[0];
  K[4] = lam * H01; K[5] = 1.0; K[6] = lam * H12; K[7] = gc[1];
  K[8] = lam * H02; K[9] = lam * H12; K[10] = 1.0; K[11] = gc[2];
  K[12] = gc[0]; K[13] = gc[1]; K[14] = gc[2]; K[15] = 0.0;
}

// d*, lam* (Newton from 0; stops after the step following the first residual <= 1e-13) and g = s + d*
__device__ void vol_kkt(const double* s, double* g, double& lam) {
  double d[3] = {0.0, 0.0, 0.0};
  lam = 0.0;
  bool last = false;
  for (int it = 0; it < 60; ++it) {
    const double z[3] = {s[0] + d[0], s[1] + d[1], s[2] + d[2]};
    double K[16], gc[3];
    vol_kkt_matrix(z, lam, K, gc);
    double r[4] = {d[0] + lam * gc[0], d[1] + lam * gc[1], d[2] + lam * gc[2], z[0] * z[1] * z[2] - 1.0};
    if (last) break;
    if (fmax(fmax(fabs(r[0]), fabs(r[1])), fmax(fabs(r[2]), fabs(r[3]))) <= 1e-13) last = true;
    for (int k = 0; k < 4; ++k) r[k] = -r[k];
    solve4(K, r, 1);
    d[0] += r[0]; d[1] += r[1]; d[2] += r[2];
    lam += r[3];
  }
  for (int i = 0; i < 3; ++i) g[i] = s[i] + d[i];
}

// J = dg/ds (3 x 3, row-major) from eq:vol_kkt: [K] [dd; dlam] = [-lam Hc e_k; -gc_k]
__device__ void vol_jac(const double* s, const double* g, double lam, double* J) {
  double K[16], gc[3];
  vol_kkt_matrix(g, lam, K, gc);
  const double H[9] = {0.0, g[2], g[1], g[2], 0.0, g[0], g[1], g[0], 0.0};
  double rhs[12];
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) rhs[i * 3 + k] = -lam * H[3 * i + k];
  for (int k = 0; k < 3; ++k) rhs[9 + k] = -gc[k];
  solve4(K, rhs, 3);
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) J[3 * i + k] = (i == k ? 1.0 : 0.0) + rhs[i * 3 + k];
  (void)s;
}

// projection data at F: R (input, the polar rotation), V, s (signed singular values), g, J
__device__ void vol_data(const double* F, const double* R, double* V, double* s, double* g, double* J) {
  double S[9], lam;
  sym_stretch(R, F, S);
  jacobi_eig3(S, s, V);
  vol_kkt(s, g, lam);
  vol_jac(s, g, lam, J);
}

// dD[dF] = U M V^T, U = R V (the chain rule above)
__device__ void vol_dD(const double* R, const double* V, const double* s, const double* g, const double* J,
                       double clamp, const double* dF, double* dD) {
  double U[9], P[9], T[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) U[3 * i + j] = R[3 * i] * V[j] + R[3 * i + 1] * V[3 + j] + R[3 * i + 2] * V[6 + j];
  for (int i = 0; i < 3; ++i)  // T = dF V
    for (int j = 0; j < 3; ++j) T[3 * i + j] = dF[3 * i] * V[j] + dF[3 * i + 1] * V[3 + j] + dF[3 * i + 2] * V[6 + j];
  for (int i = 0; i < 3; ++i)  // P = U^T T
    for (int j = 0; j < 3; ++j) P[3 * i + j] = U[i] * T[j] + U[3 + i] * T[3 + j] + U[6 + i] * T[6 + j];
  const double smax = fmax(fabs(s[0]), fmax(fabs(s[1]), fabs(s[2])));
  double M[9];
  for (int i = 0; i < 3; ++i) M[4 * i] = J[3 * i] * P[0] + J[3 * i + 1] * P[4] + J[3 * i + 2] * P[8];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      if (i == j) continue;
      const double sym = 0.5 * (P[3 * i + j] + P[3 * j + i]), skw = 0.5 * (P[3 * i + j] - P[3 * j + i]);
      const double ds = s[i] - s[j];
      const double r1 = fabs(ds) <= 1e-9 * smax ? J[3 * i + i] - J[3 * i + j] : (g[i] - g[j]) / ds;
      const double den = fmax(s[i] + s[j], clamp * smax);
      M[3 * i + j] = r1 * sym + (g[i] + g[j]) / den * skw;
    }
  for (int i = 0; i < 3; ++i)  // T = U M
    for (int j = 0; j < 3; ++j) T[3 * i + j] = U[3 * i] * M[j] + U[3 * i + 1] * M[3 + j] + U[3 * i + 2] * M[6 + j];
  for (int i = 0; i < 3; ++i)  // dD = T V^T
    for (int j = 0; j < 3; ++j) dD[3 * i + j] = T[3 * i] * V[3 * j] + T[3 * i + 1] * V[3 * j + 1] + T[3 * i + 2] * V[3 * j + 2];
}

// D = R V diag(g) V^T
__device__ void vol_D(const double* R, const double* V, const double* g, double* D) {
  double SD[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) SD[3 * i + j] = V[3 * i] * g[0] * V[3 * j] + V[3 * i + 1] * g[1] * V[3 * j + 1] + V[3 * i + 2] * g[2] * V[3 * j + 2];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) D[3 * i + j] = R[3 * i] * SD[j] + R[3 * i + 1] * SD[3 + j] + R[3 * i + 2] * SD[6 + j];
}

// Volume-term kernels: one thread per (element, sim, quad point) like K1/K4, launched after the corotated kernel
// of the same pass when material.volume is set; they ADD their element forces to EF (store_force_add) and their
// energy to EE, so the tuned corotated-only kernels keep their register allocation.
__device__ __forceinline__ void store_force_add(const double* Pm, const DNTab& dt, int e, int b, int q, int B,
                                                double* Ps, double* __restrict__ EF) {
#pragma unroll
  for (int k = 0; k < 9; ++k) Ps[10 * q + k] = Pm[k];
  __syncwarp();
  const int a = q;
  double o0 = 0, o1 = 0, o2 = 0;
#pragma unroll
  for (int qq = 0; qq < 8; ++qq) {
    const double d0 = dt.b[(qq * 3) * 8 + a], d1 = dt.b[(qq * 3 + 1) * 8 + a], d2 = dt.b[(qq * 3 + 2) * 8 + a];
    const double* P = Ps + 10 * qq;
    o0 = fma(P[0], d0, fma(P[1], d1, fma(P[2], d2, o0)));
    o1 = fma(P[3], d0, fma(P[4], d1, fma(P[5], d2, o1)));
    o2 = fma(P[6], d0, fma(P[7], d1, fma(P[8], d2, o2)));
  }
  __syncwarp();
  if (EF) {
    double* o = EF + ((8 * (int64_t)e + a) * 3) * B + b;
    o[0] += o0;
    o[B] += o1;
    o[2 * B] += o2;
  }
}

// mode 0 (forward): EF += w_v V G^T (F - D), EE += (w_v V/2) ||F - D||^2
// mode 1 (A_N p, cached): EF += w_v V G^T (dF - dD[dF]) with R and the projection data from the per-step cache
// mode 2 (A_N p, recomputed from x: the pd_apply_AN hook)
// mode 3 (per-step cache): JC slots kJC .. kJC + kJCV of the projection data
// mode 4 (parameter term): DWV[e][b] = -sum_q V <G_q u_e, F_q - D_q>
template <int MODE>
__global__ void __launch_bounds__(256) k_vol(const double* __restrict__ X, const double* __restrict__ Pv, Stencil st,
                                             ElemArgs ea, double* __restrict__ JC, double* __restrict__ EF,
                                             double* __restrict__ EE) {
  PDL_ENTRY();
  __shared__ DNTab dnt;
  __shared__ __align__(16) double Psm[32][kPsSlot];
  dn_fill(dnt, st);
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int B = ea.B;
  const int64_t nq = (int64_t)ea.m * B * 8;
  const int64_t pair = tid >> 3;
  const int q = (int)(tid & 7);
  const bool live = pair < (int64_t)ea.m * B;
  const int pr = live ? (int)pair : 0;
  const int e = pr / B, b = pr - e * B;
  const int64_t t = live ? tid : q;
  const double wv = ea.w_sim[b] * st.kappa * st.V;
  double F[9], R[9], V[9], sv[3], g[3], J[9], dF[9], dD[9], Pm[9];
  if (MODE == 1) {
    load_F(Pv, ea.hex8, dnt, e, b, q, B, dF);
    for (int k = 0; k < 9; ++k) R[k] = JC[k * nq + t];
    for (int k = 0; k < 9; ++k) V[k] = JC[(kJC + k) * nq + t];
    for (int k = 0; k < 3; ++k) sv[k] = JC[(kJC + 9 + k) * nq + t];
    for (int k = 0; k < 3; ++k) g[k] = JC[(kJC + 12 + k) * nq + t];
    const int sy[9] = {0, 1, 2, 1, 3, 4, 2, 4, 5};
    for (int k = 0; k < 9; ++k) J[k] = JC[(kJC + 15 + sy[k]) * nq + t];
  } else {
    load_F(X, ea.hex8, dnt, e, b, q, B, F);
    polar_rotation(F, R);
    vol_data(F, R, V, sv, g, J);
  }
  if (MODE == 3) {
    if (live) {
      for (int k = 0; k < 9; ++k) JC[(kJC + k) * nq + tid] = V[k];
      for (int k = 0; k < 3; ++k) JC[(kJC + 9 + k) * nq + tid] = sv[k];
      for (int k = 0; k < 3; ++k) JC[(kJC + 12 + k) * nq + tid] = g[k];
      const int up[6] = {0, 1, 2, 4, 5, 8};
      for (int k = 0; k < 6; ++k) JC[(kJC + 15 + k) * nq + tid] = J[up[k]];
    }
    return;
  }
  if (MODE == 0 || MODE == 4) {
    double D[9];
    vol_D(R, V, g, D);
    if (MODE == 4) {  // EF = DWV here, Pv = u
      load_F(Pv, ea.hex8, dnt, e, b, q, B, dF);
      double a2 = 0;
      for (int k = 0; k < 9; ++k) a2 += dF[k] * (F[k] - D[k]);
      const double dwv = qsum8(-st.V * a2);
      if (live && q == 0) EF[(int64_t)e * B + b] = dwv;
      return;
    }
    double en = 0;
    for (int k = 0; k < 9; ++k) {
      const double d = F[k] - D[k];
      en += d * d;
      Pm[k] = wv * d;
    }
    en = qsum8(0.5 * wv * en);
    if (live && q == 0 && EE) EE[(int64_t)e * B + b] += en;
  } else {
    if (MODE == 2) load_F(Pv, ea.hex8, dnt, e, b, q, B, dF);
    vol_dD(R, V, sv, g, J, st.clamp, dF, dD);
    for (int k = 0; k < 9; ++k) Pm[k] = wv * (dF[k] - dD[k]);
  }
  store_force_add(Pm, dnt, e, b, q, B, Psm[threadIdx.x >> 3], live ? EF : nullptr);
}
constexpr int kJCV = 21;  // extra cached doubles per quad point with the volume term

// ----------------------------------------------------------------- K2: deterministic gather
// mode 0: G = M/h^2 (X - Y) + sum EF   (grad g)       W = M/h^2 Y  (residual normaliser)
// mode 1: G = M/h^2 X + sum EF         (A_N p, X = p)  W unused
// Constrained DoFs (fixed nodes; pinned z DoFs when PIN != null) get G = 0, W = 0; the raw
// value of a pinned DoF is stored in LAM[j*B + b] (contact multiplier).
__global__ void k_gather(const double* __restrict__ X, const double* __restrict__ Y, const double* __restrict__ EF,
                         const double* __restrict__ mass, const int32_t* __restrict__ inc_ptr,
                         const int32_t* __restrict__ inc_ec, const uint8_t* __restrict__ fixed,
                         const int32_t* __restrict__ pos_of_node, int n, int B, double inv_h2, int mode,
                         double* __restrict__ G, double* __restrict__ W, double* __restrict__ RHS,
                         const int32_t* __restrict__ cand_of_node, const uint8_t* __restrict__ PIN,
                         double* __restrict__ LAM, int pin_all = 0) {
  PDL_ENTRY();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= (int64_t)n * B) return;
  const int node = (int)(tid / B), b = (int)(tid - (int64_t)node * B);
  const int R = 3 * B;
  const double mh = mass[node] * inv_h2;
  const int k0 = inc_ptr[node], k1 = inc_ptr[node + 1];
  const bool fx = fixed[node] != 0;
  const int pos = pos_of_node[node];
  const int cj = cand_of_node ? cand_of_node[node] : -1;
  // the <= 8 incident (element, corner) slots of a hex-mesh node: indices first, then all 24 loads in flight,
  // summed in element order (the order of the CSR, so the result is the same as a sequential loop)
  const int cnt = k1 - k0;
  int ec[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) ec[k] = k < cnt ? inc_ec[k0 + k] : 0;
  double vv[3][8];
#pragma unroll
  for (int ax = 0; ax < 3; ++ax)
#pragma unroll
    for (int k = 0; k < 8; ++k) vv[ax][k] = k < cnt ? EF[((int64_t)ec[k] * 3 + ax) * B + b] : 0.0;
  for (int ax = 0; ax < 3; ++ax) {
    const int64_t i = (3 * (int64_t)node + ax) * B + b;
    double s = 0;
    if (cnt <= 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < cnt) s += vv[ax][k];
    } else {
      for (int k = k0; k < k1; ++k) s += EF[((int64_t)inc_ec[k] * 3 + ax) * B + b];
    }
    double g = mode == 0 ? mh * (X[i] - Y[i]) + s : mh * X[i] + s;
    double wv = mode == 0 ? mh * Y[i] : 0.0;
    bool pinned = false;
    if ((ax == 2 || pin_all) && cj >= 0 && PIN) {  // pin_all: sticky contact holds all DoFs of the node
      pinned = PIN[(int64_t)cj * B + b] != 0;
      if (LAM && ax == 2) LAM[(int64_t)cj * B + b] = pinned ? g : 0.0;  // lambda = normal force
    }
    if (fx || pinned) { g = 0.0; wv = 0.0; }
    G[i] = g;
    if (W && mode == 0) W[i] = wv;
    if (RHS && pos >= 0) RHS[(int64_t)pos * R + ax * B + b] = g;
  }
}

// state (free nodes) -> permuted solve vector
__global__ void k_to_solve(const double* __restrict__ Xs, const int32_t* __restrict__ node_of_pos, int nfree, int B,
                           double* __restrict__ S) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int R = 3 * B;
  if (i >= (int64_t)nfree * R) return;
  const int64_t pos = i / R;
  const int rr = (int)(i - pos * R);
  S[i] = Xs[3 * (int64_t)node_of_pos[pos] * B + rr];
}
// permuted solve vector -> state: OUT = beta*OUT + alpha[b]*S on free nodes (fixed: OUT = beta*OUT)
// masked by ACTIVE[b] (inactive sims untouched).
__global__ void k_from_solve(const double* __restrict__ S, const int32_t* __restrict__ pos_of_node, int n, int B,
                             const double* __restrict__ alpha, double alpha_c, double beta,
                             const int32_t* __restrict__ active, double* __restrict__ OUT) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)3 * n * B) return;
  const int64_t d = i / B;
  const int b = (int)(i - d * B);
  if (active && !active[b]) return;
  const int node = (int)(d / 3), ax = (int)(d - 3 * (int64_t)node);
  const int pos = pos_of_node[node];
  const double a = alpha ? alpha[b] * alpha_c : alpha_c;
  const double base = beta == 0.0 ? 0.0 : beta * OUT[i];
  OUT[i] = pos >= 0 ? base + a * S[(int64_t)pos * 3 * B + ax * B + b] : base;
}

// ----------------------------------------------------------------- K3: supernodal solves
// One launch per ND-tree level and sweep + one reduce launch.  Work item = <= 128 k-steps
// of one 32-lane output (lane = output row forward, output column backward), stored in the stream in MMA
// fragment order; a chain = consecutive items of one output, accumulated in registers by one CTA of 4
// warps (the warps split each item's k-steps; their tiles are added in warp order at the chain's end).
// Each item is ONE TMA round (cp.async.bulk of the factor block + its right-hand-side rows, mbarrier
// transaction count).  Chains covering a whole output write it directly; the others write partial rows
// summed by the level's k_sweep_reduce in a fixed order: deterministic, no float atomics.

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
// ---- TMA bulk copies (cp.async.bulk, 1-D) completing on an mbarrier (tx-count)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// bounded: a byte-count bug becomes a trap (launch error) instead of a hung GPU.  The bound is 20 s of
// globaltimer and the barrier is re-tested after the timer read, so a CTA that was preempted or time-sliced
// between a failed try_wait and the timer read (the timer keeps running while it is off the SM) re-checks the
// completed barrier before giving up; only a transaction count that can never complete reaches the trap.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  if (mbar_try_wait(bar, parity)) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (!mbar_try_wait(bar, parity)) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 20000000000ull) {
      if (mbar_try_wait(bar, parity)) return;
      __trap();
    }
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

constexpr int kItemK = 128;  // max k-steps per item (the planner's kc)
// row stride (doubles) of the per-warp 32 x RC output tiles of k_sweep_level: RC rounded up so that a row is
// an odd number of 16-byte units (conflict-free 16-byte fragment stores)
template <int RC>
__host__ __device__ constexpr int tile_ld() { return ((RC + 1) / 2 % 2 == 1) ? ((RC + 1) / 2) * 2 : ((RC + 1) / 2 + 1) * 2; }

constexpr int kGY = 16;  // max column chunks (gridDim.y)

// CTA c takes the level's chains c, c + G, c + 2G, ... (G = gridDim.x) and walks their items through a ring
// of nbuf item buffers: while item j computes, the TMA rounds of the next nbuf-1 items are in flight.
//
// MMA = true: the item product runs on the fp64 tensor cores (mma.sync m8n8k4, DMMA): warp w takes k-groups
// of 4 steps; per group one conflict-free double2 pair of A fragments (the stream's fragment layout) and RC/8
// B fragments (right-hand-side columns), 4 x RC/8 MMAs into a 32 x RC accumulator tile held as fragments.
// MMA = false: the same product on the fp64 FMA pipe, lane (rg, cg) = 4 rows x RC/4 columns.
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
template <int RC, bool VEC, bool MMA>
__global__ void __launch_bounds__(128, RC <= 24 ? 4 : 3) k_sweep_level(SweepDev sw, int ch0, int nchains, int R,
                                                        const double* __restrict__ zc, const double* __restrict__ zi,
                                                        const int32_t* __restrict__ rows, double* __restrict__ direct,
                                                        double* __restrict__ partial, int kmax, int nbuf) {
  constexpr int CW = RC / 4;
  constexpr int NT = (RC + 7) / 8;
  constexpr int LD = tile_ld<RC>();
  extern __shared__ __align__(16) double sm[];
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int rg = lane & 7, cg = lane >> 3;
  const int y = blockIdx.y;
  const int c0 = y * RC;
  const int rcn = min(RC, R - c0);
  const int G = gridDim.x;
  const int bufd = kmax * (32 + RC);  // doubles per buffer
  __shared__ __align__(8) uint64_t mb[4];
  if (tid == 0) {
    for (int i = 0; i < nbuf; ++i) mbar_init(mb + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // per-buffer item metadata, written by the load phase one item ahead (the compute phase reads no global
  // metadata): k-steps, output, valid lanes, chain flags (bit 0 first, bit 1 last)
  __shared__ int4 meta[4];
  // one TMA round for the item with record (ra, rb) into buffer `slot`
  auto load = [&](const int4& ra, const int4& rb, int slot) {
    double* As = sm + slot * bufd;
    double* Zs = As + kmax * 32;
    const int nk = ra.y & 0xffff, nkd = ra.y >> 16, nkp = (nk + 3) & ~3;
    if (tid == 0) meta[slot] = make_int4(nk, rb.x, rb.y & 0xff, (rb.y >> 8) & 3);
    const double* Ag = sw.A + (int64_t)ra.x * 32;
    const int zr = ra.z;
    const int32_t* idx = rows + ra.w - nkd;
    if (VEC) {
      const bool whole = rcn == RC && RC == R && nkd == nk;
      if (tid == 0) {
        mbar_arrive_expect_tx(mb + slot, (unsigned)(nkp * 256 + nk * rcn * 8));
        bulk_g2s(As, Ag, (unsigned)(nkp * 256), mb + slot);
        if (whole) bulk_g2s(Zs, zc + (int64_t)zr * R, (unsigned)(nk * R * 8), mb + slot);
      }
      if (!whole)
        for (int kk = tid; kk < nk; kk += 128) {
          const bool ct = kk < nkd;
          const int row = ct ? zr + kk : __ldg(idx + kk);
          bulk_g2s(Zs + kk * RC, (ct ? zc : zi) + (int64_t)row * R + c0, (unsigned)(rcn * 8), mb + slot);
        }
    } else {
      if (tid == 0) {
        mbar_arrive_expect_tx(mb + slot, (unsigned)(nkp * 256));
        bulk_g2s(As, Ag, (unsigned)(nkp * 256), mb + slot);
      }
      for (int i = tid; i < nk * RC; i += 128) {
        const int k = i / RC, c = i - k * RC;
        const bool ct = k < nkd;
        const int row = ct ? zr + k : __ldg(idx + k);
        if (c < rcn) cp_async8(Zs + k * RC + c, (ct ? zc : zi) + (int64_t)row * R + c0 + c);
        else Zs[k * RC + c] = 0.0;
      }
      cp_async_commit();
    }
  };
  // cursors over this CTA's item sequence: (chain, item); item -1 = exhausted
  // load cursor over this CTA's items: item lit (-1 = exhausted) of chain lc, its record (ra, rb) and the first
  // item of the CTA's next chain are always prefetched one load ahead (no dependent global load between an
  // item's barrier and its TMA issue)
  int lc = blockIdx.x, lit = lc < nchains ? sw.chain[ch0 + lc] : -1;
  int nxt = lc + G < nchains ? sw.chain[ch0 + lc + G] : -1;
  int4 ra = make_int4(0, 0, 0, 0), rb = ra;
  if (lit >= 0) {
    ra = __ldg(sw.rec + 2 * lit);
    rb = __ldg(sw.rec + 2 * lit + 1);
  }
  int nload = 0;  // items loaded so far (uniform over the CTA)
  auto load_next = [&](int slot) {
    load(ra, rb, slot);
    ++nload;
    if (!((rb.y >> 9) & 1)) {
      ++lit;
    } else {
      lc += G;
      lit = nxt;
      nxt = lc + G < nchains ? sw.chain[ch0 + lc + G] : -1;
    }
    if (lit >= 0) {
      ra = __ldg(sw.rec + 2 * lit);
      rb = __ldg(sw.rec + 2 * lit + 1);
    }
  };
  for (int p = 0; p < nbuf - 1 && lit >= 0; ++p) load_next(p);
  // accumulators live across the items of a chain
  double accm[2][4][NT][2];  // MMA: fragments (two sets: even / odd k-groups)
  double accf[4][CW];        // FMA: 4 rows x CW columns
  for (int j = 0; j < nload; ++j) {
    const int slot = j % nbuf;
    if (!VEC) cp_async_wait_all();
    mbar_wait(mb + slot, (j / nbuf) & 1);
    __syncthreads();  // item j (data + meta) visible to all; every thread is past item j-1's epilogue
    const int4 md = meta[slot];
    const int nk = md.x;
    const bool first = md.w & 1, last = md.w & 2;
    if (lit >= 0) {  // refill the buffer of item j-1
      fence_proxy_async();
      load_next((j + nbuf - 1) % nbuf);
    }
    const double* As = sm + slot * bufd;
    const double* Zs = As + kmax * 32;
    double* redb = sm + slot * bufd;
    if constexpr (MMA) {
      const int g = lane >> 2, t = lane & 3;
      constexpr int NU = 1;  // one accumulator set: fewer registers, 4 CTAs/SM for RC <= 24 (measured faster than 2 sets at 3/SM)
      if (first) {
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int n = 0; n < NT; ++n) accm[u][m][n][0] = accm[u][m][n][1] = 0.0;
      }
      const int nq = (nk + 3) >> 2, per = (nq + 3) >> 2;
      const int q0 = min(nq, w * per), q1 = min(nq, q0 + per);
      const double2* A2 = reinterpret_cast<const double2*>(As);
      auto kstep = [&](int q, double (&ac)[4][NT][2]) {
        const double2 a01 = A2[(q * 2) * 32 + lane];
        const double2 a23 = A2[(q * 2 + 1) * 32 + lane];
        const int k = 4 * q + t;
        double b[NT];
#pragma unroll
        for (int n = 0; n < NT; ++n) {  // padded k-steps read stale rows: their (zero) factor needs b = 0
          const int col = 8 * n + g;
          b[n] = (k < nk && col < RC) ? Zs[k * RC + col] : 0.0;
        }
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          dmma_8x8x4(ac[0][n][0], ac[0][n][1], a01.x, b[n]);
          dmma_8x8x4(ac[1][n][0], ac[1][n][1], a01.y, b[n]);
          dmma_8x8x4(ac[2][n][0], ac[2][n][1], a23.x, b[n]);
          dmma_8x8x4(ac[3][n][0], ac[3][n][1], a23.y, b[n]);
        }
      };
      int q = q0;
      if (NU == 2) {
        for (; q + 1 < q1; q += 2) {
          kstep(q, accm[0]);
          kstep(q + 1, accm[NU - 1]);
        }
      } else {
#pragma unroll 2
        for (; q + 1 < q1; ++q) kstep(q, accm[0]);
      }
      if (q < q1) kstep(q, accm[0]);
      if (last) {
        __syncthreads();  // all warps done with this buffer: reuse it for the 4 warp tiles
        // fragment (m, n): rows 4g + m, columns 8n + 2t + {0, 1}: one 16-byte store each; rows padded to LD
        // doubles (an odd number of 16-byte units: the 8 lanes of a store phase hit 8 distinct bank groups)
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            const int col = 8 * n + 2 * t;
            if (col < RC)
              *reinterpret_cast<double2*>(redb + w * 32 * LD + (4 * g + m) * LD + col) =
                  NU == 2 ? make_double2(accm[0][m][n][0] + accm[NU - 1][m][n][0],
                                         accm[0][m][n][1] + accm[NU - 1][m][n][1])
                          : make_double2(accm[0][m][n][0], accm[0][m][n][1]);
          }
      }
    } else {
      if (first) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < CW; ++c) accf[r][c] = 0.0;
      }
      const int per = (nk + 3) >> 2;
      const int k0 = min(nk, w * per), k1 = min(nk, k0 + per);
#pragma unroll 2
      for (int k = k0; k < k1; ++k) {
        // fragment layout (plan.h sweep_frag_pos): rows 4rg..4rg+3 of step k are two double2
        const double2 a01 = *reinterpret_cast<const double2*>(As + (((k >> 2) * 2) * 32 + 4 * rg + (k & 3)) * 2);
        const double2 a23 = *reinterpret_cast<const double2*>(As + (((k >> 2) * 2 + 1) * 32 + 4 * rg + (k & 3)) * 2);
        const double av[4] = {a01.x, a01.y, a23.x, a23.y};
        double zv[CW];
#pragma unroll
        for (int c = 0; c < CW; ++c) zv[c] = Zs[k * RC + cg * CW + c];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < CW; ++c) accf[r][c] = fma(av[r], zv[c], accf[r][c]);
      }
      if (last) {
        __syncthreads();  // all warps done with this buffer: reuse it for the 4 warp tiles
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < CW; ++c) redb[w * 32 * LD + (4 * rg + r) * LD + cg * CW + c] = accf[r][c];
      }
    }
    if (last) {
      __syncthreads();
      // ---- output rows: fixed-order sum of the 4 warp tiles, coalesced over columns
      const int out = md.y;
      const int nv = md.z;
      double* __restrict__ dst =
          out >= 0 ? direct + (int64_t)out * R + c0 : partial + (int64_t)(-out - 1) * 32 * R + c0;
      if constexpr (RC % 2 == 0) {
        // column pairs: thread = (row slot, pair); 128-bit tile loads, 128-bit stores when the row stride allows
        constexpr int CP = RC / 2, RPP = 128 / CP;  // pairs per row, rows per pass
        const int cp = tid % CP, rs = tid / CP, c = 2 * cp;
        const bool st2 = (R & 1) == 0;
        if (rs < RPP)
          for (int r = rs; r < nv; r += RPP) {
            const double* rb = redb + r * LD + c;
            const double2 t0 = *reinterpret_cast<const double2*>(rb);
            const double2 t1 = *reinterpret_cast<const double2*>(rb + 32 * LD);
            const double2 t2 = *reinterpret_cast<const double2*>(rb + 64 * LD);
            const double2 t3 = *reinterpret_cast<const double2*>(rb + 96 * LD);
            const double v0 = ((t0.x + t1.x) + t2.x) + t3.x, v1 = ((t0.y + t1.y) + t2.y) + t3.y;
            double* d = dst + (int64_t)r * R + c;
            if (c + 1 < rcn) {
              if (st2) {
                *reinterpret_cast<double2*>(d) = make_double2(v0, v1);
              } else {
                d[0] = v0;
                d[1] = v1;
              }
            } else if (c < rcn) {
              d[0] = v0;
            }
          }
      } else {
        for (int e = tid; e < nv * RC; e += 128) {
          const int r = e / RC, c = e - r * RC;
          const double* rb = redb + r * LD + c;
          if (c < rcn) dst[(int64_t)r * R + c] = ((rb[0] + rb[32 * LD]) + rb[64 * LD]) + rb[96 * LD];
        }
      }
      // the tile writes (generic proxy) precede the TMA refill of this buffer (async proxy) after the next barrier
      fence_proxy_async();
    }
    // (the buffer is refilled after the next item's barrier: no barrier needed here)
  }
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

__global__ void k_sweep_reduce(SweepDev sw, int r0, int ntarget, int R, const double* __restrict__ partial,
                               double* __restrict__ dst_assign, double* __restrict__ dst_sub) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= (int64_t)ntarget * R) return;
  const int t = r0 + (int)(g / R), c = (int)(g % R);
  // all independent loads first (target row, mode, source range, the z value), then the fixed-order sum
  const int q0 = sw.red_ptr[t], q1 = sw.red_ptr[t + 1], mode = sw.red_mode[t];
  const int64_t o = (int64_t)sw.red_row[t] * R + c;
  const double zo = mode == 0 ? 0.0 : dst_sub[o];
  // sources in batches of 4: indices, then the 4 partial loads in flight, then the in-order sum
  double acc = 0;
  int q = q0;
  for (; q + 4 <= q1; q += 4) {
    const int s0 = sw.red_src[q], s1 = sw.red_src[q + 1], s2 = sw.red_src[q + 2], s3 = sw.red_src[q + 3];
    const double p0 = partial[(int64_t)s0 * R + c], p1 = partial[(int64_t)s1 * R + c];
    const double p2 = partial[(int64_t)s2 * R + c], p3 = partial[(int64_t)s3 * R + c];
    acc += p0;
    acc += p1;
    acc += p2;
    acc += p3;
  }
  for (; q < q1; ++q) acc += partial[(int64_t)sw.red_src[q] * R + c];
  if (mode == 0) dst_assign[o] = acc;
  else dst_sub[o] = zo - acc;
}

// ----------------------------------------------------------------- K3 v4: warp ranges
// One launch per level and sweep.  Warp w of the level streams the contiguous k-group range [wg[w], wg[w+1]) (or,
// with vpw > 1 when several column chunks share the SMs, the vpw consecutive ranges [wg[w], wg[w+vpw])) of
// the factor stream through its own ring of kStages stages (no CTA barrier anywhere): a stage is 4 k-groups
// (16 k-steps): the 4 KB factor block arrives by one cp.async.bulk (TMA) on the stage's mbarrier, the 16
// right-hand-side rows (k-step sources, krow) by cp.async into padded rows; lane 0 issues stage j + kStages - 1
// before the warp computes stage j.  Per k-group 4 x NT DMMA (m8n8k4 fp64) into a 32 x 8NT tile held in
// registers; at the end of each piece the tile is stored to its direct rows or to its partial slot.  The
// level's reduce (k_sweep_reduce4) then adds partial slots into their targets in piece order.
constexpr int kStages = 3;         // ring depth per warp
constexpr int kWarpsK3 = 8;        // warps per CTA
template <int NT>
__host__ __device__ constexpr int rhs_ld() { return NT == 1 ? 8 : 28; }  // padded RHS row (doubles): conflict-free B reads
template <int NT>
__host__ __device__ constexpr int stage_doubles() { return 4 * 128 + 16 * rhs_ld<NT>(); }

// Piece metadata of a warp's range held one piece per lane (lane i: piece pb + i): end k-group, output, valid
// rows.  A piece change is a shuffle instead of dependent global loads on the critical path (reloaded for the
// next 32 pieces when a range has more).
__device__ __forceinline__ void piece_fetch(const Sweep4Dev& sw, int pb, int pend, int lane, int& pe_l, int& po_l,
                                            int& pn_l) {
  const int q = pb + lane;
  pe_l = q < pend ? sw.pstart[q] + sw.pkg[q] : 0;
  po_l = q < pend ? sw.pout[q] : 0;
  pn_l = q < pend ? sw.pnv[q] : 0;
}

template <int NT, bool VEC>
__global__ void __launch_bounds__(32 * kWarpsK3, 1) k_sweep_warp(Sweep4Dev sw, int w0, int nwarps, int vpw, int R,
                                                                const double* __restrict__ srcA,
                                                                const double* __restrict__ srcB,
                                                                double* __restrict__ direct,
                                                                double* __restrict__ partial) {
  constexpr int RC = 8 * NT, LD = rhs_ld<NT>(), SD = stage_doubles<NT>();
  // the next launch (reduce / next level) may be scheduled at once; its CTAs block in griddepcontrol.wait until
  // this grid has completed and its writes are visible, so signalling at entry only hides launch latency
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  extern __shared__ __align__(128) double smem4[];
  __shared__ __align__(8) uint64_t bars[kWarpsK3][kStages];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int c0 = blockIdx.y * RC, rcn = min(RC, R - c0);
  double* ring = smem4 + (size_t)wl * kStages * SD;
  // RHS areas start finite (padding k-steps multiply stale rows by an exact zero factor entry)
  for (int i = lane; i < kStages * 16 * LD; i += 32) ring[(i / (16 * LD)) * SD + 512 + i % (16 * LD)] = 0.0;
  if (lane == 0)
    for (int i = 0; i < kStages; ++i) mbar_init(&bars[wl][i], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncwarp();
  const int w = (blockIdx.x * kWarpsK3 + wl) * vpw;  // first of this warp's vpw consecutive ranges
  if (w >= nwarps) {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    return;
  }
  // Everything but the right-hand side is static plan data: the warp range, its first piece, the k-step rows
  // and the factor blocks of the first kStages - 1 stages are fetched BEFORE griddepcontrol.wait, overlapping
  // the previous launch (its tail / the previous level's reduce); only the RHS copies wait for it.
  const int w1 = min(w + vpw, nwarps);
  const int g0 = sw.wg[w0 + w], g1 = sw.wg[w0 + w1];
  const int nst = (g1 - g0 + 3) >> 2;
  // k-step source rows of stage j (lane i < 16: k-step i)
  auto krow_of = [&](int j) {
    const int gs = g0 + 4 * j;
    return (j < nst && lane < 4 * min(4, g1 - gs)) ? __ldg(sw.krow + 4 * (int64_t)gs + lane) : -1;
  };
  // factor block of stage j by TMA (lane 0) on the stage's mbarrier
  auto issue_factor = [&](int j) {
    if (j >= nst || lane != 0) return;
    const int slot = j % kStages;
    const int gs = g0 + 4 * j, nkg = min(4, g1 - gs);
    mbar_arrive_expect_tx(&bars[wl][slot], (unsigned)(nkg * 1024));
    bulk_g2s(ring + slot * SD, sw.A + (int64_t)gs * 128, (unsigned)(nkg * 1024), &bars[wl][slot]);
  };
  // RHS rows of stage j by cp.async (16 rows x rcn columns over the lanes), one commit group per stage
  auto issue_rhs = [&](int j, int kr) {
    if (j < nst) {
      double* zs = ring + (j % kStages) * SD + 512;
      if (VEC) {  // 16-byte copies: (row, column pair) over the lanes
        constexpr int CP = RC / 2;  // (16 * CP and 16 * RC are multiples of 32: every lane runs the same trips)
        for (int e = lane; e < 16 * CP; e += 32) {
          const int j2 = e / CP, c = 2 * (e - j2 * CP);
          const int v = __shfl_sync(0xffffffffu, kr, j2 & 15);
          if (v != -1 && c < rcn) {
            const double* src = v >= 0 ? srcA + (int64_t)v * R : srcB + (int64_t)(-2 - v) * R;
            cp_async16(zs + j2 * LD + c, src + c0 + c);
          }
        }
      } else {
        for (int e = lane; e < 16 * RC; e += 32) {
          const int j2 = e / RC, c = e - j2 * RC;
          const int v = __shfl_sync(0xffffffffu, kr, j2 & 15);
          if (v != -1 && c < rcn) {
            const double* src = v >= 0 ? srcA + (int64_t)v * R : srcB + (int64_t)(-2 - v) * R;
            cp_async8(zs + j2 * LD + c, src + c0 + c);
          }
        }
      }
    }
    cp_async_commit();
  };
  int krs[kStages - 1];
#pragma unroll
  for (int j = 0; j < kStages - 1; ++j) {
    issue_factor(j);
    krs[j] = krow_of(j);
  }
  int kr_next = krow_of(kStages - 1);
  int pb = sw.wpiece[w0 + w], pi = 0;
  const int pend = sw.wpiece[w0 + w1];
  int pe_l, po_l, pn_l;
  piece_fetch(sw, pb, pend, lane, pe_l, po_l, pn_l);
  int pe = __shfl_sync(0xffffffffu, pe_l, 0);  // end (global k-group) of the current piece
  int pout = __shfl_sync(0xffffffffu, po_l, 0), pnv = __shfl_sync(0xffffffffu, pn_l, 0);
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
#pragma unroll
  for (int j = 0; j < kStages - 1; ++j) issue_rhs(j, krs[j]);
  double acc[4][NT][2];
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
  for (int j = 0; j < nst; ++j) {
    __syncwarp();
    fence_proxy_async();
    issue_factor(j + kStages - 1);  // refills the slot of stage j - 1 (every lane is past it)
    issue_rhs(j + kStages - 1, kr_next);
    kr_next = krow_of(j + kStages);
    const int slot = j % kStages;
    cp_async_wait_group<kStages - 1>();
    mbar_wait(&bars[wl][slot], (j / kStages) & 1);
    __syncwarp();  // every lane's RHS copies of this stage are visible to the warp
    const double2* As = reinterpret_cast<const double2*>(ring + slot * SD);
    const double* Zs = ring + slot * SD + 512;
    const int gs = g0 + 4 * j, nkg = min(4, g1 - gs);
    for (int q = 0; q < nkg; ++q) {
      const double2 a01 = As[(q * 2) * 32 + lane], a23 = As[(q * 2 + 1) * 32 + lane];
      double b[NT];
#pragma unroll
      for (int n = 0; n < NT; ++n) b[n] = Zs[(4 * q + t) * LD + 8 * n + g];
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        dmma_8x8x4(acc[0][n][0], acc[0][n][1], a01.x, b[n]);
        dmma_8x8x4(acc[1][n][0], acc[1][n][1], a01.y, b[n]);
        dmma_8x8x4(acc[2][n][0], acc[2][n][1], a23.x, b[n]);
        dmma_8x8x4(acc[3][n][0], acc[3][n][1], a23.y, b[n]);
      }
      if (gs + q + 1 == pe) {  // end of the piece: store the tile (rows 4g + m, columns 8n + 2t + {0, 1})
        double* dst = pout >= 0 ? direct + (int64_t)pout * R : partial + (int64_t)(-1 - pout) * 32 * R;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int row = 4 * g + m;
          if (row < pnv) {
#pragma unroll
            for (int n = 0; n < NT; ++n) {
              const int c = 8 * n + 2 * t;
              double* d = dst + (int64_t)row * R + c0 + c;
              if (VEC && c + 1 < rcn) {
                *reinterpret_cast<double2*>(d) = make_double2(acc[m][n][0], acc[m][n][1]);
              } else {
                if (c < rcn) d[0] = acc[m][n][0];
                if (c + 1 < rcn) d[1] = acc[m][n][1];
              }
            }
          }
#pragma unroll
          for (int n = 0; n < NT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
        }
        if (gs + q + 1 < g1) {
          if (++pi == 32) {
            pb += 32;
            pi = 0;
            piece_fetch(sw, pb, pend, lane, pe_l, po_l, pn_l);
          }
          pe = __shfl_sync(0xffffffffu, pe_l, pi);
          pout = __shfl_sync(0xffffffffu, po_l, pi);
          pnv = __shfl_sync(0xffffffffu, pn_l, pi);
        }
      }
    }
  }
  cp_async_wait_all();
}

// Level reduce of K3 v4: target t (row, mode) = fixed-order sum of its partial rows; mode 0: dst_assign[row] = sum,
// mode 1: dst_sub[row] -= sum.  NB source loads in flight per batch (8: c5 A^-1 464 -> 461 us against 4; same order,
// bitwise-identical results).
template <int NB>
__global__ void k_sweep_reduce4(Sweep4Dev sw, int r0, int ntarget, int R, const double* __restrict__ partial,
                                double* __restrict__ dst_assign, double* __restrict__ dst_sub) {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const int64_t gi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool live = gi < (int64_t)ntarget * R;
  // the target's static metadata and its first NB source indices before griddepcontrol.wait
  const int t = live ? r0 + (int)(gi / R) : r0, c = live ? (int)(gi % R) : 0;
  const int q0 = sw.red_ptr[t], q1 = sw.red_ptr[t + 1], mode = sw.red_mode[t];
  const int64_t o = (int64_t)sw.red_row[t] * R + c;
  int sq[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) sq[k] = q0 + k < q1 ? sw.red_src[q0 + k] : 0;
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (!live) return;
  const double zo = mode == 0 ? 0.0 : dst_sub[o];
  double acc = 0;
  {
    double pv[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) pv[k] = q0 + k < q1 ? partial[(int64_t)sq[k] * R + c] : 0.0;
#pragma unroll
    for (int k = 0; k < NB; ++k)
      if (q0 + k < q1) acc += pv[k];
  }
  int q = q0 + NB;
  for (; q + NB <= q1; q += NB) {  // NB loads in flight, then the in-order sum
    int sk[NB];
    double p[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) sk[k] = sw.red_src[q + k];
#pragma unroll
    for (int k = 0; k < NB; ++k) p[k] = partial[(int64_t)sk[k] * R + c];
#pragma unroll
    for (int k = 0; k < NB; ++k) acc += p[k];
  }
  for (; q < q1; ++q) acc += partial[(int64_t)sw.red_src[q] * R + c];
  if (mode == 0) dst_assign[o] = acc;
  else dst_sub[o] = zo - acc;
}
template __global__ void k_sweep_reduce4<8>(Sweep4Dev, int, int, int, const double*, double*, double*);

// ----------------------------------------------------------------- K5: contact
// The candidate nodes V are ordered last: their rows form the root supernode, whose assembled
// front is the Schur complement S = S_CC of A_s onto V.  For the z-column of sim b with pinned
// set a_b (x_a = xbar = 0, P:380-383 eq:dirichlet/eq:complement, reading §2.9-2.10) the root
// block of the constrained solve is x_f = (S_ff)^{-1} r_f, x_a = 0, where r = z[J_root] after
// the forward sweep; every other level is unchanged.  Q_b = (S_ff)^{-1} is rebuilt (gather +
// blocked Gauss-Jordan) only when the active set changes.
constexpr int kGJ = 32;  // Gauss-Jordan pivot block

// flist[b][0..k) = root-local indices of UNPINNED candidates (ascending), fpos[b][loc] = index or -1,
// kcount[b] = k.  One CTA per selected sim; deterministic block scan.
__global__ void __launch_bounds__(1024) k_contact_flist(const uint8_t* __restrict__ PIN, const int32_t* __restrict__ cand_of_loc,
                                                        int c, int B, const int32_t* __restrict__ sel,
                                                        int32_t* __restrict__ flist, int32_t* __restrict__ fpos,
                                                        int32_t* __restrict__ kcount) {
  PDL_ENTRY();
  const int b = blockIdx.x;
  if (sel && !sel[b]) return;
  __shared__ int32_t warp_tot[32];
  __shared__ int32_t base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int l0 = 0; l0 < c; l0 += blockDim.x) {
    const int loc = l0 + threadIdx.x;
    const int fr = (loc < c && !PIN[(int64_t)cand_of_loc[loc] * B + b]) ? 1 : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, fr);
    const int pre = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) warp_tot[wid] = __popc(bal);
    __syncthreads();
    int off = base;
    for (int w = 0; w < wid; ++w) off += warp_tot[w];
    if (loc < c) {
      const int idx = off + pre;
      fpos[(int64_t)b * c + loc] = fr ? idx : -1;
      if (fr) flist[(int64_t)b * c + idx] = loc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += warp_tot[w];
      base += t;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) kcount[b] = base;
}

// Q_b[i][j] = S[flist_i][flist_j]   (leading dimension c)
__global__ void k_contact_gather_S(const double* __restrict__ S, int c, const int32_t* __restrict__ sel,
                                   const int32_t* __restrict__ flist, const int32_t* __restrict__ kcount,
                                   double* __restrict__ Q) {
  PDL_ENTRY();
  const int b = blockIdx.z;
  if (sel && !sel[b]) return;
  const int k = kcount[b];
  const int i = blockIdx.y * 8 + threadIdx.y, j = blockIdx.x * 32 + threadIdx.x;
  if (i >= k || j >= k) return;
  const int32_t* fl = flist + (int64_t)b * c;
  Q[((int64_t)b * c + i) * c + j] = S[(int64_t)fl[i] * c + fl[j]];
}

// Block Gauss-Jordan step kb, part 1: Pinv = (Q_KK)^{-1} (SPD, in shared memory, no pivoting),
// C = Q[:, K] copied to Cb (k x kGJ), M = C Pinv into Mb, Rw = Q[K, :] copied to Rb (kGJ x k).
__global__ void __launch_bounds__(256) k_gj_pivot(double* __restrict__ Q, int c, int kb, const int32_t* __restrict__ sel,
                                                  const int32_t* __restrict__ kcount, double* __restrict__ PI) {
  PDL_ENTRY();
  const int b = blockIdx.x;
  if (sel && !sel[b]) return;
  const int k = kcount[b];
  const int k0 = kb * kGJ;
  if (k0 >= k) return;
  const int nbk = min(kGJ, k - k0);
  __shared__ double P[kGJ][kGJ + 1];
  const double* Qb = Q + (int64_t)b * c * c;
  for (int idx = threadIdx.x; idx < kGJ * kGJ; idx += blockDim.x) {
    const int i = idx / kGJ, j = idx % kGJ;
    P[i][j] = (i < nbk && j < nbk) ? Qb[(int64_t)(k0 + i) * c + k0 + j] : (i == j ? 1.0 : 0.0);
  }
  __syncthreads();
  // in-place Gauss-Jordan inversion of the kGJ x kGJ block (padding = identity)
  for (int p = 0; p < kGJ; ++p) {
    const double piv = P[p][p];
    double rowp = 0, colp = 0;
    const int i = threadIdx.x / kGJ, j = threadIdx.x % kGJ;  // 256 threads: 8 rows per pass
    __syncthreads();
    // snapshot of row p and column p
    __shared__ double rp[kGJ], cp[kGJ];
    if (threadIdx.x < kGJ) { rp[threadIdx.x] = P[p][threadIdx.x]; cp[threadIdx.x] = P[threadIdx.x][p]; }
    __syncthreads();
    const double ipiv = 1.0 / piv;
    for (int ii = i; ii < kGJ; ii += blockDim.x / kGJ) {
      double v;
      if (ii == p && j == p) v = ipiv;
      else if (ii == p) v = rp[j] * ipiv;
      else if (j == p) v = -cp[ii] * ipiv;
      else v = P[ii][j] - cp[ii] * rp[j] * ipiv;
      P[ii][j] = v;
    }
    (void)rowp; (void)colp;
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < kGJ * kGJ; idx += blockDim.x)
    PI[(int64_t)b * kGJ * kGJ + idx] = P[idx / kGJ][idx % kGJ];
}

// part 2 (grid: row tiles x sims): Cb[i][t] = Q[i][k0+t], Mb[i][:] = Cb[i] Pinv, Rb[t][i] = Q[k0+t][i]
__global__ void __launch_bounds__(256) k_gj_panel(const double* __restrict__ Q, int c, int kb, const int32_t* __restrict__ sel,
                                                  const int32_t* __restrict__ kcount, const double* __restrict__ PI,
                                                  double* __restrict__ Cb, double* __restrict__ Mb, double* __restrict__ Rb) {
  PDL_ENTRY();
  const int b = blockIdx.y;
  if (sel && !sel[b]) return;
  const int k = kcount[b];
  const int k0 = kb * kGJ;
  if (k0 >= k) return;
  const int nbk = min(kGJ, k - k0);
  __shared__ double Pi[kGJ][kGJ + 1];
  __shared__ double Ct[8][kGJ];
  for (int idx = threadIdx.x; idx < kGJ * kGJ; idx += blockDim.x) Pi[idx / kGJ][idx % kGJ] = PI[(int64_t)b * kGJ * kGJ + idx];
  const double* Qb = Q + (int64_t)b * c * c;
  const int t = threadIdx.x % kGJ, r = threadIdx.x / kGJ;  // 8 rows x 32 cols per pass
  for (int i0 = blockIdx.x * 64; i0 < min(k, (int)(blockIdx.x + 1) * 64); i0 += 8) {
    const int i = i0 + r;
    __syncthreads();
    const double cv = (i < k && t < nbk) ? Qb[(int64_t)i * c + k0 + t] : 0.0;
    Ct[r][t] = cv;
    if (i < k) {
      Cb[((int64_t)b * c + i) * kGJ + t] = cv;
      Rb[((int64_t)b * kGJ + t) * c + i] = t < nbk ? Qb[(int64_t)(k0 + t) * c + i] : 0.0;
    }
    __syncthreads();
    if (i < k) {
      double acc = 0;
#pragma unroll 8
      for (int u = 0; u < kGJ; ++u) acc = fma(Ct[r][u], Pi[u][t], acc);
      Mb[((int64_t)b * c + i) * kGJ + t] = acc;
    }
  }
}

// part 3 (grid: 32x32 tiles of Q x sims):  Q_KK = Pinv, Q_KO = Pinv Rw, Q_OK = -M, Q_OO -= M Rw.
__global__ void __launch_bounds__(256) k_gj_update(double* __restrict__ Q, int c, int kb, const int32_t* __restrict__ sel,
                                                   const int32_t* __restrict__ kcount, const double* __restrict__ PI,
                                                   const double* __restrict__ Mb, const double* __restrict__ Rb) {
  PDL_ENTRY();
  const int b = blockIdx.z;
  if (sel && !sel[b]) return;
  const int k = kcount[b];
  const int k0 = kb * kGJ;
  if (k0 >= k) return;
  const int nbk = min(kGJ, k - k0);
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  if (i0 >= k || j0 >= k) return;
  __shared__ double Ms[32][kGJ + 1];   // M rows i0.. (or Pinv rows when the tile is in the pivot rows)
  __shared__ double Rs[kGJ][32 + 1];   // Rw columns j0..
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // 32 x 8
  const bool iK = (i0 == k0), jK = (j0 == k0);             // tiles align with pivot blocks (kGJ = 32)
  for (int idx = threadIdx.x; idx < 32 * kGJ; idx += blockDim.x) {
    const int a = idx / kGJ, u = idx % kGJ;
    const int i = i0 + a, j = j0 + a;
    Ms[a][u] = iK ? PI[(int64_t)b * kGJ * kGJ + a * kGJ + u] : (i < k ? Mb[((int64_t)b * c + i) * kGJ + u] : 0.0);
    Rs[u][a] = j < k ? Rb[((int64_t)b * kGJ + u) * c + j] : 0.0;
  }
  __syncthreads();
  double* Qb = Q + (int64_t)b * c * c;
  for (int a = ty; a < 32; a += 8) {
    const int i = i0 + a, j = j0 + tx;
    if (i >= k || j >= k) continue;
    double v;
    if (iK && jK) {
      v = (a < nbk && tx < nbk) ? Ms[a][tx] : 0.0;
    } else if (iK) {        // Q_KO = Pinv Rw
      double acc = 0;
#pragma unroll 8
      for (int u = 0; u < kGJ; ++u) acc = fma(Ms[a][u], Rs[u][tx], acc);
      v = acc;
    } else if (jK) {        // Q_OK = -M
      v = -Ms[a][tx];
    } else {                // Q_OO -= M Rw
      double acc = 0;
#pragma unroll 8
      for (int u = 0; u < nbk; ++u) acc = fma(Ms[a][u], Rs[u][tx], acc);
      v = Qb[(int64_t)i * c + j] - acc;
    }
    Qb[(int64_t)i * c + j] = v;
  }
}

// Constrained root block of the solve for the z-columns (col = 2B + b) of sims with pins:
// x_loc = 0 if pinned, else sum_l Q_b[fpos(loc)][l] r[flist_l].  One warp per output row,
// lanes stride the dot product, fixed-order shuffle reduction (deterministic).
__global__ void __launch_bounds__(256) k_contact_fix(const double* __restrict__ Rsave, int c, int R, int B,
                                                     const int32_t* __restrict__ kcount, const int32_t* __restrict__ flist,
                                                     const int32_t* __restrict__ fpos, const double* __restrict__ Q,
                                                     double* __restrict__ Xroot) {
  PDL_ENTRY();
  // blockIdx.y = a*B + b over the pinned axes (frictionless: only z; sticky: x, y, z -> gridDim.y = 3B)
  const int b = blockIdx.y % B;
  const int ax = gridDim.y == (unsigned)B ? 2 : (int)(blockIdx.y / B);
  const int k = kcount[b];
  if (k == c) return;  // no pins: the unconstrained root solve stands
  const int lane = threadIdx.x & 31;
  const int loc = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (loc >= c) return;
  const int col = ax * B + b;
  const int fi = fpos[(int64_t)b * c + loc];
  double acc = 0;
  if (fi >= 0) {
    const double* Qr = Q + ((int64_t)b * c + fi) * c;
    const int32_t* fl = flist + (int64_t)b * c;
    for (int l = lane; l < k; l += 32) acc = fma(Qr[l], Rsave[(int64_t)fl[l] * R + col], acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  }
  if (lane == 0) Xroot[(int64_t)loc * R + col] = acc;
}

// x^0 of an outer iteration (Alg. 1): X = Xp for outer-active sims, pinned z DoFs at the plane.
// warm = 1: start from the previous outer iteration's converged x instead (the inner
// solve's converged point does not depend on its start; only the iteration count does).
__global__ void k_contact_restart(double* __restrict__ X, const double* __restrict__ Xp, int n, int B,
                                  const int32_t* __restrict__ cand_of_node, const uint8_t* __restrict__ PIN,
                                  const int32_t* __restrict__ oact, int warm, int pin_all = 0) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)3 * n * B) return;
  const int64_t d = i / B;
  const int b = (int)(i - d * B);
  if (!oact[b]) return;
  const int node = (int)(d / 3), ax = (int)(d - 3 * (int64_t)node);
  const int cj = cand_of_node[node];
  const bool pinned = (ax == 2 || pin_all) && cj >= 0 && PIN[(int64_t)cj * B + b];
  // frictionless: the normal DoF on the plane z = 0; sticky: every DoF at x_i
  X[i] = pinned ? (pin_all ? Xp[i] : 0.0) : (warm ? X[i] : Xp[i]);
}

// Predictor (Alg. 1, reading §2.11): active' = (phi < -eps_phi) or (lambda > 0), phi = z
// (plane z = 0), lambda = (A x - d)_j for pinned j (LAM, from the gather), 0 otherwise.
__global__ void k_contact_predict(const double* __restrict__ X, const double* __restrict__ LAM,
                                  const int32_t* __restrict__ cand_node, int c, int B, double eps_phi,
                                  const uint8_t* __restrict__ PIN, const int32_t* __restrict__ oact,
                                  uint8_t* __restrict__ NEWPIN, int32_t* __restrict__ changed) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)c * B) return;
  const int j = (int)(i / B), b = (int)(i - (int64_t)j * B);
  if (!oact[b]) return;
  const double phi = X[(3 * (int64_t)cand_node[j] + 2) * B + b];
  const double lam = PIN[i] ? LAM[i] : 0.0;
  const uint8_t nw = (phi < -eps_phi || lam > 0.0) ? 1 : 0;
  NEWPIN[i] = nw;
  if (nw != PIN[i]) changed[b] = 1;  // integer flag, value independent of thread order
}

// Outer-loop bookkeeping: continue with the new set if it changed and the cap is not reached.
__global__ void k_contact_outer(const int32_t* __restrict__ oact, const int32_t* __restrict__ changed,
                                const uint8_t* __restrict__ NEWPIN, uint8_t* __restrict__ PIN, int c, int B,
                                int outer, int max_outer, int32_t* __restrict__ onext,
                                int32_t* __restrict__ outer_out, int32_t* __restrict__ flag_out) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)c * B) return;
  const int j = (int)(i / B), b = (int)(i - (int64_t)j * B);
  if (!oact[b]) {
    if (j == 0) onext[b] = 0;
    return;
  }
  const bool go = changed[b] && outer < max_outer;
  if (go) PIN[i] = NEWPIN[i];
  if (j == 0) {
    onext[b] = go ? 1 : 0;
    outer_out[b] = outer;
    if (changed[b] && !go) flag_out[b] = 1;  // hit the outer cap
  }
}

// ----------------------------------------------------------------- per-sim reductions
// Per-sim sums over a state-layout vector (element d*B + b): chunk c = DoFs [c*kRedC, (c+1)*kRedC); in a chunk,
// thread j < kRedJ of sim b adds DoFs c*kRedC + j, + kRedJ, ... in ascending order, then the kRedJ thread sums are
// added in j order -> partial[(p*nchunk + c)*B + b]; k_dot_final adds the chunks.  Every constant here is
// independent of B, so a sim's sum — and with it every iterate — is bitwise the same whatever batch it runs in
// (a sharded batch reproduces the single-GPU run exactly).  Blocks: kRedJ x min(B, kRedS) threads,
// sims fastest (coalesced over b), grid.y (or .z) over groups of kRedS sims.
constexpr int kRedC = 128;
constexpr int kRedJ = 8;
constexpr int kRedS = 32;

struct RedLane {
  int b, j, bl;
  bool ok;
};
__device__ __forceinline__ RedLane red_lane(int B, int group) {
  const int Bb = blockDim.x / kRedJ;
  RedLane r;
  r.bl = threadIdx.x % Bb;
  r.j = threadIdx.x / Bb;
  r.b = group * kRedS + r.bl;
  r.ok = r.b < B;
  return r;
}
// red[p][j][bl] holds the thread sums; thread j == 0 adds them in j order and stores the chunk partial
__device__ __forceinline__ void red_store(double (*red)[kRedJ][kRedS], int np, const RedLane& r, int B, int nchunk,
                                          int c, double* __restrict__ partial) {
  __syncthreads();
  if (r.j == 0 && r.ok)
    for (int p = 0; p < np; ++p) {
      double t = red[p][0][r.bl];
#pragma unroll
      for (int jj = 1; jj < kRedJ; ++jj) t += red[p][jj][r.bl];
      partial[((int64_t)p * nchunk + c) * B + r.b] = t;
    }
}
// partial[c][b] = sum over chunk c of u*v (up to 3 pairs; v = null means 1)
__global__ void k_dot_partial(DotArgs da, int64_t len, int B, double* __restrict__ partial) {
  PDL_ENTRY();
  __shared__ double red[3][kRedJ][kRedS];
  const RedLane r = red_lane(B, blockIdx.y);
  const int c = blockIdx.x;
  double acc[3] = {0, 0, 0};
  if (r.ok) {
    const int64_t d1 = min(len, (int64_t)(c + 1) * kRedC);
    int64_t d = (int64_t)c * kRedC + r.j;
    for (; d + kRedJ < d1; d += 2 * kRedJ) {  // two DoFs per trip: loads first, then the in-order fma chain
      const int64_t i0 = d * B + r.b, i1 = (d + kRedJ) * B + r.b;
      double u0[3], v0[3], u1[3], v1[3];
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        u0[p] = p < da.npairs ? da.u[p][i0] : 0.0;
        u1[p] = p < da.npairs ? da.u[p][i1] : 0.0;
        v0[p] = (p < da.npairs && da.v[p]) ? da.v[p][i0] : 1.0;
        v1[p] = (p < da.npairs && da.v[p]) ? da.v[p][i1] : 1.0;
      }
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        acc[p] = fma(u0[p], v0[p], acc[p]);
        acc[p] = fma(u1[p], v1[p], acc[p]);
      }
    }
    for (; d < d1; d += kRedJ) {
      const int64_t i = d * B + r.b;
#pragma unroll
      for (int p = 0; p < 3; ++p)
        if (p < da.npairs) acc[p] = fma(da.u[p][i], da.v[p] ? da.v[p][i] : 1.0, acc[p]);
    }
  }
#pragma unroll
  for (int p = 0; p < 3; ++p) red[p][r.j][r.bl] = acc[p];
  red_store(red, da.npairs, r, B, gridDim.x, c, partial);
}
// one warp per (pair, sim): lane l sums chunks l, l+32, ... in order, then a fixed xor tree (deterministic)
// one 128-thread block per (pair, sim): thread t sums chunks t, t+128, ... with 4 independent accumulators (loads
// in flight together), then a fixed xor tree per warp and the 4 warp sums in warp order (deterministic)
__global__ void __launch_bounds__(128) k_dot_final(const double* __restrict__ partial, int nchunk, int B, int npairs,
                                                   double* __restrict__ out, int accumulate = 0) {
  PDL_ENTRY();
  const int i = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (i >= npairs * B) return;
  const int p = i / B, b = i - p * B;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  const double* pp = partial + (int64_t)p * nchunk * B + b;
  int c = tid;
  for (; c + 384 < nchunk; c += 512) {
    s0 += pp[(int64_t)c * B];
    s1 += pp[(int64_t)(c + 128) * B];
    s2 += pp[(int64_t)(c + 256) * B];
    s3 += pp[(int64_t)(c + 384) * B];
  }
  for (; c < nchunk; c += 128) s0 += pp[(int64_t)c * B];
  double s = (s0 + s1) + (s2 + s3);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ double ws[4];
  if (lane == 0) ws[w] = s;
  __syncthreads();
  if (tid == 0) {
    const double t = ((ws[0] + ws[1]) + ws[2]) + ws[3];
    out[i] = accumulate ? out[i] + t : t;
  }
}
// sum over elements of E[e][b] (deterministic) -> out[b] (+= if accumulate)
__global__ void k_sum_elems(const double* __restrict__ E, int m, int B, double* __restrict__ out, int accumulate) {
  PDL_ENTRY();
  extern __shared__ double red[];
  const int b = blockIdx.x;
  double s = 0;
  for (int e = threadIdx.x; e < m; e += blockDim.x) s += E[(int64_t)e * B + b];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[b] = accumulate ? out[b] + red[0] : red[0];
}

// ----------------------------------------------------------------- forward quasi-Newton (L-BFGS, H0 = A^{-1})
// The quasi-Newton PD of P:79/P:254 (Liu et al.): minimise g (eq:opt) with L-BFGS whose initial inverse
// Hessian is the prefactorised A^{-1}; Armijo backtracking on g.  Same minimiser as plain PD.

// partial[c][b] = sum over chunk c of (m_node/h^2) (X - Y)^2 (the per-sim chunking of k_dot_partial); with G: a
// second pair, sum of G^2 (the gradient norm of the same evaluation)
__global__ void k_inertia_partial(const double* __restrict__ X, const double* __restrict__ Y,
                                  const double* __restrict__ mass, double inv_h2, int64_t len, int B,
                                  double* __restrict__ partial, const double* __restrict__ G = nullptr) {
  PDL_ENTRY();
  __shared__ double red[2][kRedJ][kRedS];
  const RedLane r = red_lane(B, blockIdx.y);
  const int c = blockIdx.x;
  double acc = 0, acc2 = 0;
  if (r.ok) {
    const int64_t d1 = min(len, (int64_t)(c + 1) * kRedC);
    for (int64_t d = (int64_t)c * kRedC + r.j; d < d1; d += kRedJ) {
      const int64_t i = d * B + r.b;
      const double e = X[i] - Y[i];
      acc += mass[d / 3] * inv_h2 * e * e;
      if (G) acc2 += G[i] * G[i];
    }
  }
  red[0][r.j][r.bl] = acc;
  red[1][r.j][r.bl] = acc2;
  red_store(red, G ? 2 : 1, r, B, gridDim.x, c, partial);
}

// f[b] = 0.5 * inert[b] + esum[b]
__global__ void k_obj_combine(const double* __restrict__ inert, const double* __restrict__ esum, double* __restrict__ f,
                              int B) {
  PDL_ENTRY();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) f[b] = 0.5 * inert[b] + esum[b];
}

// two-loop recursion steps, per sim coefficient from a dot product:
//   mode 0: a = rho*dot; aj[b] = a; Y -= a V          (newest -> oldest)
//   mode 1: beta = rho*dot; Y += (aj - beta) V        (oldest -> newest)
__global__ void k_lbfgs_axpy(double* __restrict__ Y, const double* __restrict__ V, const double* __restrict__ rho,
                             const double* __restrict__ dot, double* __restrict__ aj, int mode, int64_t len, int B,
                             const int32_t* __restrict__ active) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= len) return;
  const int b = (int)(i % B);
  if (active && !active[b]) return;
  const double t = rho[b] * dot[b];
  if (mode == 0) {
    if (i < B) aj[b] = t;
    Y[i] -= t * V[i];
  } else {
    Y[i] += (aj[b] - t) * V[i];
  }
}

// Host-visible iteration control: the check kernels publish the three loop counters
// ([0] sims still searching / adjoint sims running, [1] forward sims running, [2] running sims within 16 tol) to a
// mapped pinned host word triple, then a sequence number; the host polls the sequence number instead of
// enqueueing a copy and synchronising the stream.  own: bit k set = slot k is the value computed by this kernel
// (v0..v2), the other slots are re-read from the device triple written by earlier kernels of the stream.
__device__ __forceinline__ void publish3(int32_t* hflag, const int32_t* nact3, int seq, int own, int v0, int v1,
                                         int v2) {
  if (!hflag) return;
  volatile int32_t* h = hflag;
  const volatile int32_t* d = nact3;
  h[0] = (own & 1) ? v0 : d[0];
  h[1] = (own & 2) ? v1 : d[1];
  h[2] = (own & 4) ? v2 : d[2];
  __threadfence_system();
  h[3] = seq;
}

// Armijo backtracking decision per sim.  Near the minimiser g no longer resolves the decrease in fp64;
// there a step that leaves g unchanged to 1e-13 relative and lowers ||grad g|| is accepted (the oracle's
// Newton uses the same rule).  After max_trial halvings the step is taken anyway and flagged.
// One block (loop over sims): the count of sims still searching is written to *nactive (no memset).
// fn[b] = 0.5 inert[b] + esum[b] is formed here (the objective of the trial point, eq:opt).
__global__ void k_ls_accept(const double* __restrict__ f, double* __restrict__ fn, const double* __restrict__ inert,
                            const double* __restrict__ esum, const double* __restrict__ gtd,
                            const double* __restrict__ g2, const double* __restrict__ gn2, double* __restrict__ alpha,
                            int32_t* __restrict__ ls_active, int trial, int max_trial, int32_t* __restrict__ nactive,
                            int32_t* __restrict__ ls_flag, int B, int32_t* hflag = nullptr,
                            const int32_t* nact3 = nullptr, int seq = 0) {
  PDL_ENTRY();
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    if (!ls_active[b]) continue;
    const double fnb = 0.5 * inert[b] + esum[b];
    fn[b] = fnb;
    const double a = alpha[b];
    const bool armijo = fnb <= f[b] + 1e-4 * a * gtd[b];
    const bool flat = fabs(fnb - f[b]) <= 1e-13 * fabs(f[b]) && gn2[b] < g2[b];
    if (armijo || flat || trial >= max_trial) {
      ls_active[b] = 0;
      if (!(armijo || flat)) ls_flag[b] = 1;
    } else {
      alpha[b] = 0.5 * a;
      atomicAdd(&cnt, 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *nactive = cnt;
    publish3(hflag, nact3, seq, 1, cnt, 0, 0);
  }
}

// rho = 1/(s^T y) if the curvature pair is positive, else 0 (pair ignored)
__global__ void k_lbfgs_rho(const double* __restrict__ sy, double* __restrict__ rho, const int32_t* __restrict__ active,
                            int B) {
  PDL_ENTRY();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B || !active[b]) return;
  rho[b] = sy[b] > 0.0 ? 1.0 / sy[b] : 0.0;
}

// ---- compact two-loop recursion (same iterates as the textbook two-loop, fewer passes)
// With the Gram matrix Gm[i][j] = s_i^T y_j kept per sim, every coefficient of the two-loop
// recursion follows from m dots with g (first loop) and m dots with r0 = A^{-1} q (second loop):
//   alpha_i = rho_i (s_i^T g - sum_{j newer} alpha_j Gm[i][j]),  q = g - sum alpha_j y_j,
//   beta_i  = rho_i (y_i^T r0 + sum_{j older} (alpha_j - beta_j) Gm[j][i]),
//   d = -(r0 + sum_j (alpha_j - beta_j) s_j).

// partial[(j*nchunk + c)*B + b] = sum over chunk c of u * V_j  (V_j = Vbase + j*vstride), j < nv; with u2:
// pairs nv + j = u2 * V2_j as well (both families of the new curvature pair in one launch).  Block (c, j, group):
// one chunk of one pair (the per-sim chunking of k_dot_partial), so every block streams two vectors.
__global__ void k_mdot_partial(const double* __restrict__ u, const double* __restrict__ Vbase, int64_t vstride,
                               int nv, int64_t len, int B, double* __restrict__ partial,
                               const double* __restrict__ u2 = nullptr, const double* __restrict__ V2base = nullptr) {
  PDL_ENTRY();
  __shared__ double red[1][kRedJ][kRedS];
  const RedLane r = red_lane(B, blockIdx.z);
  const int jp = blockIdx.y;
  const bool second = jp >= nv;
  const double* __restrict__ uu = second ? u2 : u;
  const double* __restrict__ V = (second ? V2base : Vbase) + (int64_t)(second ? jp - nv : jp) * vstride;
  const int c = blockIdx.x;
  double acc = 0.0;
  if (r.ok) {
    const int64_t d1 = min(len, (int64_t)(c + 1) * kRedC);
    int64_t d = (int64_t)c * kRedC + r.j;
    // four DoFs per trip: all eight loads in flight, then the in-order accumulation
    for (; d + 3 * kRedJ < d1; d += 4 * kRedJ) {
      const int64_t i = d * B + r.b, st = (int64_t)kRedJ * B;
      const double a0 = uu[i], a1 = uu[i + st], a2 = uu[i + 2 * st], a3 = uu[i + 3 * st];
      const double b0 = V[i], b1 = V[i + st], b2 = V[i + 2 * st], b3 = V[i + 3 * st];
      acc += a0 * b0;
      acc += a1 * b1;
      acc += a2 * b2;
      acc += a3 * b3;
    }
    for (; d < d1; d += kRedJ) acc += uu[d * B + r.b] * V[d * B + r.b];
  }
  red[0][r.j][r.bl] = acc;
  red_store(red, 1, r, B, gridDim.x, c, partial + (int64_t)jp * gridDim.x * B);
}

constexpr int kMaxHist = 16;  // largest L-BFGS memory the two-loop kernels support
// slot of the k-th newest pair at iteration `iter` (ring of m)
__device__ __forceinline__ int lb_slot(int iter, int k, int m) { return ((iter - 1 - k) % m + m) % m; }

// one warp per sim: the per-sim Gram data staged in shared memory, the (tiny, sequential) recursion in lane 0
__global__ void k_lbfgs_alpha(const double* __restrict__ sg, const double* __restrict__ Gm, const double* __restrict__ rho,
                              double* __restrict__ alpha, int m, int hist, int iter, int B,
                              const int32_t* __restrict__ active) {
  PDL_ENTRY();
  __shared__ double g[kMaxHist * kMaxHist], sv[kMaxHist], rv[kMaxHist], av[kMaxHist];
  const int b = blockIdx.x, lane = threadIdx.x;
  if (!active[b]) return;
  for (int i = lane; i < m * m; i += 32) g[i] = Gm[(int64_t)i * B + b];
  if (lane < m) {
    sv[lane] = sg[lane * B + b];
    rv[lane] = rho[lane * B + b];
  }
  __syncwarp();
  if (lane == 0)
    for (int k = 0; k < hist; ++k) {
      const int i = lb_slot(iter, k, m);
      double t = sv[i];
      for (int kk = 0; kk < k; ++kk) {
        const int j = lb_slot(iter, kk, m);
        t -= av[j] * g[i * m + j];
      }
      av[i] = rv[i] * t;
    }
  __syncwarp();
  if (lane < hist) {
    const int i = lb_slot(iter, lane, m);
    alpha[i * B + b] = av[i];
  }
}

__global__ void k_lbfgs_beta(const double* __restrict__ yr, const double* __restrict__ Gm, const double* __restrict__ rho,
                             const double* __restrict__ alpha, double* __restrict__ beta, int m, int hist, int iter,
                             int B, const int32_t* __restrict__ active) {
  PDL_ENTRY();
  __shared__ double g[kMaxHist * kMaxHist], yv[kMaxHist], rv[kMaxHist], av[kMaxHist], bv[kMaxHist];
  const int b = blockIdx.x, lane = threadIdx.x;
  if (!active[b]) return;
  for (int i = lane; i < m * m; i += 32) g[i] = Gm[(int64_t)i * B + b];
  if (lane < m) {
    yv[lane] = yr[lane * B + b];
    rv[lane] = rho[lane * B + b];
    av[lane] = alpha[lane * B + b];
  }
  __syncwarp();
  if (lane == 0)
    for (int k = hist - 1; k >= 0; --k) {
      const int i = lb_slot(iter, k, m);
      double t = yv[i];
      for (int kk = hist - 1; kk > k; --kk) {
        const int j = lb_slot(iter, kk, m);
        t += (av[j] - bv[j]) * g[j * m + i];
      }
      bv[i] = rv[i] * t;
    }
  __syncwarp();
  if (lane < hist) {
    const int i = lb_slot(iter, lane, m);
    beta[i * B + b] = bv[i];
  }
}

// Y = sgn * (X + csgn * sum_{j < nv} (c1_j - c2_j) V_j) per sim (c2 may be null), masked by active
__global__ void k_multi_axpy(double* __restrict__ Y, const double* __restrict__ X, double sgn, double csgn,
                             const double* __restrict__ Vbase, int64_t vstride, const double* __restrict__ c1,
                             const double* __restrict__ c2, int nv, int64_t len, int B,
                             const int32_t* __restrict__ active, double* __restrict__ Xn = nullptr,
                             const double* __restrict__ Xc = nullptr, const double* __restrict__ alpha_ls = nullptr) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= len) return;
  const int b = (int)(i % B);
  if (active && !active[b]) return;
  double v = X[i];
  for (int j = 0; j < nv; ++j) v += csgn * (c1[j * B + b] - (c2 ? c2[j * B + b] : 0.0)) * Vbase[j * vstride + i];
  const double d = sgn * v;
  Y[i] = d;
  // fused first line-search trial (k_axpby's arithmetic: x_trial = 1.0 x + (alpha 1.0) d, alpha = 1 from k_fwd_check)
  if (Xn) {
    double t = 1.0 * Xc[i];
    t += (alpha_ls[b] * 1.0) * d;
    Xn[i] = t;
  }
}

// The first multi-axpy of the two-loop recursion written straight into the solve layout (k_multi_axpy followed by
// k_to_solve in one pass, same arithmetic per entry): S[pos][3B] = sgn (X + csgn sum_j c1_j V_j) at the node of pos;
// the columns of inactive sims are zero (their solution is never read: k_from_solve is masked).
__global__ void k_multi_axpy_solve(double* __restrict__ S, const double* __restrict__ X, double sgn, double csgn,
                                   const double* __restrict__ Vbase, int64_t vstride, const double* __restrict__ c1,
                                   const double* __restrict__ c2, int nv, int nfree, int B,
                                   const int32_t* __restrict__ active, const int32_t* __restrict__ node_of_pos) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int R = 3 * B;
  if (i >= (int64_t)nfree * R) return;
  const int64_t pos = i / R;
  const int rr = (int)(i - pos * R);
  const int b = rr % B;
  if (active && !active[b]) {
    S[i] = 0.0;
    return;
  }
  const int64_t src = 3 * (int64_t)node_of_pos[pos] * B + rr;
  double v = X[src];
  for (int j = 0; j < nv; ++j) v += csgn * (c1[j * B + b] - (c2 ? c2[j * B + b] : 0.0)) * Vbase[j * vstride + src];
  S[i] = sgn * v;
}

// new pair in slot sl: Gm[sl][j] = s_sl^T y_j (da[j]), Gm[j][sl] = s_j^T y_sl (db[j]); rho_sl.
// Also commits the accepted point's scalars: f = f_new, |grad g|^2 (gg[b], read by the next convergence
// check) = |grad g_new|^2.
__global__ void k_gram_store(double* __restrict__ Gm, double* __restrict__ rho, const double* __restrict__ da,
                             const double* __restrict__ db, int sl, int m, int nv, int B,
                             const int32_t* __restrict__ active, double* __restrict__ f, const double* __restrict__ fn,
                             double* __restrict__ gg, const double* __restrict__ gn2,
                             double* __restrict__ gamma = nullptr, const double* __restrict__ step = nullptr,
                             const double* __restrict__ gtd = nullptr) {
  PDL_ENTRY();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B || !active[b]) return;
  for (int j = 0; j < nv; ++j) {
    Gm[(sl * m + j) * B + b] = da[j * B + b];
    Gm[(j * m + sl) * B + b] = db[j * B + b];
  }
  const double sy = da[sl * B + b];
  rho[sl * B + b] = sy > 0.0 ? 1.0 / sy : 0.0;
  // Per-sim scaling of the initial inverse Hessian, H0 = gamma A^{-1}: after the first step of a
  // solve, s = step * d with d = -gamma A^{-1} grad g, so s^T A s = -step^2 gamma (grad g . d) needs no extra solve,
  // and gamma <- s^T A s / s^T y is the Rayleigh quotient of the prefactorised A against the sim's true Hessian
  // along s (sims whose own E differs from the factorised E_ref; A_N below A under large rotations).
  if (gamma) {
    const double a = step[b], gd = gtd[b], g0 = gamma[b];
    if (sy > 0.0 && gd < 0.0) gamma[b] = fmin(16.0, fmax(0.0625, -a * a * g0 * gd / sy));
  }
  if (f) {
    f[b] = fn[b];
    gg[b] = gn2[b];
  }
}

// commit of an accepted L-BFGS step (one pass): S_sl = Xn - X, Y_sl = Gn - G, X = Xn, G = Gn (masked)
__global__ void k_lbfgs_commit(double* __restrict__ S, double* __restrict__ Yv, double* __restrict__ X,
                               double* __restrict__ G, const double* __restrict__ Xn, const double* __restrict__ Gn,
                               int64_t len, int B, const int32_t* __restrict__ active) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= len) return;
  const int b = (int)(i % B);
  if (!active[b]) return;
  const double xn = Xn[i], gn = Gn[i];
  S[i] = xn - X[i];
  Yv[i] = gn - G[i];
  X[i] = xn;
  G[i] = gn;
}

// Newton-PCG forward (accel_fwd = 2): commit of an accepted trial, X <- Xn, G <- Gn (state vectors, masked)
__global__ void k_newton_commit(double* __restrict__ X, double* __restrict__ G, const double* __restrict__ Xn,
                                const double* __restrict__ Gn, int64_t len, int B, const int32_t* __restrict__ active) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= len) return;
  const int b = (int)(i % B);
  if (!active[b]) return;
  X[i] = Xn[i];
  G[i] = Gn[i];
}
// ... and its per-sim scalars: f <- f_new, |grad g|^2 <- that of the trial
__global__ void k_newton_commit_s(double* __restrict__ f, const double* __restrict__ fn, double* __restrict__ g2,
                                  const double* __restrict__ gn2, int B, const int32_t* __restrict__ active) {
  PDL_ENTRY();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B || !active[b]) return;
  f[b] = fn[b];
  g2[b] = gn2[b];
}
// Truncated CG on a non-convex Hessian: a sim whose search direction has p^T A_N p <= 0 stops its CG (its
// direction so far is kept; a zero direction falls back to the PD step below).
__global__ void k_negcurv(const double* __restrict__ pq, int32_t* __restrict__ active, int B) {
  PDL_ENTRY();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B && active[b] && !(pq[b] > 0.0)) active[b] = 0;
}
// Descent guard: where <grad g, D> >= 0 (not a descent direction), D = the PD direction -A^{-1} grad g (Z0)
__global__ void k_descent_guard(double* __restrict__ D, const double* __restrict__ Z0, const double* __restrict__ gtd,
                                int64_t len, int B, const int32_t* __restrict__ active) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= len) return;
  const int b = (int)(i % B);
  if (active[b] && !(gtd[b] < 0.0)) D[i] = Z0[i];
}

// v[b] = c (per-sim scalar fill)
__global__ void k_fill_double(double* __restrict__ v, double c, int B) {
  PDL_ENTRY();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) v[b] = c;
}

// masked copy of per-sim scalars
__global__ void k_copy_masked(double* __restrict__ dst, const double* __restrict__ src, const int32_t* __restrict__ active,
                              int B) {
  PDL_ENTRY();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B && (!active || active[b])) dst[b] = src[b];
}

// ----------------------------------------------------------------- iteration control
// Forward convergence: res = sqrt(res2/den2); active[b] for the NEXT update.  One block (loop over sims):
// the active count is written to *nactive (no memset).  With alpha/ls_act: line-search state of the
// coming iteration (alpha = 1, ls_act = active).
__global__ void k_fwd_check(const double* __restrict__ dots, int B, double tol, int iter, int fixed_iter,
                            int max_iter, int32_t* __restrict__ active, int32_t* __restrict__ iters_out,
                            double* __restrict__ res_out, int32_t* __restrict__ flag_out,
                            int32_t* __restrict__ nactive, const int32_t* __restrict__ iter_base,
                            double* __restrict__ alpha = nullptr, int32_t* __restrict__ ls_act = nullptr,
                            int32_t* __restrict__ nnear = nullptr, int32_t* hflag = nullptr,
                            const int32_t* nact3 = nullptr, int seq = 0) {
  PDL_ENTRY();
  __shared__ int cnt, near;
  if (threadIdx.x == 0) cnt = near = 0;
  __syncthreads();
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    int act = active[b];
    if (act) {
      const double den = dots[B + b];
      const double res = den > 0 ? sqrt(dots[b] / den) : sqrt(dots[b]);
      bool go;
      if (fixed_iter > 0) go = iter < fixed_iter;
      else go = res > tol && iter < max_iter;
      res_out[b] = res;
      iters_out[b] = iter + (iter_base ? iter_base[b] : 0);
      if (!go) {
        active[b] = act = 0;
        flag_out[b] = (fixed_iter == 0 && res > tol) ? 1 : 0;
      } else {
        atomicAdd(&cnt, 1);  // integer count only (no effect on arithmetic)
        if (res < 16.0 * tol) atomicAdd(&near, 1);
      }
    }
    if (alpha) {
      alpha[b] = 1.0;
      ls_act[b] = act;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *nactive = cnt;
    if (nnear) *nnear = near;
    // (L-BFGS / Newton: nactive = nact3 + 1, nnear = nact3 + 2; plain PD: nactive = nact3)
    if (nnear) publish3(hflag, nact3, seq, 6, 0, cnt, near);
    else publish3(hflag, nact3, seq, 1, cnt, 0, 0);
  }
}

// v = (x - xprev)/h
__global__ void k_velocity(const double* __restrict__ X, const double* __restrict__ Xp, double* __restrict__ V,
                           int64_t len, double inv_h) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < len) V[i] = (X[i] - Xp[i]) * inv_h;
}

// generic per-sim axpy on state vectors: Y[i] = a*X[i] + c[b]*cs*Z[i] (+ masks)
__global__ void k_axpby(double* __restrict__ Y, const double* __restrict__ X, double a, const double* __restrict__ Z,
                        const double* __restrict__ c, double cs, int64_t len, int B, const int32_t* __restrict__ active) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= len) return;
  const int b = (int)(i % B);
  if (active && !active[b]) return;
  double v = X ? a * X[i] : 0.0;
  if (Z) v += (c ? c[b] : 1.0) * cs * Z[i];
  Y[i] = v;
}
// zero fixed nodes (and pinned z DoFs) of a state vector
__global__ void k_zero_constrained(double* __restrict__ Y, const uint8_t* __restrict__ fixed, int n, int B,
                                   const int32_t* __restrict__ cand_of_node, const uint8_t* __restrict__ PIN,
                                   int pin_all = 0) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)3 * n * B) return;
  const int64_t d = i / B;
  const int b = (int)(i - d * B);
  const int node = (int)(d / 3), ax = (int)(d - 3 * (int64_t)node);
  bool z = fixed[node] != 0;
  if (!z && (ax == 2 || pin_all) && PIN && cand_of_node[node] >= 0) z = PIN[(int64_t)cand_of_node[node] * B + b] != 0;
  if (z) Y[i] = 0.0;
}

// Sticky contact adjoint (x_{i+1,a} = x_{i,a}): EX = (a_x + a_v/h - A_N u) on pinned DoFs, 0 elsewhere; added to
// dL/dx_i after the state-adjoint update (oracle/adjoint.py).
__global__ void k_sticky_extra(double* __restrict__ EX, const double* __restrict__ AX, const double* __restrict__ AV,
                               const double* __restrict__ ANu, double inv_h, int n, int B,
                               const int32_t* __restrict__ cand_of_node, const uint8_t* __restrict__ PIN) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)3 * n * B) return;
  const int64_t d = i / B;
  const int b = (int)(i - d * B);
  const int cj = cand_of_node[d / 3];
  EX[i] = (cj >= 0 && PIN[(int64_t)cj * B + b]) ? AX[i] + AV[i] * inv_h - ANu[i] : 0.0;
}

// Adjoint PCG scalars.  dots layout: [0:B) first pair, [B:2B) second ...
// alpha = rz / pq ; converged check on rr / bb.
// PCG (preconditioner A^{-1}) fused updates, per-sim coefficients formed per element:
//   k_pcg_update: alpha = rz / pq; U += alpha P; R -= alpha Q
//   k_pcg_dir:    beta = rz_new / rz; P = Z + beta P
__global__ void k_pcg_update(double* __restrict__ U, double* __restrict__ Rv, const double* __restrict__ P,
                             const double* __restrict__ Q, const double* __restrict__ rz, const double* __restrict__ pq,
                             int64_t len, int B, const int32_t* __restrict__ active, double* __restrict__ S = nullptr,
                             const int32_t* __restrict__ pos_of_node = nullptr) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= len) return;
  const int b = (int)(i % B);
  // the new residual also in the solve layout (fused k_to_solve of the coming z = A^{-1} r); the columns of
  // converged sims are zero (their solution is never read: k_from_solve is masked)
  int64_t si = -1;
  if (S) {
    const int64_t dof = i / B;
    const int node = (int)(dof / 3), ax = (int)(dof - 3 * (int64_t)node);
    const int pos = pos_of_node[node];
    if (pos >= 0) si = (int64_t)pos * 3 * B + ax * B + b;
  }
  if (!active[b]) {
    if (si >= 0) S[si] = 0.0;
    return;
  }
  const double d = pq[b];
  const double alpha = d != 0.0 ? rz[b] / d : 0.0;
  U[i] = U[i] + alpha * P[i];
  const double r = Rv[i] + (-alpha) * Q[i];
  Rv[i] = r;
  if (si >= 0) S[si] = r;
}
__global__ void k_pcg_dir(double* __restrict__ P, const double* __restrict__ Z, const double* __restrict__ rz_new,
                          const double* __restrict__ rz, int64_t len, int B, const int32_t* __restrict__ active) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= len) return;
  const int b = (int)(i % B);
  if (!active[b]) return;
  const double beta = rz[b] != 0.0 ? rz_new[b] / rz[b] : 0.0;
  P[i] = Z[i] + beta * P[i];
}
// Adjoint convergence; one block (loop over sims), the active count written to *nactive (no memset).  With
// rz: rz[b] = rz_new[b] for the sims that ran the previous PCG iteration.
__global__ void k_adj_check(const double* __restrict__ rr, const double* __restrict__ bb, int B, double tol, int iter,
                            int max_iter, int32_t* __restrict__ active, int32_t* __restrict__ iters_out,
                            double* __restrict__ res_out, int32_t* __restrict__ flag_out, int32_t* __restrict__ nactive,
                            double* __restrict__ rz = nullptr, const double* __restrict__ rz_new = nullptr,
                            int32_t* hflag = nullptr, const int32_t* nact3 = nullptr, int seq = 0) {
  PDL_ENTRY();
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    if (!active[b]) continue;
    if (rz) rz[b] = rz_new[b];
    const double res = bb[b] > 0 ? sqrt(rr[b] / bb[b]) : 0.0;
    res_out[b] = res;
    iters_out[b] = iter;
    const bool go = res > tol && iter < max_iter;
    if (!go) {
      active[b] = 0;
      flag_out[b] = res > tol ? 1 : 0;
    } else {
      atomicAdd(&cnt, 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *nactive = cnt;
    publish3(hflag, nact3, seq, 1, cnt, 0, 0);
  }
}

// a_x = (M/h^2) u - a_v/h ; a_v = (M/h) u ; zero on fixed nodes  (eq:pre_adjoint)
__global__ void k_adj_state(const double* __restrict__ U, const double* __restrict__ mass, const uint8_t* __restrict__ fixed,
                            double* __restrict__ AX, double* __restrict__ AV, int n, int B, double h) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)3 * n * B) return;
  const int node = (int)(i / B / 3);
  if (fixed[node]) { AX[i] = 0.0; AV[i] = 0.0; return; }
  const double u = U[i], mm = mass[node];
  const double av = AV[i];
  AX[i] = mm / (h * h) * u - av / h;
  AV[i] = mm / h * u;
}

}  // namespace pdb
