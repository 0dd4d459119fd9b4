/*
 * diffpd_b200.h — C-ABI of the B200-native DiffPD hot path (arXiv 2101.05917).
 *
 * One opaque handle per (mesh, material, h, Dirichlet set, contact set).  The
 * library owns every device allocation it makes (factor, caches, workspaces,
 * trajectory store); every array ARGUMENT is caller-owned.  Unless stated
 * otherwise array arguments are fp64 DEVICE pointers (e.g. a contiguous torch
 * CUDA tensor's data_ptr()) in the layout [B][3n], DoF index = 3*node + axis
 * ("the floor(i/3) convention").  Mesh/material/option structs and
 * their pointers are HOST memory.  Work is enqueued on `cuda_stream` (a
 * cudaStream_t, NULL = legacy default stream); every call returns after the
 * work completed (results are host-visible on return).  No allocation happens
 * inside pd_forward / pd_backward.  A handle is not re-entrant; separate handles
 * may be used concurrently from separate threads/streams.
 *
 * Errors: every entry point returns a pd_status; the message of the last
 * failure is available from pd_last_error(handle) (or pd_last_error(NULL) for
 * a failed pd_create).  Non-convergence of an iteration is NOT an error: the
 * call returns PD_OK with the per-step flags/counters in pd_stats.
 */
#ifndef DIFFPD_B200_H
#define DIFFPD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pd_sim pd_sim;

typedef enum {
  PD_OK = 0,
  PD_ERR_INVALID_ARGUMENT = 1, /* bad sizes, non-voxel mesh, nu outside (-1, .5), h <= 0, ... */
  PD_ERR_NUMERICAL = 2,        /* A not SPD at setup; singular contact capacitance matrix     */
  PD_ERR_CUDA = 3,             /* a CUDA runtime call failed (message has the CUDA error)     */
  PD_ERR_STATE = 4             /* e.g. pd_backward without a preceding pd_forward             */
} pd_status;

/* Hexahedral voxel mesh ("FEM-discretization", P:189 G_e).
 * rest_xyz: host [n_nodes][3] rest positions (m).  hex8: host [n_elems][8]
 * node indices, corner a = di + 2 dj + 4 dk (x-fastest).  Every element must be
 * an axis-aligned cube of edge dx (checked; otherwise INVALID_ARGUMENT): all
 * elements then share one constant G stencil (8-point Gauss). */
typedef struct {
  int32_t n_nodes, n_elems;
  const double* rest_xyz;
  const int32_t* hex8;
  double dx;
} pd_mesh;

/* Material.  Corotated PD weight w = E/(1+nu) (= 2 mu, the
 * reading of DESIGN.md §2.2).  muscle_w > 0 enables the muscle-fiber energy
 * (w_m/2)||Fm - p||^2, p = r Fm/||Fm|| with the
 * uniform unit fiber direction `fiber`; actuation r is given per (sim, step,
 * element) to pd_forward.  gravity (m/s^2) enters f_ext as M g. */
typedef struct {
  double youngs, poisson, density;
  double muscle_w;
  double gravity[3];
  double fiber[3];
  int32_t volume;         /* 1: add the volume-preserving PD energy (w_v/2)||F - D||^2, D the projection of F onto
                             det D = 1, with w_v = lambda = E nu / ((1+nu)(1-2nu)) per sim (SPEC lame_weights,
                             DESIGN.md §2.16); its Jacobian from the differentiated KKT system.
                             pd_backward's dL_dE and dL_dnu then include the w_v terms.  0: corotated only.      */
  const double* fiber_dir; /* [n_elems][3] HOST per-element fiber directions (normalised by the library; zero rows
                             -> INVALID_ARGUMENT), or NULL = the uniform `fiber`.  The muscle energy of element e
                             is (w_m/2) ||F m_e - p||^2 with its own m_e; A stays A_s (x) I_3       */
} pd_material;

/* Solver options.  Tolerances are on the relative residual
 * ||grad g(x)||_2 / ||(M/h^2) y||_2 over unconstrained DoFs (forward, P:527 and
 * DESIGN.md §2.8) and ||A_N u - b|| / ||b|| (adjoint). */
typedef struct {
  double tol_fwd, tol_adj;
  int32_t max_iter_fwd, max_iter_adj;
  int32_t fixed_iter;     /* > 0: exactly this many plain local-global iterations per step
                             from x^0 = x_i, no convergence test (config c1)               */
  int32_t accel_fwd;      /* 0: plain PD x <- A^{-1} d(x); 1: L-BFGS with
                             H0 = A^{-1} and line search (the quasi-Newton PD of P:79/P:254);
                             2: the Newton baseline as Newton-PCG: truncated CG on the
                             Hessian A_N(x) preconditioned by the prefactorised A^{-1}, forcing term
                             1e-2, descent guard, same line search (comparison system) */
  int32_t accel_adj;      /* 0: fixed point u <- A^{-1}(b + dA u);
                             1: its quasi-Newton acceleration, run as
                             A-preconditioned CG — BFGS with exact line search on a(u)   */
  int32_t check_every;    /* host polls convergence flags every k iterations (>= 1)        */
  int32_t max_batch;      /* largest B passed to pd_forward; at most 256 (the solve splits the 3B right-hand
                             sides into <= 16 column chunks of 48; pd_create returns INVALID_ARGUMENT above) */
  int32_t max_steps;      /* largest `steps` passed to pd_forward (trajectory store size)  */
  double youngs_ref;      /* Young's modulus of the ONE factorised A (0 = material.youngs).
                             Sims with other E use the majorising step of DESIGN.md §2.12  */
  /* Frictionless node-plane contact (Alg. 1):
   * candidate nodes V (host, node indices); the plane is plane_n / plane_d below (default z = 0, normal +z). */
  const int32_t* contact_nodes;
  int32_t n_contact;
  int32_t max_outer;      /* Alg. 1 "maximum iteration" (default 10)                     */
  double eps_phi;         /* predictor penetration threshold (m), default 1e-6 dx          */
  int32_t profile;        /* 1: bracket each kernel family with CUDA events (pd_profile)   */
  int32_t outer_warm;     /* 1: outer iterations k > 1 of Alg. 1 start from iteration k-1's x
                             (pinned DoFs moved to the plane) instead of x_i; the converged x
                             of each corrector solve is the same            */
  int32_t contact_mode;   /* 1 (or 0): frictionless — an active candidate's normal DoF is pinned on the
                             plane (reading §2.10); 2: sticky — all three DoFs of an active candidate
                             are held at x_i (the paper's infinite-friction nodes)  */
  int32_t x0_predict;     /* 1: start each step's solve from x_i + h v_i instead of x_i (converged
                             configurations only; fixed_iter keeps x^0 = x_i, reading §2.6).
                             Changes iteration counts, not the converged minimiser          */
  int32_t lbfgs_warm;     /* accel_fwd = 1 with contact: 1 keeps the L-BFGS curvature pairs across the Alg. 1
                             outer iterations of a time step (restricted to the new free DoFs, Gram matrix
                             recomputed); 0 restarts the history with every corrector solve.  Changes
                             iteration counts, not the converged minimiser   */
  /* Contact plane n . x = d ("phi is a linear function and n ... a constant vector"): plane_n need not be
   * unit (normalised; all zero = +z), the free side is n . x > d; phi_j = n . x_j - d, lambda_j = n . grad_j g.
   * Default (zero-initialised or {0, 0, 1}, 0): the ground z = 0 of BASELINE configs[3-4].  Internally the
   * library works in plane coordinates x' = Q x - d e_z (a rigid motion: the PD energy is invariant; gravity,
   * f_ext and all ABI vectors are rotated at the boundary, results are returned in world coordinates).
   * Non-finite values -> INVALID_ARGUMENT.  Ignored without contact candidates. */
  double plane_n[3];
  double plane_d;
} pd_options;

/* Per-step statistics, caller-owned HOST arrays of length B*steps (index
 * b*steps + i) or NULL each; filled by pd_forward / pd_backward. */
typedef struct {
  int32_t* iters_fwd;
  int32_t* iters_adj;
  int32_t* contact_outer;
  double* final_res_fwd;
  double* final_res_adj;
  int32_t n_nonconverged; /* output: number of (sim, step) that hit a cap or stagnated */
} pd_stats;

/* Build a handle: validate the mesh, assemble A = M/h^2 + sum w G^T G
 * on the free DoFs (fixed_dofs: host list of DoFs held at their rest
 * values; must cover whole nodes), order it (nested dissection), factor it
 * ONCE ("its Cholesky decomposition can be precomputed"), upload the
 * factor and, with contact candidates, the cache (A^{-1})_{VV}.
 * Returns INVALID_ARGUMENT / NUMERICAL / CUDA on failure (*out = NULL). */
pd_status pd_create(const pd_mesh* mesh, const pd_material* mat, double h,
                    const int32_t* fixed_dofs, int32_t n_fixed,
                    const pd_options* opts, pd_sim** out);

/* Forward simulation of B independent sims for `steps` backward-Euler steps
 * by PD local-global iterations, Alg. 1 contact when
 * candidates exist.
 *   q0, v0          device [B][3n]
 *   f_ext           device non-gravity external force (N): [B][3n] constant over steps
 *                   (f_ext_step_stride = 0), [B][steps][3n] per step (f_ext_step_stride = 3n), or NULL
 *   actuation       device [B][steps][n_elems] muscle activation r, or NULL
 *   youngs_per_sim  device [B] Young's modulus per sim, or NULL (= material.youngs)
 *   q_traj, v_traj  device [B][steps+1][3n] outputs, or NULL
 * The library keeps the trajectory for pd_backward until the next pd_forward. */
pd_status pd_forward(pd_sim* sim, int32_t B, const double* q0, const double* v0,
                     const double* f_ext, int64_t f_ext_step_stride,
                     const double* actuation, const double* youngs_per_sim,
                     int32_t steps, double* q_traj, double* v_traj,
                     pd_stats* stats, void* cuda_stream);

/* Reverse pass over the stored trajectory (adjoint method, with the
 * PD fixed point / quasi-Newton solve of A_N u = b; contact steps use
 * the same constrained matrix).
 *   dL_dqT, dL_dvT   device [B][3n] terminal loss gradients (NULL = 0)
 *   dL_dq0, dL_dv0   device [B][3n] outputs (or NULL)
 *   dL_dfext         device [B][3n] output, summed over steps (or NULL)
 *   dL_dE, dL_dnu    device [B] outputs (or NULL)
 *   dL_dact          device [B][steps][n_elems] output (or NULL)
 * Gradients on Dirichlet DoFs are exactly 0.  PD_ERR_STATE without a forward. */
pd_status pd_backward(pd_sim* sim, const double* dL_dqT, const double* dL_dvT,
                      double* dL_dq0, double* dL_dv0, double* dL_dfext,
                      double* dL_dE, double* dL_dnu, double* dL_dact,
                      pd_stats* stats, void* cuda_stream);

/* Reverse pass for per-step losses L = sum_i l_i(q_i, v_i) (the per-step losses of the paper's tasks, e.g.
 * "loss at each time step"):
 *   dL_dq_steps, dL_dv_steps  device [B][steps+1][3n] (dl_i/dq_i, dl_i/dv_i; NULL = 0)
 *   dL_dfext_steps            device [B][steps][3n] output: dL/df_ext of each step (or NULL)
 * other arguments as pd_backward.  Use f_ext_step_stride = 3n in pd_forward for per-step f_ext. */
pd_status pd_backward_steps(pd_sim* sim, const double* dL_dq_steps, const double* dL_dv_steps,
                            double* dL_dq0, double* dL_dv0, double* dL_dfext_steps,
                            double* dL_dE, double* dL_dnu, double* dL_dact,
                            pd_stats* stats, void* cuda_stream);

/* Diagnostics / kernel-level parity hooks (same conventions as above). */
/* grad_g[B][3n] = M/h^2 (x - y) + grad E_int(x) (eq:time_integration LHS) and
 * g[B] = eq:opt objective at x; act device [B][n_elems] or NULL. */
pd_status pd_eval_objective(pd_sim* sim, int32_t B, const double* x, const double* y,
                            const double* youngs_per_sim, const double* act,
                            double* grad_g, double* g, void* cuda_stream);
/* out[B][3n] = A^{-1} rhs on free DoFs (0 on Dirichlet DoFs): the factored global solve. */
pd_status pd_apply_Ainv(pd_sim* sim, int32_t B, const double* rhs, double* out, void* cuda_stream);
/* out[B][3n] = A_N(x) p = (M/h^2) p + Hess E_int(x) p on all DoFs (matrix-free). */
pd_status pd_apply_AN(pd_sim* sim, int32_t B, const double* x, const double* youngs_per_sim,
                      const double* act, const double* p, double* out, void* cuda_stream);
/* R[B][n_elems][8][9] = rotation R(F) of every quadrature point of x (local step projection). */
pd_status pd_project_rotations(pd_sim* sim, int32_t B, const double* x, double* R, void* cuda_stream);
/* Local-step statistics of x (device [B][3n]): out (HOST int64[3]) = {Newton-Schulz iterations summed over every
 * quadrature point K1's polar takes on x, quadrature points on that path, points that take the SVD / scaled-Newton
 * fallback}.  bench.py turns the mean iteration count into K1's algorithmic flops per quadrature point
 * (DESIGN.md §5).  Diagnostic: not on the hot path. */
pd_status pd_polar_stats(pd_sim* sim, int32_t B, const double* x, int64_t* out, void* cuda_stream);

/* Integer facts about the handle: out[0..n) = {n_nodes, n_free_nodes, n_supernodes,
 * n_levels, nnz(L_s) (stored entries of the scalar factor), n_contact,
 * setup_ms_factor (rounded), kernel launches of the last pd_forward+pd_backward}. */
pd_status pd_info(const pd_sim* sim, int64_t* out, int32_t n);

/* Per-kernel-family device time (CUDA events on the work stream) accumulated since the
 * start of the last pd_forward (forward + backward), when opts.profile = 1.
 * Families: 0 local step K1, 1 gather K2, 2 global solve K3 (one A^{-1} application),
 * 3 A_N product K4 (element pass + gather), 4 contact K5, 5 parameter terms.
 * ms[k] = total milliseconds, count[k] = number of timed regions. */
pd_status pd_profile(const pd_sim* sim, double* ms, int64_t* count, int32_t n);

/* Final active set of Alg. 1 for every (sim, step) of the last pd_forward:
 * out = HOST uint8 [B][steps][n_contact], 1 = normal DoF of candidate j pinned at the plane
 * (candidate order = opts.contact_nodes).  PD_ERR_STATE without a forward or without contact. */
pd_status pd_contact_sets(const pd_sim* sim, uint8_t* out);

const char* pd_last_error(const pd_sim* sim);
void pd_destroy(pd_sim* sim);

#ifdef __cplusplus
}
#endif
#endif /* DIFFPD_B200_H */
