// C-ABI of the B200 DiffPD hot path (include/diffpd_b200.h): handle lifetime,
// device residency and the per-step orchestration of the sm_100a kernels.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: per-phase ranges for nsys / ncu --nvtx (no-ops without a tool)

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/diffpd_b200.h"
#include "kernels.cu"  // single translation unit: kernels + orchestration
#include "plan.h"

using namespace pdb;

namespace {
thread_local std::string g_create_error;

__global__ void k_fill_int(int32_t* p, int32_t v, int n) {
  PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};
}  // namespace

struct pd_sim {
  HostPlan plan;
  std::string err;
  double youngs = 0, poisson = 0, density = 0, h = 0, w_m = 0;
  double gravity[3] = {0, 0, 0};
  pd_options opt{};
  int Bmax = 1, Tmax = 1;
  Stencil st{};
  std::vector<DevBuf> bufs;
  // plan on device
  double* d_fib = nullptr;  // [m][3] per-element unit fibers (material.fiber_dir) or null
  int32_t *d_hex8 = nullptr, *d_inc_ptr = nullptr, *d_inc_ec = nullptr, *d_pos = nullptr, *d_nodepos = nullptr;
  double* d_mass = nullptr;
  uint8_t* d_fixed = nullptr;
  uint8_t* d_nofix = nullptr;  // all-zero node mask (diagnostics on all DoFs)
  SweepDev swf{}, swb{};
  Sweep4Dev sw4f{}, sw4b{};  // K3 v4 (warp ranges), when plan.k3_version == 4
  int k3_mma = 1;   // K3 item products on the fp64 tensor cores (1) or the FMA pipe (0, env PD_K3_MMA=0)
  int nsm = 148;     // SMs of the device
  int k3_nbuf = 2;  // K3 item ring depth (2..4, env PD_K3_NBUF)
  bool poll = true;  // iteration control by polled host flags (env PD_POLL=0: D2H copy + stream synchronisation)
  bool lb_gamma = true;  // per-sim scaling gamma_b of H0 = gamma A^{-1} in the L-BFGS forward (env PD_LBFGS_GAMMA=0: 1)
  double* gamma = nullptr;
  // Probe only (env PD_ACTIVE_WARM=1, off by default, NOT Alg. 1 as printed): a time step's first outer iteration
  // starts from the previous step's final active set instead of the empty set of P:339
  bool active_warm = false;
  bool fuse = true;  // layout/trial passes fused into their producers (env PD_FUSE=0: separate passes, same bits)
  int lb_hist = 0, lb_gi = 0;  // L-BFGS history state carried across Alg. 1 outer iterations (lbfgs_warm)
  int32_t* d_rows = nullptr;
  double* Spart = nullptr;  // partial rows of the K3 sweeps
  int64_t* nactive_ll = nullptr;  // 3 x 64-bit device counters (pd_polar_stats)
  // general contact plane n . x = d: plane coordinates x' = Q x - d e_z inside the library
  bool frame = false;
  FrameQ fq{};
  // Newton-PCG forward (accel_fwd = 2): CG mask, CG statistics, forcing term (relative CG residual)
  int32_t *pact = nullptr, *nt_iters = nullptr, *nt_flag = nullptr;
  double* nt_res = nullptr;
  double newton_eta = 1e-2;
  // work
  double *X, *V, *Y, *Xp, *Fext, *G, *W, *EF, *EE, *S0, *S1, *S2;
  double *U, *Rv, *Z, *Pv, *Q, *AX, *AV, *Bv, *DF, *DW, *DR, *JC;
  double *w_sim, *youngs_sim, *dots, *partial, *alpha, *beta, *rz, *bb, *dw_acc, *act;
  double *DWV = nullptr, *dwv_acc = nullptr;  // volume-weight parameter terms (material.volume)
  // per-sim weights of the diagnostic hooks (pd_eval_objective / pd_apply_AN): kept apart from w_sim / youngs_sim,
  // which pd_backward reuses from the last pd_forward
  double *w_diag = nullptr, *youngs_diag = nullptr;
  const double* w_cur = nullptr;  // the weights the element kernels read (w_sim or w_diag)
  int32_t *active, *nactive, *it_buf, *flag_buf;
  double* res_buf;
  int32_t* h_nactive = nullptr;  // pinned, device-mapped: [0:3) the loop counters, [3] the published sequence number
  int flag_seq = 0;              // last sequence number handed to a check kernel (poll_flags waits for it)
  // contact K5
  int nc = 0, csup_first = 0;
  bool pins_live = false;          // the solve applies the constrained root block
  int sticky = 0;                  // contact_mode 2: active nodes hold all DoFs at x_i (infinite friction)
  int32_t *d_cand_node = nullptr, *d_cand_of_node = nullptr, *d_cand_of_loc = nullptr;
  double *d_S = nullptr, *LAM = nullptr, *Qc = nullptr, *PIc = nullptr, *Cb = nullptr, *Mb = nullptr, *Rb = nullptr,
         *Rsave = nullptr;
  uint8_t *PIN = nullptr, *NEWPIN = nullptr, *traj_pin = nullptr;
  int32_t *flist = nullptr, *fpos = nullptr, *kcount = nullptr, *need = nullptr, *oact = nullptr, *onext = nullptr,
          *changed = nullptr, *it_base = nullptr;
  int32_t* h_small = nullptr;      // pinned [2*Bmax]
  // forward L-BFGS (accel_fwd = 1)
  int nhist = 0;
  double *LS = nullptr, *LY = nullptr, *Dv = nullptr, *Xn = nullptr, *Gn = nullptr, *rho_h = nullptr, *aj_h = nullptr;
  double *fcur = nullptr, *fnew = nullptr, *alpha_ls = nullptr, *gtd = nullptr, *g2 = nullptr, *gn2 = nullptr,
         *inert = nullptr, *esum = nullptr, *dtmp = nullptr;
  int32_t *ls_act = nullptr, *ls_flag = nullptr;
  double *lb_sg = nullptr, *lb_yr = nullptr, *lb_beta = nullptr, *lb_da = nullptr, *lb_db = nullptr, *lb_G = nullptr;
  double* traj = nullptr;
  int32_t *st_iters_f, *st_iters_a, *st_flag_f, *st_flag_a, *st_outer;
  double *st_res_f, *st_res_a;
  int64_t max_partial_blocks = 0;
  // last forward
  bool have_traj = false;
  int B = 0, T = 0;
  bool has_act = false;
  int64_t launches = 0;
  cudaStream_t stream = nullptr;
  // profiler (opts.profile): event pairs per kernel family, resolved at host sync points
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, int>> ev_open;  // (family, index of start event)
  int ev_next = 0;
  // one scope in prof_every per family is timed (env PD_PROF_EVERY, default 4): an event boundary interrupts the
  // programmatic-dependent-launch chain, and timing every scope cost c5 3.9 % and c3 12.4 % of the timed region
  int prof_every = 4;
  int64_t prof_calls[6] = {0, 0, 0, 0, 0, 0};
  double prof_ms[6] = {0, 0, 0, 0, 0, 0};
  int64_t prof_cnt[6] = {0, 0, 0, 0, 0, 0};

  template <class T>
  T* alloc(size_t count) {
    DevBuf b;
    b.bytes = std::max<size_t>(count * sizeof(T), 16);
    if (cudaMalloc(&b.p, b.bytes) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
    cudaMemset(b.p, 0, b.bytes);
    bufs.push_back(b);
    return static_cast<T*>(b.p);
  }
  template <class T>
  T* upload(const std::vector<T>& v) {
    T* d = alloc<T>(v.size());
    if (!v.empty()) cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
    return d;
  }
  std::map<int, std::pair<cudaGraphExec_t, int64_t>> solve_graphs;  // (B, fixup) -> graph, kernels in it
  cudaStream_t cap_stream = nullptr;
  ~pd_sim() {
    if (cap_stream) cudaStreamDestroy(cap_stream);
    for (auto& g : solve_graphs) cudaGraphExecDestroy(g.second.first);
    for (auto& e : ev_pool) cudaEventDestroy(e);
    for (auto& b : bufs) cudaFree(b.p);
    if (h_nactive) cudaFreeHost(h_nactive);
    if (h_small) cudaFreeHost(h_small);
  }
};

namespace {

inline unsigned nblk(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }
// per-sim reductions (kernels.cu kRed*): chunks of kRedC DoFs, kRedJ threads per sim, groups of kRedS sims
inline int red_chunks(int64_t len) { return (int)((len + kRedC - 1) / kRedC); }
inline unsigned red_threads(int B) { return (unsigned)(kRedJ * std::min(B, kRedS)); }
inline unsigned red_groups(int B) { return (unsigned)((B + kRedS - 1) / kRedS); }

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
#define CK(x)                                                                                         \
  do {                                                                                                \
    cudaError_t e_ = (x);                                                                             \
    if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));          \
  } while (0)
#define LAUNCH_CHECK(s) \
  do {                  \
    (s)->launches++;    \
    CK(cudaGetLastError()); \
  } while (0)

// Kernel launch on the handle's stream with programmatic stream serialisation (PDL; kernels.cu PDL_ENTRY): the
// kernel's grid may be scheduled while its predecessor runs and waits in griddepcontrol.wait for it, hiding launch
// latency and ramp between the many short dependent kernels of an iteration.  PD_PDL=0 launches
// plainly (same results: the wait is then a no-op).
inline bool pdl_enabled() {
  static const bool on = !(std::getenv("PD_PDL") && std::atoi(std::getenv("PD_PDL")) == 0);
  return on;
}
template <typename... KArgs, typename... Args>
void pdl_launch(pd_sim* s, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, Args&&... args) {
  cudaLaunchConfig_t c = {};
  c.gridDim = grid;
  c.blockDim = block;
  c.dynamicSmemBytes = smem;
  c.stream = s->stream;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  c.attrs = a;
  c.numAttrs = 1;
  CK(cudaLaunchKernelEx(&c, kernel, std::forward<Args>(args)...));
}

pd_status fail(pd_sim* s, pd_status st, const std::string& msg) {
  if (s) s->err = msg;
  else g_create_error = msg;
  return st;
}

cudaEvent_t prof_event(pd_sim* s) {
  if (s->ev_next == (int)s->ev_pool.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    s->ev_pool.push_back(e);
  }
  return s->ev_pool[s->ev_next++];
}
// NVTX range for the lifetime of a scope (phases: pd_forward / pd_backward, time step, inner solve, kernel family)
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};
const char* const kFamilyName[6] = {"local_K1", "gather_K2", "solve_K3", "AN_K4", "contact_K5", "param"};
struct ProfScope {
  pd_sim* s;
  int fam;
  bool on = false;
  Nvtx range;
  ProfScope(pd_sim* s_, int f) : s(s_), fam(f), range(kFamilyName[f]) {
    if (!s->opt.profile) return;
    on = s->prof_calls[fam]++ % s->prof_every == 0;  // a 1-in-prof_every sample of the family's scopes
    if (!on) return;
    s->ev_open.push_back({fam, s->ev_next});
    CK(cudaEventRecord(prof_event(s), s->stream));
  }
  ~ProfScope() {
    if (on) cudaEventRecord(prof_event(s), s->stream);
  }
};
// resolve recorded pairs (the stream must have been synchronised)
void prof_flush(pd_sim* s) {
  if (!s->opt.profile) return;
  // (after a poll the stream has passed the check kernel, hence every event recorded before it; the wait below
  // returns at once and only covers the driver's bookkeeping of the last event)
  if (!s->ev_open.empty()) CK(cudaEventSynchronize(s->ev_pool[s->ev_open.back().second + 1]));
  for (auto& pr : s->ev_open) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, s->ev_pool[pr.second], s->ev_pool[pr.second + 1]));
    s->prof_ms[pr.first] += ms;
    s->prof_cnt[pr.first] += 1;
  }
  s->ev_open.clear();
  s->ev_next = 0;
}

ElemArgs elem_args(pd_sim* s, int B, const double* act_step, int64_t act_bstride) {
  ElemArgs ea;
  ea.hex8 = s->d_hex8;
  ea.m = s->plan.m;
  ea.B = B;
  ea.w_sim = s->w_cur ? s->w_cur : s->w_sim;
  ea.act = act_step;
  ea.act_bstride = act_bstride;
  ea.fib = s->d_fib;
  return ea;
}

// per-sim dot products of state-layout vectors of length len (*B) -> s->dots[p*B + b]
void dots(pd_sim* s, int B, int64_t len, std::initializer_list<std::pair<const double*, const double*>> pairs,
          double* out = nullptr, int accumulate = 0) {
  DotArgs da{};
  int p = 0;
  for (auto& pr : pairs) {
    da.u[p] = pr.first;
    da.v[p] = pr.second;
    ++p;
  }
  da.npairs = p;
  const int nchunk = red_chunks(len);
  pdl_launch(s, k_dot_partial, dim3(nchunk, red_groups(B)), red_threads(B), 0, da, len, B, s->partial);
  LAUNCH_CHECK(s);
  pdl_launch(s, k_dot_final, p * B, 128, 0, s->partial, nchunk, B, p, out ? out : s->dots, accumulate);
  LAUNCH_CHECK(s);
}

// ABI <-> state conversions at the library boundary; with a general contact plane they also change coordinates
// (kind 1: positions, 2: vectors; kind 0: no coordinates, e.g. scalars per DoF).  Without a plane the plain
// layout kernels run (bitwise the default path).
void abi_in(pd_sim* s, const double* in, double* out, int B, int64_t bstride, int kind) {
  const int n3 = 3 * s->plan.n;
  if (s->frame && kind) {
    pdl_launch(s, k_abi_to_state_frame, nblk((int64_t)s->plan.n * B), 256, 0, in, out, s->plan.n, B, bstride, s->fq,
                                                                            kind == 1);
  } else {
    pdl_launch(s, k_abi_to_state, nblk((int64_t)n3 * B), 256, 0, in, out, n3, B, bstride);
  }
  LAUNCH_CHECK(s);
}
void abi_out(pd_sim* s, const double* in, double* out, int B, int64_t bstride, int kind) {
  const int n3 = 3 * s->plan.n;
  if (s->frame && kind) {
    pdl_launch(s, k_state_to_abi_frame, nblk((int64_t)s->plan.n * B), 256, 0, in, out, s->plan.n, B, bstride, s->fq,
                                                                            kind == 1);
  } else {
    pdl_launch(s, k_state_to_abi, nblk((int64_t)n3 * B), 256, 0, in, out, n3, B, bstride);
  }
  LAUNCH_CHECK(s);
}
void abi_add(pd_sim* s, double* out, const double* in, int B, int64_t bstride) {  // vectors, non-Dirichlet nodes
  const int n3 = 3 * s->plan.n;
  if (s->frame) {
    pdl_launch(s, k_add_abi_frame, nblk((int64_t)s->plan.n * B), 256, 0, out, in, s->plan.n, B, bstride, s->d_fixed,
                                                                       s->fq);
  } else {
    pdl_launch(s, k_add_abi, nblk((int64_t)n3 * B), 256, 0, out, in, n3, B, bstride, s->d_fixed);
  }
  LAUNCH_CHECK(s);
}

// x = A^{-1} rhs in solve layout: S0 = rhs (consumed as the working z), S2 = y, S0 = x out
template <int RC, bool VEC>
void solve_rc(pd_sim* s, int B) {  // (contact fixup of the root block when s->pins_live)
  const HostPlan& P = s->plan;
  const int R = 3 * B;
  const unsigned gy = (unsigned)((R + RC - 1) / RC);
  if (gy > (unsigned)kGY) throw CudaError("batch too large for the solve's column chunking");
  int nsm = 0, dev = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  // each item buffer also holds the 4 padded warp tiles of a chain's epilogue
  auto kpad_of = [&](int kmax) { return std::max(kmax, (4 * 32 * tile_ld<RC>() + 32 + RC - 1) / (32 + RC)); };
  // programmatic dependent launch (PDL): a kernel's CTAs may be scheduled while its predecessor drains;
  // they block in griddepcontrol.wait until the predecessor's writes are visible
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  auto cfg_of = [&](dim3 grid, dim3 block, size_t smem) {
    cudaLaunchConfig_t c = {};
    c.gridDim = grid;
    c.blockDim = block;
    c.dynamicSmemBytes = smem;
    c.stream = s->stream;
    c.attrs = pdl;
    c.numAttrs = 1;
    return c;
  };
  auto* const level_fn = s->k3_mma ? k_sweep_level<RC, VEC, true> : k_sweep_level<RC, VEC, false>;
  CK(cudaFuncSetAttribute(level_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448 - 1024));
  auto resident_lvl = [&](int bytes) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, level_fn, 128, bytes));
    return std::max(1, per_sm) * (int64_t)nsm;
  };
  // forward: sources z (S0), direct y (S2), reduce: y (S2) / z -= (S0);
  // backward: D part y (S2), W part x (S0), direct x (S0)
  auto level = [&](const HostPlan::Sweep& S, const SweepDev& d, bool fwd, int j) {
    const int ch0 = S.lvl_chain[j], nch = S.lvl_chain[j + 1] - ch0;
    if (nch > 0) {
      const int kp = kpad_of(S.lvl_kmax[j]);
      // ring depth (default 2: 2 buffers x several CTAs/SM), clamped to what fits the shared-memory opt-in limit
      const int nbuf = std::max(2, std::min(s->k3_nbuf, (232448 - 1024) / (kp * (32 + RC) * 8)));
      const int smem = nbuf * kp * (32 + RC) * 8;
      const unsigned gx = (unsigned)std::min<int64_t>(nch, std::max<int64_t>(1, resident_lvl(smem) / gy));
      cudaLaunchConfig_t c = cfg_of(dim3(gx, gy), dim3(128), smem);
      CK(cudaLaunchKernelEx(&c, level_fn, d, ch0, nch, R, (const double*)(fwd ? s->S0 : s->S2), (const double*)s->S0,
                            (const int32_t*)s->d_rows, fwd ? s->S2 : s->S0, s->Spart, kp, nbuf));
      LAUNCH_CHECK(s);
    }
    const int r0 = S.lvl_red[j], nr = S.lvl_red[j + 1] - r0;
    if (nr > 0) {
      cudaLaunchConfig_t c = cfg_of(dim3(nblk((int64_t)nr * R)), dim3(256), 0);
      CK(cudaLaunchKernelEx(&c, k_sweep_reduce, d, r0, nr, R, (const double*)s->Spart, fwd ? s->S2 : s->S0, s->S0));
      LAUNCH_CHECK(s);
    }
  };
  for (int j = 0; j < P.nlevels; ++j) level(P.fw, s->swf, true, j);
  if (s->pins_live) {
    // the root (= candidate block) first, then its constrained fixup, then every other level
    double* root = s->S0 + (int64_t)s->csup_first * R;
    CK(cudaMemcpyAsync(s->Rsave, root, sizeof(double) * (int64_t)s->nc * R, cudaMemcpyDeviceToDevice, s->stream));
    level(P.bw, s->swb, false, 0);
    pdl_launch(s, k_contact_fix, dim3((s->nc + 7) / 8, (s->sticky ? 3 : 1) * B), 256, 0, 
        s->Rsave, s->nc, R, B, s->kcount, s->flist, s->fpos, s->Qc, root);
    LAUNCH_CHECK(s);
    for (int j = 1; j < P.nlevels; ++j) level(P.bw, s->swb, false, j);
  } else {
    for (int j = 0; j < P.nlevels; ++j) level(P.bw, s->swb, false, j);
  }
}
// K3 v4: one k_sweep_warp launch per level and sweep (warps stream equal k-group ranges) plus
// the level's reduce when it has partial slots; chained with programmatic dependent launch.
template <int NT, bool VEC>
void solve_v4(pd_sim* s, int B) {
  const HostPlan& P = s->plan;
  const int R = 3 * B;
  constexpr int RC = 8 * NT;
  const unsigned gy = (unsigned)((R + RC - 1) / RC);
  const int smem = kWarpsK3 * kStages * stage_doubles<NT>() * 8;
  auto* const fn = k_sweep_warp<NT, VEC>;
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  auto cfg_of = [&](dim3 grid, dim3 block, size_t sm) {
    cudaLaunchConfig_t c = {};
    c.gridDim = grid;
    c.blockDim = block;
    c.dynamicSmemBytes = sm;
    c.stream = s->stream;
    c.attrs = pdl;
    c.numAttrs = 1;
    return c;
  };
  // forward: sources z (S0), direct y (S2), reduce: y (S2) = / z (S0) -= ; backward: sources y (S2) and x (S0),
  // direct x (S0), reduce x (S0) =
  // timing experiments only (wrong results): PD_K3_EXP=1 skips the reduces, 2 skips the level kernels
  static const int exp_mode = std::getenv("PD_K3_EXP") ? std::atoi(std::getenv("PD_K3_EXP")) : 0;
  // The level's nw warp ranges are fixed by the plan (independent of B, so a sim's result does not depend on the
  // batch it runs in); with gy column chunks a physical warp streams vpw consecutive ranges (one
  // contiguous span of the stream, same pieces and partial slots, bitwise the same result) so that the launch's
  // gy x ceil(nw / vpw / kWarpsK3) CTAs fit one wave (c3, gy = 8: A^-1 119 -> 108 us measured)
  const int wcap = std::max(1, s->nsm / (int)gy) * kWarpsK3;
  auto level = [&](const HostPlan::Sweep4& S, const Sweep4Dev& d, bool fwd, int j) {
    const int w0 = S.lvl_warp[j], nw = S.lvl_warp[j + 1] - w0 - 1;
    if (exp_mode != 2 && S.lvl_g[j + 1] > S.lvl_g[j]) {  // (the forward sweep's merged root level is empty)
    const int vpw = (nw + wcap - 1) / wcap, nphys = (nw + vpw - 1) / vpw;
    cudaLaunchConfig_t c = cfg_of(dim3((unsigned)((nphys + kWarpsK3 - 1) / kWarpsK3), gy), dim3(32 * kWarpsK3), smem);
    CK(cudaLaunchKernelEx(&c, fn, d, w0, nw, vpw, R, (const double*)(fwd ? s->S0 : s->S2), (const double*)s->S0,
                          fwd ? s->S2 : s->S0, s->Spart));
    LAUNCH_CHECK(s);
    }
    const int r0 = S.lvl_red[j], nr = S.lvl_red[j + 1] - r0;
    if (nr > 0 && exp_mode != 1) {
      cudaLaunchConfig_t c2 = cfg_of(dim3(nblk((int64_t)nr * R)), dim3(256), 0);
      CK(cudaLaunchKernelEx(&c2, k_sweep_reduce4<8>, d, r0, nr, R, (const double*)s->Spart, fwd ? s->S2 : s->S0,
                            s->S0));
      LAUNCH_CHECK(s);
    }
  };
  for (int j = 0; j < P.nlevels; ++j) level(P.fw4, s->sw4f, true, j);
  if (s->pins_live) {
    double* root = s->S0 + (int64_t)s->csup_first * R;
    CK(cudaMemcpyAsync(s->Rsave, root, sizeof(double) * (int64_t)s->nc * R, cudaMemcpyDeviceToDevice, s->stream));
    level(P.bw4, s->sw4b, false, 0);
    pdl_launch(s, k_contact_fix, dim3((s->nc + 7) / 8, (s->sticky ? 3 : 1) * B), 256, 0, 
        s->Rsave, s->nc, R, B, s->kcount, s->flist, s->fpos, s->Qc, root);
    LAUNCH_CHECK(s);
    for (int j = 1; j < P.nlevels; ++j) level(P.bw4, s->sw4b, false, j);
  } else {
    for (int j = 0; j < P.nlevels; ++j) level(P.bw4, s->sw4b, false, j);
  }
}

void solve_launch(pd_sim* s, int B) {
  const int R = 3 * B;
  if (s->plan.k3_version == 4) {
    if (R <= 8) (R % 2 == 0) ? solve_v4<1, true>(s, B) : solve_v4<1, false>(s, B);
    else (R % 2 == 0) ? solve_v4<3, true>(s, B) : solve_v4<3, false>(s, B);
    return;
  }
  if (R <= 4) solve_rc<4, false>(s, B);
  else if (R <= 8) (R % 2 == 0) ? solve_rc<8, true>(s, B) : solve_rc<8, false>(s, B);
  else if (R <= 24) (R % 2 == 0) ? solve_rc<24, true>(s, B) : solve_rc<24, false>(s, B);
  else (R % 2 == 0) ? solve_rc<48, true>(s, B) : solve_rc<48, false>(s, B);
}
// The whole two-sweep solve (≈ 2 x levels kernels) is captured once per (B, contact fixup) as a CUDA
// graph and replayed: one launch per A^{-1} application.
void solve(pd_sim* s, int B) {
  const int key = 2 * B + (s->pins_live ? 1 : 0);
  auto it = s->solve_graphs.find(key);
  if (it == s->solve_graphs.end()) {
    cudaGraph_t g;
    const int64_t l0 = s->launches;
    if (!s->cap_stream) CK(cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking));
    cudaStream_t user = s->stream;
    s->stream = s->cap_stream;  // capture on a private stream (the caller's may be the legacy stream)
    CK(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
    try {
      solve_launch(s, B);
    } catch (...) {
      cudaStreamEndCapture(s->stream, &g);
      s->stream = user;
      throw;
    }
    s->stream = user;
    CK(cudaStreamEndCapture(s->cap_stream, &g));
    cudaGraphExec_t ge;
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphDestroy(g));
    it = s->solve_graphs.emplace(key, std::make_pair(ge, s->launches - l0)).first;
    s->launches = l0;
  }
  CK(cudaGraphLaunch(it->second.first, s->stream));
  s->launches += it->second.second;
}

// state vector V (free nodes) -> A^{-1} V -> OUT = beta OUT + alpha_c*alpha[b]*sol (masked)
// (Vin = nullptr: the right-hand side is already in S0 in the solve layout)
void apply_Ainv(pd_sim* s, int B, const double* Vin, double* OUT, const double* alpha, double alpha_c, double beta,
                const int32_t* active) {
  const HostPlan& P = s->plan;
  ProfScope ps(s, 2);
  if (Vin) {
    pdl_launch(s, k_to_solve, nblk((int64_t)P.nfree * 3 * B), 256, 0, Vin, s->d_nodepos, P.nfree, B, s->S0);
    LAUNCH_CHECK(s);
  }
  solve(s, B);
  pdl_launch(s, k_from_solve, nblk((int64_t)3 * P.n * B), 256, 0, s->S0, s->d_pos, P.n, B, alpha, alpha_c, beta,
                                                                   active, OUT);
  LAUNCH_CHECK(s);
}

// grad g(X) into G (+ W normaliser, S0 permuted RHS), element energies in EE
void residual(pd_sim* s, int B, const double* X, const double* Y, const double* act_step, int64_t act_bstride,
              const uint8_t* fixed_mask, double* Gout = nullptr) {
  const HostPlan& P = s->plan;
  {
    ProfScope ps(s, 0);
    pdl_launch(s, s->d_fib ? k_elem_residual<true> : k_elem_residual<false>, nblk((int64_t)P.m * B * 8, 256), 256, 0, X, s->st, elem_args(s, B, act_step, act_bstride),
                                                                         s->EF, s->EE);
    LAUNCH_CHECK(s);
    if (s->st.kappa != 0.0) {  // volume-preserving term added to the element forces and energies
      pdl_launch(s, k_vol<0>, nblk((int64_t)P.m * B * 8, 256), 256, 0, X, nullptr, s->st,
                                                                      elem_args(s, B, act_step, act_bstride), nullptr,
                                                                      s->EF, s->EE);
      LAUNCH_CHECK(s);
    }
  }
  ProfScope ps(s, 1);
  const bool pin = s->pins_live;
  pdl_launch(s, k_gather, nblk((int64_t)P.n * B), 256, 0, X, Y, s->EF, s->d_mass, s->d_inc_ptr, s->d_inc_ec, fixed_mask,
                                                          s->d_pos, P.n, B, 1.0 / (s->h * s->h), 0, Gout ? Gout : s->G,
                                                          s->W, s->S0,
                                                          pin ? s->d_cand_of_node : nullptr, pin ? s->PIN : nullptr,
                                                          pin ? s->LAM : nullptr, s->sticky);
  LAUNCH_CHECK(s);
}

// OUT = A_N(X) Pin, zero on constrained DoFs.  jc: per-step Jacobian cache of X (k_elem_jac) or null.
void apply_AN(pd_sim* s, int B, const double* X, const double* Pin, double* OUT, const double* act_step,
              int64_t act_bstride, const double* jc = nullptr) {
  const HostPlan& P = s->plan;
  ProfScope ps(s, 3);
  if (jc)
    pdl_launch(s, k_elem_AN_cached, nblk((int64_t)P.m * B * 8, 256), 256, 0, 
        Pin, s->st, elem_args(s, B, act_step, act_bstride), jc, s->EF);
  else
    pdl_launch(s, k_elem_AN, nblk((int64_t)P.m * B * 8, 256), 256, 0, X, Pin, s->st,
                                                                   elem_args(s, B, act_step, act_bstride), s->EF);
  LAUNCH_CHECK(s);
  if (s->st.kappa != 0.0) {
    if (jc)
      pdl_launch(s, k_vol<1>, nblk((int64_t)P.m * B * 8, 256), 256, 0, nullptr, Pin, s->st,
                                                                      elem_args(s, B, act_step, act_bstride),
                                                                      const_cast<double*>(jc), s->EF, nullptr);
    else
      pdl_launch(s, k_vol<2>, nblk((int64_t)P.m * B * 8, 256), 256, 0, X, Pin, s->st,
                                                                      elem_args(s, B, act_step, act_bstride), nullptr,
                                                                      s->EF, nullptr);
    LAUNCH_CHECK(s);
  }
  const bool pin = s->pins_live;
  pdl_launch(s, k_gather, nblk((int64_t)P.n * B), 256, 0, Pin, nullptr, s->EF, s->d_mass, s->d_inc_ptr, s->d_inc_ec,
                                                          s->d_fixed, s->d_pos, P.n, B, 1.0 / (s->h * s->h), 1, OUT,
                                                          nullptr, nullptr, pin ? s->d_cand_of_node : nullptr,
                                                          pin ? s->PIN : nullptr, nullptr, s->sticky);
  LAUNCH_CHECK(s);
}

// w = E/(1+nu) per sim into the forward's w_sim / youngs_sim (diag = false: youngs_sim keeps E for
// dL/dE, dL/dnu of the following pd_backward) or into the diagnostic hooks' own scratch (diag = true)
void set_w(pd_sim* s, int B, const double* youngs_per_sim, bool diag = false) {
  double* E = diag ? s->youngs_diag : s->youngs_sim;
  double* w = diag ? s->w_diag : s->w_sim;
  std::vector<double> ones(B, s->youngs);
  if (youngs_per_sim)
    CK(cudaMemcpyAsync(E, youngs_per_sim, B * sizeof(double), cudaMemcpyDeviceToDevice, s->stream));
  else
    CK(cudaMemcpyAsync(E, ones.data(), B * sizeof(double), cudaMemcpyHostToDevice, s->stream));
  pdl_launch(s, k_axpby, 1, 256, 0, w, E, 1.0 / (1.0 + s->poisson), nullptr, nullptr, 0.0, B, B, nullptr);
  LAUNCH_CHECK(s);
  CK(cudaStreamSynchronize(s->stream));
  s->w_cur = w;
}

// Iteration control without a stream synchronisation: the check kernel whose result the host
// needs next is handed a fresh sequence number (flag_args) and publishes the three loop counters
// ([0] the last k_ls_accept / k_adj_check / plain-PD k_fwd_check count, [1] the L-BFGS / Newton running count,
// [2] running sims already within 16 tol) into the mapped pinned triple followed by that number (kernels.cu
// publish3); the host spins on the number (wait_flags).  The GPU is idle only for the PCIe write and the next
// launch, not for a D2H copy operation plus the wake-up of a blocked thread.  PD_POLL=0 restores the copy + sync.
struct FlagArgs {
  int32_t* hflag;
  const int32_t* nact3;
  int seq;
};
// arguments for a check kernel whose counters the host reads next (want = false: nothing is published)
FlagArgs flag_args(pd_sim* s, bool want = true) {
  if (!want || !s->poll) return {nullptr, nullptr, 0};
  if (++s->flag_seq == 0x7fffffff) s->flag_seq = 1;
  return {s->h_nactive, s->nactive, s->flag_seq};
}
void wait_flags(pd_sim* s, int nread) {
  if (!s->poll) {
    CK(cudaMemcpyAsync(s->h_nactive, s->nactive, nread * sizeof(int32_t), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    prof_flush(s);
    return;
  }
  volatile int32_t* h = s->h_nactive;
  const int32_t seq = s->flag_seq;
  for (uint64_t spin = 1; h[3] != seq; ++spin) {
    if ((spin & 0x3fff) == 0) {  // a failed kernel never publishes: surface its error instead of spinning
      const cudaError_t e = cudaStreamQuery(s->stream);
      if (e == cudaSuccess) {
        if (h[3] != seq) throw CudaError("iteration control: the check kernel finished without publishing");
      } else if (e != cudaErrorNotReady) {
        throw CudaError(std::string("iteration control: ") + cudaGetErrorString(e));
      }
    }
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  prof_flush(s);
}
void read_nactive3(pd_sim* s, int* a, int* b, int* c) {
  wait_flags(s, 3);
  *a = s->h_nactive[0];
  *b = s->h_nactive[1];
  *c = s->h_nactive[2];
}
int read_nactive(pd_sim* s) {
  wait_flags(s, 1);
  return *s->h_nactive;
}

// out[j*B + b] = <u_b, V_j,b> for j < nv, V_j = Vbase + j * (3n B)   (deterministic, 2 launches);
// with u2: out[(nv + j)*B + b] = <u2_b, V2_j,b> in the same pass
void mdot(pd_sim* s, int B, const double* u, const double* Vbase, int nv, double* out, const double* u2 = nullptr,
          const double* V2base = nullptr) {
  const int64_t n3 = 3LL * s->plan.n;
  const int nchunk = red_chunks(n3);
  const int np = u2 ? 2 * nv : nv;
  pdl_launch(s, k_mdot_partial, dim3(nchunk, np, red_groups(B)), red_threads(B), 0, u, Vbase, n3 * B, nv, n3, B,
                                                                                    s->partial, u2, V2base);
  LAUNCH_CHECK(s);
  pdl_launch(s, k_dot_final, np * B, 128, 0, s->partial, nchunk, B, np, out, 0);
  LAUNCH_CHECK(s);
}

// objective g (eq:opt) and its gradient at X: Gout = grad g (constrained rows 0), and either
// fout[b] = g (with_f) or, for line-search trials, the parts inert[b] = sum m/h^2 |x - y|^2,
// esum[b] = sum of element energies and inert[B + b] = |grad g|^2 (k_ls_accept forms g)
void eval_f(pd_sim* s, int B, const double* X, double* Gout, double* fout, const double* act_step, int64_t act_bs,
            bool with_gn2 = false) {
  const HostPlan& P = s->plan;
  residual(s, B, X, s->Y, act_step, act_bs, s->d_fixed, Gout);
  const int64_t n3 = 3LL * P.n;
  const int nchunk = red_chunks(n3);
  const int np = with_gn2 ? 2 : 1;
  pdl_launch(s, k_inertia_partial, dim3(nchunk, red_groups(B)), red_threads(B), 0, 
      X, s->Y, s->d_mass, 1.0 / (s->h * s->h), n3, B, s->partial, with_gn2 ? Gout : nullptr);
  LAUNCH_CHECK(s);
  pdl_launch(s, k_dot_final, np * B, 128, 0, s->partial, nchunk, B, np, s->inert, 0);
  LAUNCH_CHECK(s);
  dots(s, B, P.m, {{s->EE, nullptr}}, s->esum);
  if (fout) {
    pdl_launch(s, k_obj_combine, nblk(B, 64), 64, 0, s->inert, s->esum, fout, B);
    LAUNCH_CHECK(s);
  }
}

// zero Dirichlet nodes and (when pins are live) the pinned z DoFs of a state vector
void zero_constrained(pd_sim* s, double* Y, int B) {
  const bool pin = s->pins_live;
  pdl_launch(s, k_zero_constrained, nblk((int64_t)3 * s->plan.n * B), 256, 0, 
      Y, s->d_fixed, s->plan.n, B, pin ? s->d_cand_of_node : nullptr, pin ? s->PIN : nullptr, s->sticky);
  LAUNCH_CHECK(s);
}

// zero Dirichlet nodes only
void zero_constrained_fixed(pd_sim* s, double* Y, int B) {
  pdl_launch(s, k_zero_constrained, nblk((int64_t)3 * s->plan.n * B), 256, 0, Y, s->d_fixed, s->plan.n, B, nullptr,
                                                                              nullptr, 0);
  LAUNCH_CHECK(s);
}

// Q_b = (S_ff)^{-1} for the current PIN of the sims in sel (device [B] or null = all): free list,
// gather, blocked Gauss-Jordan.  One host sync (kcount) per call.
void build_Q(pd_sim* s, int B, const int32_t* sel) {
  ProfScope ps(s, 4);
  const int c = s->nc;
  pdl_launch(s, k_contact_flist, B, 1024, 0, s->PIN, s->d_cand_of_loc, c, B, sel, s->flist, s->fpos, s->kcount);
  LAUNCH_CHECK(s);
  std::vector<int32_t> selh(B, 1);
  if (sel) CK(cudaMemcpyAsync(s->h_small + B, sel, B * sizeof(int32_t), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaMemcpyAsync(s->h_small, s->kcount, B * sizeof(int32_t), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  int kmax = 0;
  for (int b = 0; b < B; ++b) {
    const int k = s->h_small[b];
    const bool want = (!sel || s->h_small[B + b]) && k > 0 && k < c;
    selh[b] = want ? 1 : 0;
    if (want) kmax = std::max(kmax, k);
  }
  if (kmax == 0) return;
  CK(cudaMemcpyAsync(s->need, selh.data(), B * sizeof(int32_t), cudaMemcpyHostToDevice, s->stream));
  const int nt = (kmax + 31) / 32;
  pdl_launch(s, k_contact_gather_S, dim3(nt, (kmax + 7) / 8, B), dim3(32, 8), 0, s->d_S, c, s->need, s->flist,
                                                                                 s->kcount, s->Qc);
  LAUNCH_CHECK(s);
  for (int kb = 0; kb < nt; ++kb) {
    pdl_launch(s, k_gj_pivot, B, 256, 0, s->Qc, c, kb, s->need, s->kcount, s->PIc);
    LAUNCH_CHECK(s);
    pdl_launch(s, k_gj_panel, dim3((kmax + 63) / 64, B), 256, 0, s->Qc, c, kb, s->need, s->kcount, s->PIc, s->Cb,
                                                                 s->Mb, s->Rb);
    LAUNCH_CHECK(s);
    pdl_launch(s, k_gj_update, dim3(nt, nt, B), 256, 0, s->Qc, c, kb, s->need, s->kcount, s->PIc, s->Mb, s->Rb);
    LAUNCH_CHECK(s);
  }
}

// Forward quasi-Newton PD (P:79, P:254-271 applied to eq:opt): L-BFGS on g with H0 = A^{-1} (the
// constrained prefactorised solve) and Armijo backtracking; per-sim masks; history slots shared by index.
void inner_lbfgs(pd_sim* s, int B, int i, const double* act_i, int64_t act_bs, const int32_t* it_base, bool warm) {
  Nvtx nv("inner_lbfgs");
  const HostPlan& P = s->plan;
  const int n3 = 3 * P.n;
  const int64_t len = (int64_t)n3 * B;
  const int m = s->nhist;
  const int max_trial = 30;
  auto LSs = [&](int k) { return s->LS + (int64_t)k * len; };
  auto LYs = [&](int k) { return s->LY + (int64_t)k * len; };
  CK(cudaMemcpyAsync(s->Xn, s->X, len * sizeof(double), cudaMemcpyDeviceToDevice, s->stream));
  eval_f(s, B, s->X, s->G, s->fcur, act_i, act_bs);
  // dots[0:B] = |grad g|^2 (refreshed from each accepted trial by k_gram_store), dots[B:2B] = |W|^2 (W depends
  // on y only: constant over the solve)
  dots(s, B, n3, {{s->G, s->G}, {s->W, s->W}});
  double* const gn2 = s->inert + B;  // |grad g(x_trial)|^2, from eval_f
  // ring position gi (slot of the next pair = gi % m) and valid pairs; kept across the Alg. 1 outer iterations
  // of a step when warm (lbfgs_warm): the pairs are restricted to the new free DoFs and their Gram matrix and
  // rho recomputed (pairs with s^T y <= 0 drop out through rho = 0)
  int hist = warm ? s->lb_hist : 0;
  const int gi0 = warm ? s->lb_gi : 0;
  if (hist > 0) {
    for (int j = 0; j < hist; ++j) {
      zero_constrained(s, LSs(j), B);
      zero_constrained(s, LYs(j), B);
    }
    for (int j = 0; j < hist; ++j) {
      mdot(s, B, LSs(j), s->LY, hist, s->lb_da, LYs(j), s->LS);
      pdl_launch(s, k_gram_store, nblk(B, 64), 64, 0, s->lb_G, s->rho_h, s->lb_da, s->lb_da + (int64_t)hist * B, j, m,
                                                      hist, B, s->active, nullptr, nullptr, nullptr, nullptr, nullptr,
                                                      nullptr, nullptr);
      LAUNCH_CHECK(s);
    }
  }
  int gi = gi0;
  const bool fuse = s->fuse;
  bool done = false, check_now = true;  // the first check of a solve is read immediately
  for (int iter = 0;; ++iter, ++gi) {
    // convergence check; also alpha = 1 and ls_act = active for the coming line search
    // Far from convergence the convergence count is read together with the first line-search decision (one
    // host sync per iteration instead of two; were every sim to converge meanwhile, the direction and trial
    // launched after the check are fully masked and the loop ends at that sync).  Once a running sim is within
    // 16 tol the check is read immediately, so no masked iteration is spent at the end of a solve.
    const FlagArgs fc = flag_args(s, check_now && iter < s->opt.max_iter_fwd);
    pdl_launch(s, k_fwd_check, 1, 256, 0, s->dots, B, s->opt.tol_fwd, iter, 0, s->opt.max_iter_fwd, s->active,
                                          s->st_iters_f + (int64_t)i * B, s->st_res_f + (int64_t)i * B,
                                          s->st_flag_f + (int64_t)i * B, s->nactive + 1, it_base, s->alpha_ls,
                                          s->ls_act, s->nactive + 2, fc.hflag, fc.nact3, fc.seq);
    LAUNCH_CHECK(s);
    if (iter >= s->opt.max_iter_fwd) break;
    if (check_now) {
      int a = 0, running = 0, nr = 0;
      read_nactive3(s, &a, &running, &nr);
      if (running == 0) break;
    }
    // D = -H grad g, compact two-loop (k_lbfgs_alpha / k_lbfgs_beta): 2 multi-dots + 2 multi-axpys + A^{-1}
    bool trial0_done = false;
    if (hist > 0) {
      mdot(s, B, s->G, s->LS, hist, s->lb_sg);
      pdl_launch(s, k_lbfgs_alpha, B, 32, 0, s->lb_sg, s->lb_G, s->rho_h, s->aj_h, m, hist, gi, B, s->active);
      LAUNCH_CHECK(s);
      // q = g - sum alpha_j y_j, written in the solve layout (fused k_to_solve; PD_FUSE=0: two passes)
      if (fuse)
        pdl_launch(s, k_multi_axpy_solve, nblk((int64_t)P.nfree * 3 * B), 256, 0, s->S0, s->G, 1.0, -1.0, s->LY, len,
                                                             s->aj_h, nullptr, hist, P.nfree, B, s->active, s->d_nodepos);
      else
        pdl_launch(s, k_multi_axpy, nblk(len), 256, 0, s->Dv, s->G, 1.0, -1.0, s->LY, len, s->aj_h, nullptr, hist, len, B,
                                                       s->active, nullptr, nullptr, nullptr);
      LAUNCH_CHECK(s);
    } else {
      CK(cudaMemcpyAsync(s->Dv, s->G, len * sizeof(double), cudaMemcpyDeviceToDevice, s->stream));
    }
    // r0 = H0 q = A^{-1} q
    apply_Ainv(s, B, (hist > 0 && fuse) ? nullptr : s->Dv, s->Dv, s->lb_gamma ? s->gamma : nullptr, 1.0, 0.0, s->active);
    if (hist > 0) {
      mdot(s, B, s->Dv, s->LY, hist, s->lb_yr);
      pdl_launch(s, k_lbfgs_beta, B, 32, 0, s->lb_yr, s->lb_G, s->rho_h, s->aj_h, s->lb_beta, m, hist, gi, B,
                                                      s->active);
      LAUNCH_CHECK(s);
      // d = -(r0 + sum (alpha_j - beta_j) s_j); fused: also the first trial point x + alpha d (alpha = 1, ls_act =
      // active from k_fwd_check)
      pdl_launch(s, k_multi_axpy, nblk(len), 256, 0, s->Dv, s->Dv, -1.0, 1.0, s->LS, len, s->aj_h, s->lb_beta, hist, len,
                                                     B, s->active, fuse ? s->Xn : nullptr, s->X, s->alpha_ls);
      LAUNCH_CHECK(s);
      trial0_done = fuse;
    } else {
      pdl_launch(s, k_axpby, nblk(len), 256, 0, s->Dv, s->Dv, -1.0, nullptr, nullptr, 0.0, len, B, s->active);
      LAUNCH_CHECK(s);
    }
    dots(s, B, n3, {{s->G, s->Dv}}, s->gtd);
    // Armijo backtracking from alpha = 1 (set by k_fwd_check); g_new and the decision in k_ls_accept
    for (int trial = 0;; ++trial) {
      if (!(trial == 0 && trial0_done)) {
        pdl_launch(s, k_axpby, nblk(len), 256, 0, s->Xn, s->X, 1.0, s->Dv, s->alpha_ls, 1.0, len, B, s->ls_act);
        LAUNCH_CHECK(s);
      }
      eval_f(s, B, s->Xn, s->Gn, nullptr, act_i, act_bs, true);
      const FlagArgs fl = flag_args(s);
      pdl_launch(s, k_ls_accept, 1, 256, 0, s->fcur, s->fnew, s->inert, s->esum, s->gtd, s->dots, gn2, s->alpha_ls,
                                            s->ls_act, trial, max_trial, s->nactive, s->ls_flag, B, fl.hflag, fl.nact3,
                                            fl.seq);
      LAUNCH_CHECK(s);
      int searching = 0, running = 1, nr = 0;
      read_nactive3(s, &searching, &running, &nr);
      if (trial == 0) {
        if (running == 0) {
          done = true;
          break;
        }
        check_now = nr > 0;
      }
      if (searching == 0) break;
    }
    if (done) break;
    // curvature pair (s, y) into slot iter % m and commit x, grad g (one pass); Gram row/column of the new
    // pair (both multi-dots in one pass); f, |grad g|^2
    const int slot = gi % m;
    pdl_launch(s, k_lbfgs_commit, nblk(len), 256, 0, LSs(slot), LYs(slot), s->X, s->G, s->Xn, s->Gn, len, B, s->active);
    LAUNCH_CHECK(s);
    const int nv = std::min(hist + 1, m);  // valid slots after this store are [0, nv)
    mdot(s, B, LSs(slot), s->LY, nv, s->lb_da, LYs(slot), s->LS);  // s_new^T y_j | y_new^T s_j
    const bool set_gamma = s->lb_gamma && hist == 0;  // (first step of a solve: d = -gamma A^{-1} grad g exactly)
    pdl_launch(s, k_gram_store, nblk(B, 64), 64, 0, s->lb_G, s->rho_h, s->lb_da, s->lb_da + (int64_t)nv * B, slot, m, nv,
                                                    B, s->active, s->fcur, s->fnew, s->dots, gn2,
                                                    set_gamma ? s->gamma : nullptr, s->alpha_ls, s->gtd);
    LAUNCH_CHECK(s);
    hist = nv;
  }
  s->lb_hist = hist;
  s->lb_gi = gi;
}

// Newton-PCG forward (accel_fwd = 2, the paper's Newton baseline of P:522-527 with an iterative
// linear solver): per iteration the projection-derivative data at x (k_elem_jac), a truncated CG on the Hessian
// A_N(x) D = -grad g preconditioned by the constrained A^{-1} (the adjoint's K4 + K3 machinery) to the relative
// residual newton_eta, a descent guard (PD direction -A^{-1} grad g where CG met negative curvature first) and the
// Armijo search of the L-BFGS path.  Same minimiser, same convergence test.
void inner_newton(pd_sim* s, int B, int i, const double* act_i, int64_t act_bs, const int32_t* it_base) {
  Nvtx nv("inner_newton_pcg");
  const HostPlan& P = s->plan;
  const int n3 = 3 * P.n;
  const int64_t len = (int64_t)n3 * B;
  const int max_trial = 30;
  double* const Z0 = s->LS;  // (no curvature history in this mode)
  CK(cudaMemcpyAsync(s->Xn, s->X, len * sizeof(double), cudaMemcpyDeviceToDevice, s->stream));
  eval_f(s, B, s->X, s->G, s->fcur, act_i, act_bs);
  dots(s, B, n3, {{s->G, s->G}, {s->W, s->W}});
  double* const gn2 = s->inert + B;
  for (int iter = 0;; ++iter) {
    const FlagArgs fc = flag_args(s, iter < s->opt.max_iter_fwd);
    pdl_launch(s, k_fwd_check, 1, 256, 0, s->dots, B, s->opt.tol_fwd, iter, 0, s->opt.max_iter_fwd, s->active,
                                          s->st_iters_f + (int64_t)i * B, s->st_res_f + (int64_t)i * B,
                                          s->st_flag_f + (int64_t)i * B, s->nactive + 1, it_base, s->alpha_ls,
                                          s->ls_act, s->nactive + 2, fc.hflag, fc.nact3, fc.seq);
    LAUNCH_CHECK(s);
    if (iter >= s->opt.max_iter_fwd) break;
    {
      int a = 0, running = 0, nr = 0;
      read_nactive3(s, &a, &running, &nr);
      if (running == 0) break;
    }
    {  // Hessian data at x (P:228's per-step Jacobian, here per Newton iteration)
      ProfScope ps(s, 3);
      pdl_launch(s, k_elem_jac, nblk((int64_t)P.m * B * 8, 256), 256, 0, s->X, s->st, elem_args(s, B, act_i, act_bs),
                                                                       s->JC);
      LAUNCH_CHECK(s);
      if (s->st.kappa != 0.0) {
        pdl_launch(s, k_vol<3>, nblk((int64_t)P.m * B * 8, 256), 256, 0, s->X, nullptr, s->st,
                                                                        elem_args(s, B, act_i, act_bs), s->JC, nullptr,
                                                                        nullptr);
        LAUNCH_CHECK(s);
      }
    }
    // CG: A_N D = -G on the running sims (pact), r0 = -G, z0 = A^{-1} r0 (kept: the PD direction)
    CK(cudaMemcpyAsync(s->pact, s->active, B * sizeof(int32_t), cudaMemcpyDeviceToDevice, s->stream));
    pdl_launch(s, k_axpby, nblk(len), 256, 0, s->Rv, s->G, -1.0, nullptr, nullptr, 0.0, len, B, nullptr);
    LAUNCH_CHECK(s);
    CK(cudaMemsetAsync(s->Dv, 0, len * sizeof(double), s->stream));
    CK(cudaMemcpyAsync(s->bb, s->dots, B * sizeof(double), cudaMemcpyDeviceToDevice, s->stream));  // |b|^2 = |G|^2
    apply_Ainv(s, B, s->Rv, Z0, nullptr, 1.0, 0.0, s->pact);
    CK(cudaMemcpyAsync(s->Pv, Z0, len * sizeof(double), cudaMemcpyDeviceToDevice, s->stream));
    dots(s, B, n3, {{s->Rv, Z0}}, s->rz);
    for (int it = 0;; ++it) {
      const bool fused = it > 0;
      if (!fused) dots(s, B, n3, {{s->Rv, s->Rv}}, s->dots + 2 * B);
      const FlagArgs fa = flag_args(s, it < s->opt.max_iter_adj);
      pdl_launch(s, k_adj_check, 1, 256, 0, s->dots + 2 * B, s->bb, B, s->newton_eta, it, s->opt.max_iter_adj, s->pact,
                                            s->nt_iters, s->nt_res, s->nt_flag, s->nactive, fused ? s->rz : nullptr,
                                            s->dots + 3 * B, fa.hflag, fa.nact3, fa.seq);
      LAUNCH_CHECK(s);
      if (it >= s->opt.max_iter_adj || read_nactive(s) == 0) break;
      apply_AN(s, B, s->X, s->Pv, s->Q, act_i, act_bs, s->JC);
      dots(s, B, n3, {{s->Pv, s->Q}}, s->dots + 3 * B);
      pdl_launch(s, k_negcurv, nblk(B, 64), 64, 0, s->dots + 3 * B, s->pact, B);
      LAUNCH_CHECK(s);
      pdl_launch(s, k_pcg_update, nblk(len), 256, 0, s->Dv, s->Rv, s->Pv, s->Q, s->rz, s->dots + 3 * B, len, B, s->pact,
                                                     nullptr, nullptr);
      LAUNCH_CHECK(s);
      apply_Ainv(s, B, s->Rv, s->Z, nullptr, 1.0, 0.0, s->pact);
      dots(s, B, n3, {{s->Rv, s->Z}, {s->Rv, s->Rv}}, s->dots + 3 * B);  // rz_new | |r|^2
      pdl_launch(s, k_pcg_dir, nblk(len), 256, 0, s->Pv, s->Z, s->dots + 3 * B, s->rz, len, B, s->pact);
      LAUNCH_CHECK(s);
      // (k_adj_check reads |r|^2 at dots[2B:3B): move it there)
      CK(cudaMemcpyAsync(s->dots + 2 * B, s->dots + 4 * B, B * sizeof(double), cudaMemcpyDeviceToDevice, s->stream));
    }
    dots(s, B, n3, {{s->G, s->Dv}}, s->gtd);
    pdl_launch(s, k_descent_guard, nblk(len), 256, 0, s->Dv, Z0, s->gtd, len, B, s->active);
    LAUNCH_CHECK(s);
    dots(s, B, n3, {{s->G, s->Dv}}, s->gtd);
    bool done = false;
    for (int trial = 0;; ++trial) {  // Armijo backtracking from alpha = 1 (as inner_lbfgs)
      pdl_launch(s, k_axpby, nblk(len), 256, 0, s->Xn, s->X, 1.0, s->Dv, s->alpha_ls, 1.0, len, B, s->ls_act);
      LAUNCH_CHECK(s);
      eval_f(s, B, s->Xn, s->Gn, nullptr, act_i, act_bs, true);
      const FlagArgs fl = flag_args(s);
      pdl_launch(s, k_ls_accept, 1, 256, 0, s->fcur, s->fnew, s->inert, s->esum, s->gtd, s->dots, gn2, s->alpha_ls,
                                            s->ls_act, trial, max_trial, s->nactive, s->ls_flag, B, fl.hflag, fl.nact3,
                                            fl.seq);
      LAUNCH_CHECK(s);
      int searching = 0, running = 1, nr = 0;
      read_nactive3(s, &searching, &running, &nr);
      if (trial == 0 && running == 0) {
        done = true;
        break;
      }
      if (searching == 0) break;
    }
    if (done) break;
    pdl_launch(s, k_newton_commit, nblk(len), 256, 0, s->X, s->G, s->Xn, s->Gn, len, B, s->active);
    LAUNCH_CHECK(s);
    pdl_launch(s, k_newton_commit_s, nblk(B, 64), 64, 0, s->fcur, s->fnew, s->dots, gn2, B, s->active);
    LAUNCH_CHECK(s);
  }
}

}  // namespace

extern "C" {

const char* pd_last_error(const pd_sim* sim) { return sim ? sim->err.c_str() : g_create_error.c_str(); }

void pd_destroy(pd_sim* sim) { delete sim; }

pd_status pd_create(const pd_mesh* mesh, const pd_material* mat, double h, const int32_t* fixed_dofs, int32_t n_fixed,
                    const pd_options* opts, pd_sim** out) {
  if (!out) return fail(nullptr, PD_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (!mesh || !mat || !opts) return fail(nullptr, PD_ERR_INVALID_ARGUMENT, "mesh, material and options are required");
  if (!(mat->poisson > -1.0 && mat->poisson < 0.5)) return fail(nullptr, PD_ERR_INVALID_ARGUMENT, "poisson must be in (-1, 0.5)");
  if (!(mat->youngs > 0) || !(mat->density > 0)) return fail(nullptr, PD_ERR_INVALID_ARGUMENT, "youngs and density must be > 0");
  if (!(h > 0)) return fail(nullptr, PD_ERR_INVALID_ARGUMENT, "h must be > 0");
  if (n_fixed < 0 || (n_fixed > 0 && !fixed_dofs)) return fail(nullptr, PD_ERR_INVALID_ARGUMENT, "bad fixed DoF list");
  if (opts->max_batch < 1 || opts->max_batch > 256) return fail(nullptr, PD_ERR_INVALID_ARGUMENT, "max_batch must be in [1, 256]");
  if (opts->max_steps < 1) return fail(nullptr, PD_ERR_INVALID_ARGUMENT, "max_steps must be >= 1");
  if (opts->n_contact < 0 || (opts->n_contact > 0 && !opts->contact_nodes))
    return fail(nullptr, PD_ERR_INVALID_ARGUMENT, "bad contact candidate list");
  std::unique_ptr<pd_sim> s(new pd_sim());
  try {
    s->youngs = mat->youngs;
    s->poisson = mat->poisson;
    s->density = mat->density;
    s->h = h;
    s->w_m = mat->muscle_w;
    for (int j = 0; j < 3; ++j) s->gravity[j] = mat->gravity[j];
    s->opt = *opts;
    {  // general contact plane n . x = d: plane coordinates x' = Q x - d e_z, Q the minimal rotation
       // (Rodrigues) taking the unit normal to e_z; gravity rotates with the frame
      double nv[3] = {opts->plane_n[0], opts->plane_n[1], opts->plane_n[2]};
      double nn = std::sqrt(nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2]);
      if (!std::isfinite(nn) || !std::isfinite(opts->plane_d))
        return fail(nullptr, PD_ERR_INVALID_ARGUMENT, "contact plane must be finite");
      if (nn == 0.0) {
        nv[0] = nv[1] = 0.0;
        nv[2] = nn = 1.0;
      }
      for (double& c : nv) c /= nn;
      const double d = opts->plane_d / nn;
      double* Q = s->fq.q;
      const double vx = nv[1], vy = -nv[0], c = nv[2];  // v = n x e_z (v_z = 0), c = n . e_z
      if (c < -1.0 + 1e-12) {  // n = -e_z: half turn about x
        const double R[9] = {1, 0, 0, 0, -1, 0, 0, 0, -1};
        for (int k = 0; k < 9; ++k) Q[k] = R[k];
      } else {  // Q = I + [v]x + [v]x^2 / (1 + c)
        const double k = 1.0 / (1.0 + c);
        const double R[9] = {1.0 - vy * vy * k, vx * vy * k, vy, vx * vy * k, 1.0 - vx * vx * k, -vx, -vy, vx,
                             1.0 - (vx * vx + vy * vy) * k};
        for (int j = 0; j < 9; ++j) Q[j] = R[j];
      }
      s->fq.d = d;
      s->frame = opts->n_contact > 0 && !(nv[0] == 0.0 && nv[1] == 0.0 && nv[2] == 1.0 && d == 0.0);
      if (s->frame) {
        double g[3];
        for (int r = 0; r < 3; ++r) g[r] = Q[3 * r] * s->gravity[0] + Q[3 * r + 1] * s->gravity[1] + Q[3 * r + 2] * s->gravity[2];
        for (int r = 0; r < 3; ++r) s->gravity[r] = g[r];
      }
    }
    if (s->opt.check_every < 1) s->opt.check_every = 1;
    if (s->opt.max_iter_fwd < 1) s->opt.max_iter_fwd = 10000;
    if (s->opt.max_iter_adj < 1) s->opt.max_iter_adj = 10000;
    if (s->opt.max_outer < 1) s->opt.max_outer = 10;
    if (!(s->opt.eps_phi > 0)) s->opt.eps_phi = 1e-6 * mesh->dx;
    if (s->opt.contact_mode == 0) s->opt.contact_mode = 1;
    if (s->opt.accel_fwd < 0 || s->opt.accel_fwd > 2)
      return fail(nullptr, PD_ERR_INVALID_ARGUMENT, "accel_fwd must be 0 (plain PD), 1 (L-BFGS) or 2 (Newton-PCG)");
    if (s->opt.accel_adj < 0 || s->opt.accel_adj > 1)
      return fail(nullptr, PD_ERR_INVALID_ARGUMENT, "accel_adj must be 0 (fixed point) or 1 (PCG)");
    if (s->opt.contact_mode != 1 && s->opt.contact_mode != 2)
      return fail(nullptr, PD_ERR_INVALID_ARGUMENT, "contact_mode must be 1 (frictionless) or 2 (sticky)");
    s->sticky = s->opt.contact_mode == 2 ? 1 : 0;
    s->Bmax = opts->max_batch;
    s->Tmax = opts->max_steps;
    double fiber[3] = {mat->fiber[0], mat->fiber[1], mat->fiber[2]};
    const double fn = std::sqrt(fiber[0] * fiber[0] + fiber[1] * fiber[1] + fiber[2] * fiber[2]);
    if (mat->muscle_w != 0.0) {
      if (!(fn > 0)) return fail(nullptr, PD_ERR_INVALID_ARGUMENT, "fiber direction must be non-zero");
      for (double& f : fiber) f /= fn;
    }
    if (mat->fiber_dir && mat->muscle_w != 0.0) {  // per-element fibers (normalised here, host copy for A)
      if (mesh->n_elems < 0) return fail(nullptr, PD_ERR_INVALID_ARGUMENT, "negative element count");
      s->plan.fib.assign(mat->fiber_dir, mat->fiber_dir + 3 * (int64_t)mesh->n_elems);
      for (int64_t e = 0; e < mesh->n_elems; ++e) {
        double* f = s->plan.fib.data() + 3 * e;
        const double nf = std::sqrt(f[0] * f[0] + f[1] * f[1] + f[2] * f[2]);
        if (!(nf > 0) || !std::isfinite(nf))
          return fail(nullptr, PD_ERR_INVALID_ARGUMENT, "fiber_dir of element " + std::to_string(e) + " is not a direction");
        for (int j = 0; j < 3; ++j) f[j] /= nf;
      }
    }
    const double yref = opts->youngs_ref > 0 ? opts->youngs_ref : mat->youngs;
    // volume-preserving term: w_v = lambda = w nu/(1 - 2 nu) per sim; A carries w + w_v
    const double kappa = mat->volume ? mat->poisson / (1.0 - 2.0 * mat->poisson) : 0.0;
    const double w_ref = yref / (1.0 + mat->poisson) * (1.0 + kappa);
    bool numerical = false;
    {  // K3 schedule version (env PD_K3_V = 3 selects the round-1 chain/item schedule) and the warps a v4 level
       // launch is split for: one CTA of kWarpsK3 warps per SM
      s->plan.k3_version = 4;
      if (const char* ev = std::getenv("PD_K3_V")) s->plan.k3_version = std::atoi(ev) == 3 ? 3 : 4;
      int dev = 0, nsm = 148;
      if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      s->nsm = std::max(1, nsm);
      s->plan.k3_warps = s->nsm * kWarpsK3;
    }
    std::string e = build_plan(s->plan, mesh->n_nodes, mesh->n_elems, mesh->rest_xyz, mesh->hex8, mesh->dx,
                               mat->density, h, fixed_dofs, n_fixed, w_ref, mat->muscle_w, fiber, opts->contact_nodes,
                               opts->n_contact, &numerical);
    if (!e.empty()) return fail(nullptr, numerical ? PD_ERR_NUMERICAL : PD_ERR_INVALID_ARGUMENT, e);
    const HostPlan& P = s->plan;
    {
      const double g = 1.0 / std::sqrt(3.0), c = 1.0 / (4.0 * mesh->dx);
      s->st.m3[0] = c * (1 - g) * (1 - g);
      s->st.m3[1] = c * (1 - g) * (1 + g);
      s->st.m3[2] = c * (1 + g) * (1 + g);
    }
    for (int j = 0; j < 3; ++j) s->st.fiber[j] = fiber[j];
    s->st.V = mesh->dx * mesh->dx * mesh->dx / 8.0;
    s->st.w_m = mat->muscle_w;
    s->st.clamp = 1e-6;
    s->st.kappa = kappa;
    // ---- device residency
    s->d_hex8 = s->upload(P.hex8);
    if (!P.fib.empty()) s->d_fib = s->upload(P.fib);
    s->d_inc_ptr = s->upload(P.inc_ptr);
    s->d_inc_ec = s->upload(P.inc_ec);
    s->d_pos = s->upload(P.pos_of_node);
    s->d_nodepos = s->upload(P.node_of_pos);
    s->d_mass = s->upload(P.node_mass);
    s->d_fixed = s->upload(P.fixed_node);
    s->d_nofix = s->alloc<uint8_t>(P.n);
    s->d_rows = s->upload(P.rows);
    auto up_sweep = [&](const HostPlan::Sweep& S, SweepDev& d) {
      d.A = s->upload(S.A);
      d.a_off = s->upload(S.a_off);
      d.zidx = s->upload(S.zidx);
      d.nk = s->upload(S.nk);
      d.nkd = s->upload(S.nkd);
      d.zrow = s->upload(S.zrow);
      d.out = s->upload(S.out);
      d.nvalid = s->upload(S.nvalid);
      d.chain = s->upload(S.chain);
      d.rec = reinterpret_cast<const int4*>(s->upload(S.rec));
      d.red_row = s->upload(S.red_row);
      d.red_mode = s->upload(S.red_mode);
      d.red_ptr = s->upload(S.red_ptr);
      d.red_src = s->upload(S.red_src);
    };
    if (const char* e = std::getenv("PD_K3_MMA")) s->k3_mma = std::atoi(e) ? 1 : 0;
    if (const char* e = std::getenv("PD_K3_NBUF")) s->k3_nbuf = std::min(4, std::max(2, std::atoi(e)));
    if (const char* e = std::getenv("PD_POLL")) s->poll = std::atoi(e) != 0;
    if (const char* e = std::getenv("PD_FUSE")) s->fuse = std::atoi(e) != 0;
    if (const char* e = std::getenv("PD_PROF_EVERY")) s->prof_every = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("PD_ACTIVE_WARM")) s->active_warm = std::atoi(e) != 0;
    if (const char* e = std::getenv("PD_LBFGS_GAMMA")) s->lb_gamma = std::atoi(e) != 0;
    auto up_sweep4 = [&](const HostPlan::Sweep4& S, Sweep4Dev& d) {
      d.A = s->upload(S.A);
      d.krow = s->upload(S.krow);
      d.pstart = s->upload(S.pstart);
      d.pkg = s->upload(S.pkg);
      d.pout = s->upload(S.pout);
      d.pnv = s->upload(S.pnv);
      d.wg = s->upload(S.wg);
      d.wpiece = s->upload(S.wpiece);
      d.red_row = s->upload(S.red_row);
      d.red_mode = s->upload(S.red_mode);
      d.red_ptr = s->upload(S.red_ptr);
      d.red_src = s->upload(S.red_src);
    };
    int64_t max_prows = 0;
    if (P.k3_version == 4) {
      up_sweep4(P.fw4, s->sw4f);
      up_sweep4(P.bw4, s->sw4b);
      max_prows = std::max(P.fw4.max_partial_rows, P.bw4.max_partial_rows);
    } else {
      up_sweep(P.fw, s->swf);
      up_sweep(P.bw, s->swb);
      max_prows = std::max(P.fw.max_partial_rows, P.bw.max_partial_rows);
    }
    s->Spart = s->alloc<double>((max_prows + 32) * 3 * s->Bmax);
    s->nactive_ll = s->alloc<int64_t>(4);
    const int64_t n3B = 3LL * P.n * s->Bmax;
    const int64_t sB = 3LL * P.nfree * s->Bmax;
    double** st_vecs[] = {&s->X, &s->V, &s->Y, &s->Xp, &s->Fext, &s->G, &s->W, &s->U, &s->Rv, &s->Z,
                          &s->Pv, &s->Q, &s->AX, &s->AV, &s->Bv, &s->DF};
    for (double** p : st_vecs) *p = s->alloc<double>(n3B);
    s->S0 = s->alloc<double>(sB);
    s->S1 = s->alloc<double>(sB);
    s->S2 = s->alloc<double>(sB);
    s->EF = s->alloc<double>((int64_t)P.m * 24 * s->Bmax);
    s->JC = s->alloc<double>((int64_t)P.m * 8 * s->Bmax * (kappa != 0.0 ? kJC + kJCV : (s->w_m != 0.0 ? kJC : 15)));
    if (kappa != 0.0) {
      s->DWV = s->alloc<double>((int64_t)P.m * s->Bmax);
      s->dwv_acc = s->alloc<double>(s->Bmax);
    }
    s->EE = s->alloc<double>((int64_t)P.m * s->Bmax);
    s->DW = s->alloc<double>((int64_t)P.m * s->Bmax);
    s->DR = s->alloc<double>((int64_t)P.m * s->Bmax);
    double** small[] = {&s->w_sim, &s->youngs_sim, &s->w_diag, &s->youngs_diag, &s->alpha, &s->beta, &s->rz, &s->bb, &s->dw_acc, &s->res_buf};
    for (double** p : small) *p = s->alloc<double>(s->Bmax);
    s->dots = s->alloc<double>(5 * s->Bmax);  // [B] slots: pairs of the multi-dots, Newton-PCG scalars at [2B, 5B)
    s->max_partial_blocks = (int64_t)red_chunks(std::max<int64_t>(3LL * P.n, P.m)) * s->Bmax;
    s->partial = s->alloc<double>(32 * s->max_partial_blocks + 64);  // up to 2 x 16 dot families (mdot pairs)
    s->active = s->alloc<int32_t>(s->Bmax);
    s->nactive = s->alloc<int32_t>(3);  // [0] last check / line-search count, [1] deferred convergence count,
                                        // [2] running sims within 16 tol (next check is immediate)
    s->it_buf = s->alloc<int32_t>(s->Bmax);
    s->flag_buf = s->alloc<int32_t>(s->Bmax);
    const int64_t TB = (int64_t)s->Tmax * s->Bmax;
    s->st_iters_f = s->alloc<int32_t>(TB);
    s->st_iters_a = s->alloc<int32_t>(TB);
    s->st_flag_f = s->alloc<int32_t>(TB);
    s->st_flag_a = s->alloc<int32_t>(TB);
    s->st_outer = s->alloc<int32_t>(TB);
    s->st_res_f = s->alloc<double>(TB);
    s->st_res_a = s->alloc<double>(TB);
    s->traj = s->alloc<double>((int64_t)(s->Tmax + 1) * n3B);
    s->act = s->w_m != 0.0 ? s->alloc<double>((int64_t)s->Bmax * s->Tmax * P.m) : nullptr;
    CK(cudaHostAlloc(&s->h_nactive, 4 * sizeof(int32_t), cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(s->h_nactive, 0, 4 * sizeof(int32_t));
    CK(cudaMallocHost(&s->h_small, 2 * s->Bmax * sizeof(int32_t)));
    if (s->opt.accel_fwd) {
      s->nhist = 4;  // L-BFGS memory (env PD_LBFGS_M, 1..16; 4 measured fastest)
      if (const char* e = std::getenv("PD_LBFGS_M")) s->nhist = std::min(16, std::max(1, std::atoi(e)));
      s->LS = s->alloc<double>(s->nhist * n3B);
      s->LY = s->alloc<double>(s->nhist * n3B);
      s->Dv = s->alloc<double>(n3B);
      s->Xn = s->alloc<double>(n3B);
      s->Gn = s->alloc<double>(n3B);
      s->rho_h = s->alloc<double>((int64_t)s->nhist * s->Bmax);
      s->gamma = s->alloc<double>(s->Bmax);
      s->aj_h = s->alloc<double>((int64_t)s->nhist * s->Bmax);
      double** sc[] = {&s->fcur, &s->fnew, &s->alpha_ls, &s->gtd, &s->g2, &s->gn2, &s->inert, &s->esum, &s->dtmp};
      for (double** p : sc) *p = s->alloc<double>(2 * s->Bmax);  // inert: [inertia | |grad g|^2]
      s->ls_act = s->alloc<int32_t>(s->Bmax);
      double** lb[] = {&s->lb_sg, &s->lb_yr, &s->lb_beta, &s->lb_da, &s->lb_db};
      for (double** p : lb) *p = s->alloc<double>((int64_t)2 * s->nhist * s->Bmax);  // lb_da: [da | db]
      s->lb_G = s->alloc<double>((int64_t)s->nhist * s->nhist * s->Bmax);
      s->ls_flag = s->alloc<int32_t>(s->Bmax);
      if (s->opt.accel_fwd == 2) {  // Newton-PCG scratch: CG mask and per-sim CG statistics
        s->pact = s->alloc<int32_t>(s->Bmax);
        s->nt_iters = s->alloc<int32_t>(s->Bmax);
        s->nt_flag = s->alloc<int32_t>(s->Bmax);
        s->nt_res = s->alloc<double>(s->Bmax);
        if (const char* e = std::getenv("PD_NEWTON_ETA")) s->newton_eta = std::atof(e);
      }
    }
    if (P.nc > 0) {
      const int c = P.nc;
      const int64_t cB = (int64_t)c * s->Bmax;
      s->nc = c;
      s->csup_first = P.sfirst[P.csup];
      s->d_cand_node = s->upload(P.cand_node);
      s->d_cand_of_node = s->upload(P.cand_of_node);
      s->d_cand_of_loc = s->upload(P.cand_of_loc);
      s->d_S = s->upload(P.Scc);
      s->LAM = s->alloc<double>(cB);
      s->PIN = s->alloc<uint8_t>(cB);
      s->NEWPIN = s->alloc<uint8_t>(cB);
      s->traj_pin = s->alloc<uint8_t>(cB * s->Tmax);
      s->flist = s->alloc<int32_t>(cB);
      s->fpos = s->alloc<int32_t>(cB);
      s->Qc = s->alloc<double>(cB * c);
      s->PIc = s->alloc<double>((int64_t)s->Bmax * 32 * 32);
      s->Cb = s->alloc<double>(cB * 32);
      s->Mb = s->alloc<double>(cB * 32);
      s->Rb = s->alloc<double>(cB * 32);
      s->Rsave = s->alloc<double>((int64_t)c * 3 * s->Bmax);
      int32_t** small_i[] = {&s->kcount, &s->need, &s->oact, &s->onext, &s->changed, &s->it_base};
      for (int32_t** p : small_i) *p = s->alloc<int32_t>(s->Bmax);
    }
    CK(cudaDeviceSynchronize());
  } catch (CudaError& e) {
    return fail(nullptr, PD_ERR_CUDA, e.what());
  } catch (std::exception& e) {
    return fail(nullptr, PD_ERR_CUDA, e.what());
  }
  *out = s.release();
  return PD_OK;
}

pd_status pd_profile(const pd_sim* s, double* ms, int64_t* count, int32_t n) {
  if (!s) return PD_ERR_INVALID_ARGUMENT;
  for (int k = 0; k < n && k < 6; ++k) {
    if (ms) ms[k] = s->prof_ms[k];
    if (count) count[k] = s->prof_cnt[k];
  }
  return PD_OK;
}

pd_status pd_contact_sets(const pd_sim* s, uint8_t* out) {
  if (!s || !out) return PD_ERR_INVALID_ARGUMENT;
  if (!s->have_traj || s->nc == 0) return PD_ERR_STATE;
  const int B = s->B, T = s->T, c = s->nc;
  std::vector<uint8_t> h((int64_t)T * c * B);  // device layout [step][j][b]
  if (cudaMemcpy(h.data(), s->traj_pin, h.size(), cudaMemcpyDeviceToHost) != cudaSuccess) return PD_ERR_CUDA;
  for (int b = 0; b < B; ++b)
    for (int i = 0; i < T; ++i)
      for (int j = 0; j < c; ++j) out[((int64_t)b * T + i) * c + j] = h[((int64_t)i * c + j) * B + b];
  return PD_OK;
}

pd_status pd_info(const pd_sim* s, int64_t* out, int32_t n) {
  if (!s || !out) return PD_ERR_INVALID_ARGUMENT;
  const HostPlan& P = s->plan;
  const int64_t v[] = {P.n, P.nfree, P.nsup, P.nlevels, P.nnzL, (int64_t)s->opt.n_contact,
                       (int64_t)std::llround(P.factor_ms), s->launches};
  for (int i = 0; i < n && i < (int)(sizeof(v) / sizeof(v[0])); ++i) out[i] = v[i];
  return PD_OK;
}

pd_status pd_forward(pd_sim* s, int32_t B, const double* q0, const double* v0, const double* f_ext,
                     int64_t f_ext_step_stride, const double* actuation, const double* youngs_per_sim, int32_t steps,
                     double* q_traj, double* v_traj, pd_stats* stats, void* cuda_stream) {
  if (!s) return PD_ERR_INVALID_ARGUMENT;
  if (B < 1 || B > s->Bmax) return fail(s, PD_ERR_INVALID_ARGUMENT, "B out of [1, max_batch]");
  if (steps < 1 || steps > s->Tmax) return fail(s, PD_ERR_INVALID_ARGUMENT, "steps out of [1, max_steps]");
  if (!q0 || !v0) return fail(s, PD_ERR_INVALID_ARGUMENT, "q0 and v0 are required");
  if (f_ext_step_stride != 0 && f_ext_step_stride != 3LL * s->plan.n)
    return fail(s, PD_ERR_INVALID_ARGUMENT, "f_ext_step_stride must be 0 (constant) or 3n ([B][steps][3n])");
  if (s->w_m != 0.0 && !actuation) return fail(s, PD_ERR_INVALID_ARGUMENT, "muscle energy needs an actuation array");
  s->stream = (cudaStream_t)cuda_stream;
  s->launches = 0;
  s->pins_live = false;
  s->have_traj = false;  // set again only when this forward completes (a failed forward leaves no trajectory)
  for (int k = 0; k < 6; ++k) { s->prof_ms[k] = 0; s->prof_cnt[k] = 0; }
  s->ev_open.clear();
  s->ev_next = 0;
  const HostPlan& P = s->plan;
  const int n3 = 3 * P.n;
  const int64_t len = (int64_t)n3 * B;
  Nvtx nv_fwd("pd_forward");
  try {
    set_w(s, B, youngs_per_sim);
    if (s->gamma) {  // H0 scaling of the L-BFGS forward starts at 1 (kept across the steps of this forward)
      const std::vector<double> ones(B, 1.0);
      CK(cudaMemcpyAsync(s->gamma, ones.data(), B * sizeof(double), cudaMemcpyHostToDevice, s->stream));
      CK(cudaStreamSynchronize(s->stream));
    }
    abi_in(s, q0, s->X, B, n3, 1);
    abi_in(s, v0, s->V, B, n3, 2);
    if (f_ext && !f_ext_step_stride) abi_in(s, f_ext, s->Fext, B, n3, 2);
    if (actuation && s->act) {
      CK(cudaMemcpyAsync(s->act, actuation, sizeof(double) * (int64_t)B * steps * P.m, cudaMemcpyDeviceToDevice,
                         s->stream));
    }
    s->has_act = actuation && s->act;
    CK(cudaMemcpyAsync(s->traj, s->X, len * sizeof(double), cudaMemcpyDeviceToDevice, s->stream));
    const double tol = s->opt.tol_fwd;
    bool q_stale = false;
    for (int i = 0; i < steps; ++i) {
      Nvtx nv_step("forward_step");
      const double* act_i = s->has_act ? s->act + (int64_t)i * P.m : nullptr;
      const int64_t act_bs = (int64_t)steps * P.m;
      if (f_ext && f_ext_step_stride)  // time-varying f_ext: this step's slice of [B][steps][3n]
        abi_in(s, f_ext + (int64_t)i * n3, s->Fext, B, (int64_t)steps * n3, 2);
      pdl_launch(s, k_y, nblk(len), 256, 0, s->X, s->V, f_ext ? s->Fext : nullptr, s->d_mass, s->Y, P.n, B, s->h,
                                            s->gravity[0], s->gravity[1], s->gravity[2]);
      LAUNCH_CHECK(s);
      CK(cudaMemcpyAsync(s->Xp, s->X, len * sizeof(double), cudaMemcpyDeviceToDevice, s->stream));
      const bool predict = s->opt.x0_predict && s->opt.fixed_iter <= 0;
      if (predict) {  // x^0 = x_i + h v_i (Dirichlet DoFs have v = 0 and stay at rest)
        pdl_launch(s, k_axpby, nblk(len), 256, 0, s->X, s->Xp, 1.0, s->V, nullptr, s->h, len, B, nullptr);
        LAUNCH_CHECK(s);
      }
      const bool contact = s->nc > 0;
      const int64_t cB = (int64_t)s->nc * B;
      if (i == 0) q_stale = false;
      if (contact) {  // Alg. 1: V_i = empty
        const bool keep_set = s->active_warm && i > 0;  // (probe: PIN, kcount and Q of the last step's final set stay)
        if (!keep_set) CK(cudaMemsetAsync(s->PIN, 0, cB, s->stream));
        pdl_launch(s, k_fill_int, 1, 256, 0, s->oact, 1, B);
        LAUNCH_CHECK(s);
        if (!keep_set) {
          pdl_launch(s, k_fill_int, 1, 256, 0, s->kcount, s->nc, B);  // no pins: unconstrained root block
          LAUNCH_CHECK(s);
        }
        CK(cudaMemsetAsync(s->it_base, 0, B * sizeof(int32_t), s->stream));
        s->pins_live = true;
      }
      for (int outer = 1; outer <= (contact ? s->opt.max_outer : 1); ++outer) {
        if (contact) {
          pdl_launch(s, k_contact_restart, nblk(len), 256, 0, s->X, s->Xp, P.n, B, s->d_cand_of_node, s->PIN, s->oact,
                                                              (s->opt.outer_warm && outer > 1) || (predict && outer == 1),
                                                              s->sticky);
          LAUNCH_CHECK(s);  // x_{i+1} = x_i, pinned normal DoFs on the plane
          if (outer > 1) build_Q(s, B, s->oact);
          else if (s->active_warm && i > 0 && q_stale) build_Q(s, B, nullptr);  // (probe: kept set whose Q is not current)
          CK(cudaMemcpyAsync(s->active, s->oact, B * sizeof(int32_t), cudaMemcpyDeviceToDevice, s->stream));
        } else {
          pdl_launch(s, k_fill_int, 1, 256, 0, s->active, 1, B);
          LAUNCH_CHECK(s);
        }
        if (s->opt.accel_fwd == 2 && s->opt.fixed_iter <= 0) {
          inner_newton(s, B, i, act_i, act_bs, contact ? s->it_base : nullptr);
        } else if (s->opt.accel_fwd && s->opt.fixed_iter <= 0) {
          inner_lbfgs(s, B, i, act_i, act_bs, contact ? s->it_base : nullptr, s->opt.lbfgs_warm && outer > 1);
        } else {
          for (int iter = 0;; ++iter) {
            residual(s, B, s->X, s->Y, act_i, act_bs, s->d_fixed);
            dots(s, B, n3, {{s->G, s->G}, {s->W, s->W}});
            const FlagArgs fc = flag_args(s, s->opt.fixed_iter <= 0 && iter < s->opt.max_iter_fwd &&
                                                 iter % s->opt.check_every == 0);
            pdl_launch(s, k_fwd_check, 1, 256, 0, s->dots, B, tol, iter, s->opt.fixed_iter,
                                                           s->opt.max_iter_fwd, s->active, s->st_iters_f + (int64_t)i * B,
                                                           s->st_res_f + (int64_t)i * B, s->st_flag_f + (int64_t)i * B,
                                                           s->nactive, contact ? s->it_base : nullptr, nullptr, nullptr, nullptr,
                                                           fc.hflag, fc.nact3, fc.seq);
            LAUNCH_CHECK(s);
            if (s->opt.fixed_iter > 0) {
              if (iter >= s->opt.fixed_iter) break;
            } else if (iter >= s->opt.max_iter_fwd) {
              break;
            } else if (iter % s->opt.check_every == 0) {
              if (read_nactive(s) == 0) break;
            }
            apply_Ainv(s, B, s->G, s->X, nullptr, -1.0, 1.0, s->active);  // x <- A^{-1} d(x)  (eq:pd_global)
          }
        }
        if (!contact) break;
        // predictor on the converged x; stop when the set is unchanged
        CK(cudaMemcpyAsync(s->it_base, s->st_iters_f + (int64_t)i * B, B * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                           s->stream));
        CK(cudaMemsetAsync(s->changed, 0, B * sizeof(int32_t), s->stream));
        {
          ProfScope ps(s, 4);
          pdl_launch(s, k_contact_predict, nblk(cB), 256, 0, s->X, s->LAM, s->d_cand_node, s->nc, B, s->opt.eps_phi,
                                                             s->PIN, s->oact, s->NEWPIN, s->changed);
          LAUNCH_CHECK(s);
          pdl_launch(s, k_contact_outer, nblk(cB), 256, 0, s->oact, s->changed, s->NEWPIN, s->PIN, s->nc, B, outer,
                                                           s->opt.max_outer, s->onext, s->st_outer + (int64_t)i * B,
                                                           s->st_flag_f + (int64_t)i * B);
          LAUNCH_CHECK(s);
        }
        CK(cudaMemcpyAsync(s->oact, s->onext, B * sizeof(int32_t), cudaMemcpyDeviceToDevice, s->stream));
        CK(cudaMemcpyAsync(s->h_small, s->onext, B * sizeof(int32_t), cudaMemcpyDeviceToHost, s->stream));
        CK(cudaStreamSynchronize(s->stream));
        prof_flush(s);
        int going = 0;
        for (int b = 0; b < B; ++b) going += s->h_small[b];
        q_stale = going != 0;  // (left through the outer cap: PIN was updated after the last build_Q)
        if (!going) break;
      }
      if (contact) {
        CK(cudaMemcpyAsync(s->traj_pin + (int64_t)i * cB, s->PIN, cB, cudaMemcpyDeviceToDevice, s->stream));
        s->pins_live = false;
      }
      pdl_launch(s, k_velocity, nblk(len), 256, 0, s->X, s->Xp, s->V, len, 1.0 / s->h);
      LAUNCH_CHECK(s);
      CK(cudaMemcpyAsync(s->traj + (int64_t)(i + 1) * len, s->X, len * sizeof(double), cudaMemcpyDeviceToDevice,
                         s->stream));
      if (q_traj) abi_out(s, s->X, q_traj + (int64_t)(i + 1) * n3, B, (int64_t)(steps + 1) * n3, 1);
      if (v_traj) abi_out(s, s->V, v_traj + (int64_t)(i + 1) * n3, B, (int64_t)(steps + 1) * n3, 2);
    }
    if (q_traj)
      CK(cudaMemcpy2DAsync(q_traj, (steps + 1) * n3 * sizeof(double), q0, n3 * sizeof(double), n3 * sizeof(double), B,
                           cudaMemcpyDeviceToDevice, s->stream));
    if (v_traj)
      CK(cudaMemcpy2DAsync(v_traj, (steps + 1) * n3 * sizeof(double), v0, n3 * sizeof(double), n3 * sizeof(double), B,
                           cudaMemcpyDeviceToDevice, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    prof_flush(s);
    if (stats) {
      const int64_t TB = (int64_t)steps * B;
      std::vector<int32_t> it(TB), fl(TB), ou(TB);
      std::vector<double> rs(TB);
      CK(cudaMemcpy(ou.data(), s->st_outer, TB * sizeof(int32_t), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(it.data(), s->st_iters_f, TB * sizeof(int32_t), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(fl.data(), s->st_flag_f, TB * sizeof(int32_t), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(rs.data(), s->st_res_f, TB * sizeof(double), cudaMemcpyDeviceToHost));
      int nnc = 0;
      for (int b = 0; b < B; ++b)
        for (int i = 0; i < steps; ++i) {  // device buffers are [step][b]; ABI stats are [b][step]
          if (stats->iters_fwd) stats->iters_fwd[b * steps + i] = it[(int64_t)i * B + b];
          if (stats->final_res_fwd) stats->final_res_fwd[b * steps + i] = rs[(int64_t)i * B + b];
          if (stats->contact_outer) stats->contact_outer[b * steps + i] = s->nc > 0 ? ou[(int64_t)i * B + b] : 0;
          nnc += fl[(int64_t)i * B + b];
        }
      stats->n_nonconverged = nnc;
    }
  } catch (CudaError& e) {
    s->pins_live = false;
    return fail(s, PD_ERR_CUDA, e.what());
  }
  s->have_traj = true;
  s->B = B;
  s->T = steps;
  return PD_OK;
}

static pd_status backward_impl(pd_sim* s, const double* dL_dqT, const double* dL_dvT, const double* dq_steps,
                               const double* dv_steps, double* dL_dq0, double* dL_dv0, double* dL_dfext,
                               double* dfext_steps, double* dL_dE, double* dL_dnu, double* dL_dact, pd_stats* stats,
                               void* cuda_stream) {
  if (!s) return PD_ERR_INVALID_ARGUMENT;
  if (!s->have_traj) return fail(s, PD_ERR_STATE, "pd_backward needs a preceding pd_forward");
  s->stream = (cudaStream_t)cuda_stream;
  s->w_cur = s->w_sim;  // the forward's per-sim weights (a diagnostic hook in between used its own scratch)
  s->launches = 0;
  s->pins_live = false;
  const HostPlan& P = s->plan;
  const int B = s->B, T = s->T;
  const int n3 = 3 * P.n;
  const int64_t len = (int64_t)n3 * B;
  const double h = s->h;
  try {
    if (dL_dqT) {
      abi_in(s, dL_dqT, s->AX, B, n3, 2);
    } else {
      CK(cudaMemsetAsync(s->AX, 0, len * sizeof(double), s->stream));
    }
    if (dL_dvT) {
      abi_in(s, dL_dvT, s->AV, B, n3, 2);
    } else {
      CK(cudaMemsetAsync(s->AV, 0, len * sizeof(double), s->stream));
    }
    CK(cudaMemsetAsync(s->DF, 0, len * sizeof(double), s->stream));
    CK(cudaMemsetAsync(s->dw_acc, 0, B * sizeof(double), s->stream));
    if (s->dwv_acc) CK(cudaMemsetAsync(s->dwv_acc, 0, B * sizeof(double), s->stream));
    const int64_t sstride = (int64_t)(T + 1) * n3;  // batch stride of [B][T+1][3n] per-step loss arrays
    if (dq_steps) abi_add(s, s->AX, dq_steps + (int64_t)T * n3, B, sstride);
    if (dv_steps) abi_add(s, s->AV, dv_steps + (int64_t)T * n3, B, sstride);
    const bool pcg = s->opt.accel_adj != 0;
    const bool fuse = s->fuse;
    Nvtx nv_bwd("pd_backward");
    for (int i = T - 1; i >= 0; --i) {
      Nvtx nv_step("backward_step");
      const double* x1 = s->traj + (int64_t)(i + 1) * len;
      const double* act_i = s->has_act ? s->act + (int64_t)i * P.m : nullptr;
      const int64_t act_bs = (int64_t)T * P.m;
      // b = a_x + a_v / h on unconstrained DoFs
      if (s->nc > 0) {  // the step's final active set, frozen ("the same modified matrix")
        CK(cudaMemcpyAsync(s->PIN, s->traj_pin + (int64_t)i * s->nc * B, (int64_t)s->nc * B, cudaMemcpyDeviceToDevice,
                           s->stream));
        s->pins_live = true;
        build_Q(s, B, nullptr);
      }
      {  // per-step Jacobian data of the projections at x_{i+1}, reused by every K4 product
        ProfScope ps(s, 3);
        pdl_launch(s, k_elem_jac, nblk((int64_t)P.m * B * 8, 256), 256, 0, x1, s->st, elem_args(s, B, act_i, act_bs),
                                                                         s->JC);
        LAUNCH_CHECK(s);
        if (s->st.kappa != 0.0) {
          pdl_launch(s, k_vol<3>, nblk((int64_t)P.m * B * 8, 256), 256, 0, x1, nullptr, s->st,
                                                                          elem_args(s, B, act_i, act_bs), s->JC,
                                                                          nullptr, nullptr);
          LAUNCH_CHECK(s);
        }
      }
      pdl_launch(s, k_axpby, nblk(len), 256, 0, s->Bv, s->AX, 1.0, s->AV, nullptr, 1.0 / h, len, B, nullptr);
      LAUNCH_CHECK(s);
      zero_constrained(s, s->Bv, B);
      dots(s, B, n3, {{s->Bv, s->Bv}}, s->bb);
      CK(cudaMemsetAsync(s->U, 0, len * sizeof(double), s->stream));
      CK(cudaMemcpyAsync(s->Rv, s->Bv, len * sizeof(double), cudaMemcpyDeviceToDevice, s->stream));
      pdl_launch(s, k_fill_int, 1, 256, 0, s->active, 1, B);
      LAUNCH_CHECK(s);
      if (pcg) {
        apply_Ainv(s, B, s->Rv, s->Z, nullptr, 1.0, 0.0, nullptr);
        CK(cudaMemcpyAsync(s->Pv, s->Z, len * sizeof(double), cudaMemcpyDeviceToDevice, s->stream));
        dots(s, B, n3, {{s->Rv, s->Z}}, s->rz);
      }
      for (int iter = 0;; ++iter) {
        // |r|^2: computed here on the first iteration (and by the fixed point), else by the fused dots at the
        // end of the previous PCG iteration (dots[2B:3B]); k_adj_check also commits rz <- rz_new there
        const bool fused_rr = pcg && iter > 0;
        if (!fused_rr) dots(s, B, n3, {{s->Rv, s->Rv}});
        const FlagArgs fa = flag_args(s, iter < s->opt.max_iter_adj && iter % s->opt.check_every == 0);
        pdl_launch(s, k_adj_check, 1, 256, 0, fused_rr ? s->dots + 2 * B : s->dots, s->bb, B, s->opt.tol_adj, iter,
                                              s->opt.max_iter_adj, s->active, s->st_iters_a + (int64_t)i * B,
                                              s->st_res_a + (int64_t)i * B, s->st_flag_a + (int64_t)i * B, s->nactive,
                                              fused_rr ? s->rz : nullptr, s->dots + B, fa.hflag, fa.nact3, fa.seq);
        LAUNCH_CHECK(s);
        if (iter >= s->opt.max_iter_adj) break;
        if (iter % s->opt.check_every == 0 && read_nactive(s) == 0) break;
        if (pcg) {
          apply_AN(s, B, x1, s->Pv, s->Q, act_i, act_bs, s->JC);  // (k_gather zeroes the constrained rows)
          dots(s, B, n3, {{s->Pv, s->Q}}, s->dots + B);
          // u += alpha p, r -= alpha q, alpha = rz / pq (one pass)
          pdl_launch(s, k_pcg_update, nblk(len), 256, 0, s->U, s->Rv, s->Pv, s->Q, s->rz, s->dots + B, len, B, s->active,
                                                         fuse ? s->S0 : nullptr, s->d_pos);
          LAUNCH_CHECK(s);
          apply_Ainv(s, B, fuse ? nullptr : s->Rv, s->Z, nullptr, 1.0, 0.0, s->active);
          dots(s, B, n3, {{s->Rv, s->Z}, {s->Rv, s->Rv}}, s->dots + B);  // rz_new | |r|^2
          // p = z + beta p, beta = rz_new / rz (rz itself is committed by the next k_adj_check)
          pdl_launch(s, k_pcg_dir, nblk(len), 256, 0, s->Pv, s->Z, s->dots + B, s->rz, len, B, s->active);
          LAUNCH_CHECK(s);
        } else {
          // fixed point u <- u + A^{-1}(b - A_N u) == A^{-1}(b + dA u)  (eq:bp_update)
          apply_Ainv(s, B, s->Rv, s->U, nullptr, 1.0, 1.0, s->active);
          apply_AN(s, B, x1, s->U, s->Q, act_i, act_bs, s->JC);  // (k_gather zeroes the constrained rows)
          pdl_launch(s, k_axpby, nblk(len), 256, 0, s->Rv, s->Bv, 1.0, s->Q, nullptr, -1.0, len, B, s->active);
          LAUNCH_CHECK(s);
        }
      }
      // parameter terms, f_ext accumulation, state adjoint update
      ProfScope ps_param(s, 5);
      pdl_launch(s, k_elem_param, nblk((int64_t)P.m * B * 8, 256), 256, 0, x1, s->U, s->st, elem_args(s, B, act_i, act_bs),
                                                                      s->DW, s->has_act ? s->DR : nullptr);
      LAUNCH_CHECK(s);
      dots(s, B, P.m, {{s->DW, nullptr}}, s->dw_acc, 1);
      if (s->DWV) {
        pdl_launch(s, k_vol<4>, nblk((int64_t)P.m * B * 8, 256), 256, 0, x1, s->U, s->st, elem_args(s, B, act_i, act_bs),
                                                                        nullptr, s->DWV, nullptr);
        LAUNCH_CHECK(s);
        dots(s, B, P.m, {{s->DWV, nullptr}}, s->dwv_acc, 1);
      }
      if (dL_dact && s->has_act) {
        pdl_launch(s, k_state_to_abi, nblk((int64_t)P.m * B), 256, 0, s->DR, dL_dact + (int64_t)i * P.m, P.m, B,
                                                                      (int64_t)T * P.m);
        LAUNCH_CHECK(s);
      }
      pdl_launch(s, k_axpby, nblk(len), 256, 0, s->DF, s->DF, 1.0, s->U, nullptr, 1.0, len, B, nullptr);
      LAUNCH_CHECK(s);
      if (dfext_steps) {  // dL/df_ext of step i = u_i (0 on Dirichlet DoFs)
        zero_constrained_fixed(s, s->U, B);
        abi_out(s, s->U, dfext_steps + (int64_t)i * n3, B, (int64_t)T * n3, 2);
      }
      const bool sticky_step = s->sticky && s->pins_live;
      if (sticky_step) {  // pinned values x_{i+1,a} = x_{i,a}: EX = b_a - (A_N u)_a
        s->pins_live = false;  // A_N u on every row, pinned rows included
        apply_AN(s, B, x1, s->U, s->Z, act_i, act_bs, s->JC);
        s->pins_live = true;
        pdl_launch(s, k_sticky_extra, nblk(len), 256, 0, s->Pv, s->AX, s->AV, s->Z, 1.0 / h, P.n, B, s->d_cand_of_node,
                                                         s->PIN);
        LAUNCH_CHECK(s);
      }
      pdl_launch(s, k_adj_state, nblk(len), 256, 0, s->U, s->d_mass, s->d_fixed, s->AX, s->AV, P.n, B, h);
      LAUNCH_CHECK(s);
      if (sticky_step) {
        pdl_launch(s, k_axpby, nblk(len), 256, 0, s->AX, s->AX, 1.0, s->Pv, nullptr, 1.0, len, B, nullptr);
        LAUNCH_CHECK(s);
      }
      if (dq_steps) abi_add(s, s->AX, dq_steps + (int64_t)i * n3, B, sstride);
      if (dv_steps) abi_add(s, s->AV, dv_steps + (int64_t)i * n3, B, sstride);
      s->pins_live = false;
    }
    if (dL_dq0) abi_out(s, s->AX, dL_dq0, B, n3, 2);
    if (dL_dv0) abi_out(s, s->AV, dL_dv0, B, n3, 2);
    if (dL_dfext) {
      pdl_launch(s, k_zero_constrained, nblk(len), 256, 0, s->DF, s->d_fixed, P.n, B, nullptr, nullptr, 0);
      LAUNCH_CHECK(s);
      abi_out(s, s->DF, dL_dfext, B, n3, 2);
    }
    // dL/dE = dL/dw / (1+nu); dL/dnu = -dL/dw E/(1+nu)^2   (w = E/(1+nu))
    // with the volume term (w_v = lambda = E nu/((1+nu)(1-2nu))) both weights enter
    std::vector<double> dw(B), dwv(B, 0.0), E(B);
    CK(cudaMemcpyAsync(dw.data(), s->dw_acc, B * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
    if (s->dwv_acc) CK(cudaMemcpyAsync(dwv.data(), s->dwv_acc, B * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaMemcpyAsync(E.data(), s->youngs_sim, B * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    std::vector<double> dE(B), dnu(B);
    const double nu = s->poisson, p1 = 1.0 + nu, m2 = 1.0 - 2.0 * nu;
    for (int b = 0; b < B; ++b) {
      dE[b] = dw[b] / p1 + dwv[b] * nu / (p1 * m2);
      dnu[b] = -dw[b] * E[b] / (p1 * p1) + dwv[b] * E[b] * (1.0 + 2.0 * nu * nu) / (p1 * p1 * m2 * m2);
    }
    if (dL_dE) CK(cudaMemcpyAsync(dL_dE, dE.data(), B * sizeof(double), cudaMemcpyHostToDevice, s->stream));
    if (dL_dnu) CK(cudaMemcpyAsync(dL_dnu, dnu.data(), B * sizeof(double), cudaMemcpyHostToDevice, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    prof_flush(s);
    if (stats) {
      const int64_t TB = (int64_t)T * B;
      std::vector<int32_t> it(TB), fl(TB);
      std::vector<double> rs(TB);
      CK(cudaMemcpy(it.data(), s->st_iters_a, TB * sizeof(int32_t), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(fl.data(), s->st_flag_a, TB * sizeof(int32_t), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(rs.data(), s->st_res_a, TB * sizeof(double), cudaMemcpyDeviceToHost));
      int nnc = 0;
      for (int b = 0; b < B; ++b)
        for (int i = 0; i < T; ++i) {
          if (stats->iters_adj) stats->iters_adj[b * T + i] = it[(int64_t)i * B + b];
          if (stats->final_res_adj) stats->final_res_adj[b * T + i] = rs[(int64_t)i * B + b];
          nnc += fl[(int64_t)i * B + b];
        }
      stats->n_nonconverged = nnc;
    }
  } catch (CudaError& e) {
    s->pins_live = false;
    return fail(s, PD_ERR_CUDA, e.what());
  }
  return PD_OK;
}

pd_status pd_backward(pd_sim* s, const double* dL_dqT, const double* dL_dvT, double* dL_dq0, double* dL_dv0,
                      double* dL_dfext, double* dL_dE, double* dL_dnu, double* dL_dact, pd_stats* stats,
                      void* cuda_stream) {
  return backward_impl(s, dL_dqT, dL_dvT, nullptr, nullptr, dL_dq0, dL_dv0, dL_dfext, nullptr, dL_dE, dL_dnu, dL_dact,
                       stats, cuda_stream);
}

pd_status pd_backward_steps(pd_sim* s, const double* dL_dq_steps, const double* dL_dv_steps, double* dL_dq0,
                            double* dL_dv0, double* dL_dfext_steps, double* dL_dE, double* dL_dnu, double* dL_dact,
                            pd_stats* stats, void* cuda_stream) {
  return backward_impl(s, nullptr, nullptr, dL_dq_steps, dL_dv_steps, dL_dq0, dL_dv0, nullptr, dL_dfext_steps, dL_dE,
                       dL_dnu, dL_dact, stats, cuda_stream);
}

pd_status pd_eval_objective(pd_sim* s, int32_t B, const double* x, const double* y, const double* youngs_per_sim,
                            const double* act, double* grad_g, double* g, void* cuda_stream) {
  if (!s) return PD_ERR_INVALID_ARGUMENT;
  if (B < 1 || B > s->Bmax || !x || !y) return fail(s, PD_ERR_INVALID_ARGUMENT, "bad arguments");
  if (s->w_m != 0.0 && !act) return fail(s, PD_ERR_INVALID_ARGUMENT, "muscle energy needs act");
  s->stream = (cudaStream_t)cuda_stream;
  const HostPlan& P = s->plan;
  const int n3 = 3 * P.n;
  const int64_t len = (int64_t)n3 * B;
  try {
    set_w(s, B, youngs_per_sim, true);
    pdl_launch(s, k_abi_to_state, nblk(len), 256, 0, x, s->X, n3, B, -1);
    LAUNCH_CHECK(s);
    pdl_launch(s, k_abi_to_state, nblk(len), 256, 0, y, s->Y, n3, B, -1);
    LAUNCH_CHECK(s);
    residual(s, B, s->X, s->Y, act, P.m, s->d_nofix);
    if (grad_g) {
      pdl_launch(s, k_state_to_abi, nblk(len), 256, 0, s->G, grad_g, n3, B, n3);
      LAUNCH_CHECK(s);
    }
    if (g) {
      // g = sum_e E_e + sum_i m_i/(2h^2) (x_i - y_i)^2   (eq:opt)
      dots(s, B, P.m, {{s->EE, nullptr}}, g);
      pdl_launch(s, k_axpby, nblk(len), 256, 0, s->Q, s->X, 1.0, s->Y, nullptr, -1.0, len, B, nullptr);
      LAUNCH_CHECK(s);
      CK(cudaMemsetAsync(s->EF, 0, (int64_t)P.m * 24 * B * sizeof(double), s->stream));
      pdl_launch(s, k_gather, nblk((int64_t)P.n * B), 256, 0, s->Q, nullptr, s->EF, s->d_mass, s->d_inc_ptr,
                                                              s->d_inc_ec, s->d_nofix, s->d_pos, P.n, B,
                                                              1.0 / (s->h * s->h), 1, s->Z, nullptr, nullptr, nullptr,
                                                              nullptr, nullptr, 0);
      LAUNCH_CHECK(s);
      dots(s, B, n3, {{s->Q, s->Z}});
      pdl_launch(s, k_axpby, 1, 64, 0, g, g, 1.0, s->dots, nullptr, 0.5, B, B, nullptr);
      LAUNCH_CHECK(s);
    }
    CK(cudaStreamSynchronize(s->stream));
  } catch (CudaError& e) {
    return fail(s, PD_ERR_CUDA, e.what());
  }
  return PD_OK;
}

pd_status pd_apply_Ainv(pd_sim* s, int32_t B, const double* rhs, double* out, void* cuda_stream) {
  if (!s) return PD_ERR_INVALID_ARGUMENT;
  if (B < 1 || B > s->Bmax || !rhs || !out) return fail(s, PD_ERR_INVALID_ARGUMENT, "bad arguments");
  s->stream = (cudaStream_t)cuda_stream;
  const int n3 = 3 * s->plan.n;
  const int64_t len = (int64_t)n3 * B;
  try {
    pdl_launch(s, k_abi_to_state, nblk(len), 256, 0, rhs, s->Rv, n3, B, -1);
    LAUNCH_CHECK(s);
    apply_Ainv(s, B, s->Rv, s->Z, nullptr, 1.0, 0.0, nullptr);
    pdl_launch(s, k_state_to_abi, nblk(len), 256, 0, s->Z, out, n3, B, n3);
    LAUNCH_CHECK(s);
    CK(cudaStreamSynchronize(s->stream));
  } catch (CudaError& e) {
    return fail(s, PD_ERR_CUDA, e.what());
  }
  return PD_OK;
}

pd_status pd_apply_AN(pd_sim* s, int32_t B, const double* x, const double* youngs_per_sim, const double* act,
                      const double* p, double* out, void* cuda_stream) {
  if (!s) return PD_ERR_INVALID_ARGUMENT;
  if (B < 1 || B > s->Bmax || !x || !p || !out) return fail(s, PD_ERR_INVALID_ARGUMENT, "bad arguments");
  if (s->w_m != 0.0 && !act) return fail(s, PD_ERR_INVALID_ARGUMENT, "muscle energy needs act");
  s->stream = (cudaStream_t)cuda_stream;
  const HostPlan& P = s->plan;
  const int n3 = 3 * P.n;
  const int64_t len = (int64_t)n3 * B;
  try {
    set_w(s, B, youngs_per_sim, true);
    pdl_launch(s, k_abi_to_state, nblk(len), 256, 0, x, s->X, n3, B, -1);
    LAUNCH_CHECK(s);
    pdl_launch(s, k_abi_to_state, nblk(len), 256, 0, p, s->Pv, n3, B, -1);
    LAUNCH_CHECK(s);
    pdl_launch(s, k_elem_AN, nblk((int64_t)P.m * B * 8, 256), 256, 0, s->X, s->Pv, s->st, elem_args(s, B, act, P.m), s->EF);
    LAUNCH_CHECK(s);
    if (s->st.kappa != 0.0) {
      pdl_launch(s, k_vol<2>, nblk((int64_t)P.m * B * 8, 256), 256, 0, s->X, s->Pv, s->st, elem_args(s, B, act, P.m),
                                                                      nullptr, s->EF, nullptr);
      LAUNCH_CHECK(s);
    }
    pdl_launch(s, k_gather, nblk((int64_t)P.n * B), 256, 0, s->Pv, nullptr, s->EF, s->d_mass, s->d_inc_ptr, s->d_inc_ec,
                                                            s->d_nofix, s->d_pos, P.n, B, 1.0 / (s->h * s->h), 1, s->Q,
                                                            nullptr, nullptr, nullptr, nullptr, nullptr, 0);
    LAUNCH_CHECK(s);
    pdl_launch(s, k_state_to_abi, nblk(len), 256, 0, s->Q, out, n3, B, n3);
    LAUNCH_CHECK(s);
    CK(cudaStreamSynchronize(s->stream));
  } catch (CudaError& e) {
    return fail(s, PD_ERR_CUDA, e.what());
  }
  return PD_OK;
}

pd_status pd_project_rotations(pd_sim* s, int32_t B, const double* x, double* R, void* cuda_stream) {
  if (!s) return PD_ERR_INVALID_ARGUMENT;
  if (B < 1 || B > s->Bmax || !x || !R) return fail(s, PD_ERR_INVALID_ARGUMENT, "bad arguments");
  s->stream = (cudaStream_t)cuda_stream;
  const HostPlan& P = s->plan;
  const int n3 = 3 * P.n;
  const int64_t len = (int64_t)n3 * B;
  try {
    pdl_launch(s, k_abi_to_state, nblk(len), 256, 0, x, s->X, n3, B, -1);
    LAUNCH_CHECK(s);
    pdl_launch(s, k_elem_rotations, nblk((int64_t)P.m * B, 128), 128, 0, s->X, s->st, s->d_hex8, P.m, B, R);
    LAUNCH_CHECK(s);
    CK(cudaStreamSynchronize(s->stream));
  } catch (CudaError& e) {
    return fail(s, PD_ERR_CUDA, e.what());
  }
  return PD_OK;
}

pd_status pd_polar_stats(pd_sim* s, int32_t B, const double* x, int64_t* out, void* cuda_stream) {
  if (!s) return PD_ERR_INVALID_ARGUMENT;
  if (B < 1 || B > s->Bmax || !x || !out) return fail(s, PD_ERR_INVALID_ARGUMENT, "bad arguments");
  s->stream = (cudaStream_t)cuda_stream;
  const HostPlan& P = s->plan;
  const int n3 = 3 * P.n;
  const int64_t len = (int64_t)n3 * B;
  try {
    pdl_launch(s, k_abi_to_state, nblk(len), 256, 0, x, s->X, n3, B, -1);
    LAUNCH_CHECK(s);
    unsigned long long* acc = reinterpret_cast<unsigned long long*>(s->nactive_ll);
    CK(cudaMemsetAsync(acc, 0, 3 * sizeof(unsigned long long), s->stream));
    pdl_launch(s, k_polar_stats, nblk((int64_t)P.m * B * 8, 256), 256, 0, s->X, s->st, s->d_hex8, P.m, B, acc);
    LAUNCH_CHECK(s);
    unsigned long long h[3];
    CK(cudaMemcpyAsync(h, acc, sizeof(h), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    for (int k = 0; k < 3; ++k) out[k] = (int64_t)h[k];
  } catch (CudaError& e) {
    return fail(s, PD_ERR_CUDA, e.what());
  }
  return PD_OK;
}

}  // extern "C"
