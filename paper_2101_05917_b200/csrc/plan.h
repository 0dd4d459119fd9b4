// Internal host-side plan of a pd_sim: mesh stencil, ordering, supernodal factor
// of the scalar PD matrix A_s (A = A_s (x) I_3) and the level
// schedule of the batched triangular solves.  Host-only (no CUDA types).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace pdb {

// Packed per-item record of a K3 sweep (one 32-byte load on the device): v[0] = a_off / 32, v[1] = nk | nkd << 16,
// v[2] = zrow, v[3] = zidx, v[4] = out, v[5] = nvalid | (first-of-chain) << 8 | (last-of-chain) << 9, v[6] = the
// first item of the chain after this item's chain on the same CTA is looked up separately (unused), v[7] unused.
struct alignas(32) int4x2 {
  int32_t v[8];
};

// Position of factor element (k, lane) inside a sweep item's block (k padded to a multiple of 4). The block
// is stored in the fragment order of the fp64 MMA m8n8k4 with output row/col `lane` = 4 g + m (g = lane / 4
// is the fragment's group, m = lane % 4 its M-tile): for k-group q = k / 4 and half h = m / 2, the 32 lanes
// (g, t = k % 4) of a warp each read one contiguous double2 {m = 2h, 2h + 1} — one conflict-free 128-bit
// shared-memory load per (q, h). The device kernels restate this index arithmetic (kernels.cu).
inline int64_t sweep_frag_pos(int k, int lane) {
  const int q = k >> 2, t = k & 3, g = lane >> 2, m = lane & 3;
  return ((int64_t)(q * 2 + (m >> 1)) * 32 + g * 4 + t) * 2 + (m & 1);
}

struct HostPlan {
  // ---- mesh ----
  int n = 0, m = 0;
  double dx = 0, h = 0;
  std::vector<double> rest;         // [n][3]
  std::vector<int32_t> hex8;        // [m][8]
  std::vector<double> node_mass;    // [n] lumped
  std::vector<uint8_t> fixed_node;  // [n]
  double dN[8][8][3];               // dN[q][a][j] = dN_a/dX_j at Gauss point q
  double Kc[8][8];                  // sum_q V dN_a . dN_b            (corotated, unit w)
  double Km[8][8];                  // sum_q V (dN_a.m)(dN_b.m)       (muscle, unit w_m)
  double Tm[8][8][3][3];            // sum_q V dN_a dN_b^T: per-element muscle blocks m_e^T Tm[a][b] m_e
  std::vector<double> fib;          // [m][3] unit per-element fibers (empty = the uniform fiber); set before build_plan
  double w_ref = 0, w_m = 0;        // weights of the factorised A
  // node -> incident (element, corner) CSR sorted by element (deterministic gather)
  std::vector<int32_t> inc_ptr, inc_ec;  // ec = 8*e + a
  // ---- ordering ----
  int nfree = 0;
  std::vector<int32_t> pos_of_node;  // [n] solver position or -1 (fixed)
  std::vector<int32_t> node_of_pos;  // [nfree]
  // ---- scalar A_s over free nodes in solver order (CSR, full symmetric) ----
  std::vector<int64_t> a_ptr;
  std::vector<int32_t> a_col;
  std::vector<double> a_val;
  // ---- supernodes (ND tree; children precede parents) ----
  int nsup = 0;
  std::vector<int32_t> sfirst, ssize, parent, height;
  std::vector<int64_t> rptr;         // [nsup+1] into rows
  std::vector<int32_t> rows;         // below-block row positions (sorted, > last col)
  std::vector<int64_t> doff, poff;   // offsets of D_s (packed lower, = L_ss^{-1}) and W_s
  std::vector<double> D, P;          // P holds W_s = L[R_s, J_s] L_ss^{-1} row-major (nr x ns)
  int64_t nnzL = 0;                  // stored entries of L_s (diag blocks packed + panels)
  double factor_flops = 0, factor_ms = 0;
  // ---- solve schedule (K3): per level and sweep, work items over a factor stream in
  // MMA fragment order (element (k, lane) of item t at a_off[t] + sweep_frag_pos(k, lane)).  An item is at
  // most 128 k-steps (one TMA round); a CHAIN is a run of consecutive items accumulating into the same
  // 32-lane output on one CTA.  A chain whose output is shared (forward W rows of several supernodes of a
  // level, outputs split over several chains) writes partial rows; the level's reduce launch sums them in
  // a fixed order into their targets — deterministic, no atomics.
  int nlevels = 0;
  struct Sweep {
    std::vector<double> A;             // factor stream in item order
    std::vector<int32_t> lvl_item;     // [nlevels+1] items of level l: [lvl_item[l], lvl_item[l+1])
    std::vector<int32_t> lvl_chain;    // [nlevels+1] chains of level l
    std::vector<int32_t> chain;        // [nchains+1] first item of each chain (chain c = [chain[c], chain[c+1]))
    std::vector<int32_t> lvl_kmax;     // [nlevels] largest item (k-steps, padded to 4) of level l
    std::vector<int64_t> a_off;        // per item
    std::vector<int32_t> nk;           // k-steps
    std::vector<int32_t> nkd;          // k < nkd: source row zrow + k of the contiguous source
    std::vector<int32_t> zrow;         //   (z forward, y backward); k >= nkd: row rows[zidx + k - nkd]
    std::vector<int64_t> zidx;         //   of the indirect source (x backward: x[R_s])
    std::vector<int32_t> out;          // per item (same for a chain): >= 0: direct output row out + lane;
                                       //   < 0: partial rows (-out-1)*32 + lane
    std::vector<int32_t> nvalid;       // valid lanes
    std::vector<int4x2> rec;           // per item, packed for one 32-byte device load (see build_solve_schedule)
    std::vector<int32_t> lvl_red;      // [nlevels+1] reduce targets of level l
    std::vector<int32_t> red_row;      // target row (solve position)
    std::vector<int32_t> red_mode;     // 0: dst[row] = sum (y or x), 1: z[row] -= sum
    std::vector<int32_t> red_ptr;      // [ntargets+1] into red_src
    std::vector<int32_t> red_src;      // partial row indices, summed in this order
    int64_t max_partial_rows = 0;      // partial rows of the largest level
  } fw, bw;
  int chain_ctas = 148 * 4;            // CTAs a level launch is balanced for (chain length cap)
  // ---- K3 v4 schedule (round 2): per level and sweep, the outputs are 32-lane tiles whose
  // k-sequences are cut into k-groups of 4 k-steps (one 1 KB block of the stream each, MMA fragment order); the
  // level's k-groups are stored tile after tile and split into equal contiguous ranges, one per warp ("stream-K":
  // every warp streams the same number of bytes).  A PIECE is the part of one tile inside one warp's range: a
  // piece covering its whole (direct-eligible) tile writes its output rows directly, every other piece writes a
  // 32-row partial slot that the level's reduce adds, in piece order, into its target rows (deterministic).
  int k3_version = 3;                  // 3: chain/item schedule (fw, bw above); 4: warp-range schedule (fw4, bw4)
  int k3_warps = 148 * 8;              // warps a v4 level launch is split for
  // v4: the root's two dependent triangular products (forward y = D z, backward x = D^T y) replaced by ONE dense
  // product x_root = S^{-1} z_root, S^{-1} = D_root^T D_root (the inverse Schur complement onto the root, same
  // bytes as the two triangles): the forward sweep has no root level and the backward sweep's first level reads
  // z_root from the x buffer (the two share it) and assigns x_root through its reduce
  bool merge_root = true;
  std::vector<double> Sinv;          // [ns_root][ns_root] row-major, when merge_root
  struct Sweep4 {
    std::vector<double> A;             // k-groups (128 doubles each) of all levels, level-major, tile-major
    std::vector<int32_t> lvl_g;        // [nlevels+1] first global k-group of each level
    std::vector<int32_t> krow;         // [4 per k-group] right-hand-side row of each k-step: v >= 0 row v of source
                                       //   A (z forward, y backward); v <= -2 row -2-v of source B (x backward);
                                       //   -1 padding (zero factor column)
    std::vector<int32_t> lvl_piece;    // [nlevels+1] pieces of level l
    std::vector<int32_t> pstart, pkg;  // per piece: first global k-group, k-groups
    std::vector<int32_t> pout;         // >= 0: direct output row of lane 0; < 0: partial slot -1-pout
    std::vector<int32_t> pnv;          // valid lanes (output rows)
    std::vector<int32_t> lvl_warp;     // [nlevels+1] offsets into wg / wpiece; level l uses W_l = lvl_warp[l+1] -
                                       //   lvl_warp[l] - 1 warps
    std::vector<int32_t> wg;           // warp range starts (global k-group), W_l + 1 per level (last = level end)
    std::vector<int32_t> wpiece;       // first piece of each warp range (same indexing as wg)
    std::vector<int32_t> lvl_red, red_row, red_mode, red_ptr, red_src;  // reduce, as in Sweep
    int64_t max_partial_rows = 0;
  } fw4, bw4;
  // ---- contact candidates: ordered LAST as one root supernode ----
  int nc = 0;                        // number of candidate nodes (0 = no contact)
  int csup = -1;                     // index of the candidate supernode (= nsup - 1)
  std::vector<int32_t> cand_node;    // [nc] node of candidate j (caller order)
  std::vector<int32_t> cand_loc;     // [nc] local row of candidate j inside the root block
  std::vector<int32_t> cand_of_loc;  // [nc] inverse of cand_loc
  std::vector<int32_t> cand_of_node; // [n]  j or -1
  std::vector<double> Scc;           // [nc][nc] Schur complement of A_s onto the candidates (local order)
};

// Build everything host-side.  Returns "" on success, else an error message;
// *numerical is set when the failure is a non-SPD pivot.
std::string build_plan(HostPlan& P, int n, int m, const double* rest, const int32_t* hex8,
                       double dx, double density, double h, const int32_t* fixed_dofs,
                       int n_fixed, double w_ref, double w_m, const double fiber[3],
                       const int32_t* contact_nodes, int n_contact, bool* numerical);

}  // namespace pdb
