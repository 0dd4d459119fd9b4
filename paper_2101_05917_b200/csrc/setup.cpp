// Host setup of the B200 DiffPD path (timed separately from the hot path).
//
//  * voxel-mesh validation, 8-point Gauss stencil of the trilinear hex (reading
//    DESIGN.md §2.1), lumped mass;
//  * the scalar PD matrix A_s = M_s/h^2 + sum_e sum_q V (w dN_a.dN_b + w_m (dN_a.m)(dN_b.m)):
//    since G maps every coordinate axis identically for the corotated and the
//    muscle energies, A = M/h^2 + sum w G^T G equals A_s (x) I_3
//    exactly, and its Cholesky factor is L_s (x) I_3;
//  * geometric nested dissection on the voxel lattice, ND-tree supernodes,
//    multifrontal numeric Cholesky computed ONCE, diagonal blocks
//    stored inverted (D_s = L_ss^{-1}) so the per-iteration solves are products;
//  * the level schedule (tiles + forward update blocks) of the batched solves.
#include "plan.h"

#include <algorithm>
#include <array>
#include <climits>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <tuple>
#include <numeric>
#include <omp.h>

namespace pdb {
namespace {

// Max nodes in an ND leaf.  Every ND level costs the batched solve a fixed ~15-20 us on the B200 (one product
// launch + one reduce), while larger leaves add fill: on large meshes (>= 32768 free nodes) leaves
// of 128 nodes remove two levels for +7.5% nnz(L_s) (c5: 13 -> 11 levels, A^-1 519 -> 477 us measured); small
// meshes, whose factor is L2-resident, keep 48 (c3: 48 -> 128 measured slower).  PD_ND_LEAF overrides.
int nd_leaf(int nfree) {
  if (const char* e = std::getenv("PD_ND_LEAF")) return std::max(2, std::atoi(e));
  return nfree >= 32768 ? 128 : 48;
}

struct NDNode {
  std::vector<int32_t> nodes;  // mesh node ids in final order
  int left = -1, right = -1;
};

}  // namespace

static void stencil(HostPlan& P, const double fiber[3]) {
  const double g = 1.0 / std::sqrt(3.0);
  for (int q = 0; q < 8; ++q) {
    const double xi[3] = {(2 * (q & 1) - 1) * g, (2 * ((q >> 1) & 1) - 1) * g,
                          (2 * ((q >> 2) & 1) - 1) * g};
    for (int a = 0; a < 8; ++a) {
      const double s[3] = {double(2 * (a & 1) - 1), double(2 * ((a >> 1) & 1) - 1),
                           double(2 * ((a >> 2) & 1) - 1)};
      for (int j = 0; j < 3; ++j) {
        double v = s[j] / 8.0;
        for (int k = 0; k < 3; ++k)
          if (k != j) v *= (1.0 + s[k] * xi[k]);
        P.dN[q][a][j] = v * 2.0 / P.dx;
      }
    }
  }
  const double V = P.dx * P.dx * P.dx / 8.0;
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 8; ++b) {
      double kc = 0, km = 0;
      for (int q = 0; q < 8; ++q) {
        double dd = 0, ma = 0, mb = 0;
        for (int j = 0; j < 3; ++j) {
          dd += P.dN[q][a][j] * P.dN[q][b][j];
          ma += P.dN[q][a][j] * fiber[j];
          mb += P.dN[q][b][j] * fiber[j];
        }
        kc += V * dd;
        km += V * ma * mb;
      }
      P.Kc[a][b] = kc;
      P.Km[a][b] = km;
      for (int j = 0; j < 3; ++j)
        for (int k = 0; k < 3; ++k) {
          double t = 0;
          for (int q = 0; q < 8; ++q) t += V * P.dN[q][a][j] * P.dN[q][b][k];
          P.Tm[a][b][j][k] = t;
        }
    }
}

// ---------------------------------------------------------------- dense kernels
// Front F is row-major f x f (lower triangle used).
static bool potrf_lower(double* F, int f, int ns, bool par) {
  // Right-looking column Cholesky of the leading ns x ns block, rows ns.. get L21.
  for (int j = 0; j < ns; ++j) {
    double d = F[(int64_t)j * f + j];
    if (!(d > 0.0) || !std::isfinite(d)) return false;
    d = std::sqrt(d);
    F[(int64_t)j * f + j] = d;
    const double inv = 1.0 / d;
    for (int i = j + 1; i < f; ++i) F[(int64_t)i * f + j] *= inv;
    // update columns j+1..ns-1 of all rows below (within the first ns columns)
#pragma omp parallel for schedule(dynamic, 16) if (par && (f - j) > 256)
    for (int i = j + 1; i < f; ++i) {
      const double lij = F[(int64_t)i * f + j];
      if (lij == 0.0) continue;
      double* Fi = F + (int64_t)i * f;
      const int kmax = std::min(i, ns - 1);
      for (int k = j + 1; k <= kmax; ++k) Fi[k] -= lij * F[(int64_t)k * f + j];
    }
  }
  return true;
}

// Blocked variant for large fronts: factor panels of nb columns, then update.
static bool partial_cholesky(double* F, int f, int ns, bool par) {
  const int nb = 64;
  if (ns <= nb || f < 512) return potrf_lower(F, f, ns, par);
  for (int j0 = 0; j0 < ns; j0 += nb) {
    const int j1 = std::min(ns, j0 + nb);
    // factor the panel columns j0..j1 (unblocked, only within the panel)
    for (int j = j0; j < j1; ++j) {
      double d = F[(int64_t)j * f + j];
      if (!(d > 0.0) || !std::isfinite(d)) return false;
      d = std::sqrt(d);
      F[(int64_t)j * f + j] = d;
      const double inv = 1.0 / d;
      for (int i = j + 1; i < f; ++i) F[(int64_t)i * f + j] *= inv;
#pragma omp parallel for schedule(static) if (par && (f - j) > 1024)
      for (int i = j + 1; i < f; ++i) {
        double* Fi = F + (int64_t)i * f;
        const double lij = Fi[j];
        const int kmax = std::min(i, j1 - 1);
        for (int k = j + 1; k <= kmax; ++k) Fi[k] -= lij * F[(int64_t)k * f + j];
      }
    }
    // trailing update of columns j1..ns-1 (rows >= j1): F[i][k] -= sum_{j in panel} L[i][j] L[k][j]
#pragma omp parallel for schedule(dynamic, 8) if (par)
    for (int i = j1; i < f; ++i) {
      double* Fi = F + (int64_t)i * f;
      const int kmax = std::min(i, ns - 1);
      for (int k = j1; k <= kmax; ++k) {
        const double* Fk = F + (int64_t)k * f;
        double s = 0;
        for (int j = j0; j < j1; ++j) s += Fi[j] * Fk[j];
        Fi[k] -= s;
      }
    }
  }
  return true;
}

// U = F22 - L21 L21^T (lower), F22 = F[ns.., ns..], L21 = F[ns.., 0..ns)
static void schur_update(double* F, int f, int ns, bool par) {
  const int nr = f - ns;
  if (nr <= 0) return;
  const int bs = 48;
#pragma omp parallel for schedule(dynamic, 1) if (par && nr > 64)
  for (int ib = 0; ib < nr; ib += bs) {
    const int ie = std::min(nr, ib + bs);
    for (int kb = 0; kb <= ib; kb += bs) {
      const int ke = std::min(nr, kb + bs);
      for (int jb = 0; jb < ns; jb += 256) {
        const int je = std::min(ns, jb + 256);
        for (int i = ib; i < ie; ++i) {
          double* Fi = F + (int64_t)(ns + i) * f;
          const int kk = std::min(ke - 1, i);
          for (int k = kb; k <= kk; ++k) {
            const double* Fk = F + (int64_t)(ns + k) * f;
            double s = 0;
            for (int j = jb; j < je; ++j) s += Fi[j] * Fk[j];
            Fi[ns + k] -= s;
          }
        }
      }
    }
  }
}

// D = L11^{-1} packed lower (row i at i(i+1)/2), from the ns x ns block of F.
static void tri_inverse(const double* F, int f, int ns, double* D, bool par) {
#pragma omp parallel for schedule(dynamic, 4) if (par && ns > 128)
  for (int c = 0; c < ns; ++c) {
    // column c of X: X[c][c] = 1/L[c][c]; X[i][c] = -(sum_{k=c}^{i-1} L[i][k] X[k][c]) / L[i][i]
    D[(int64_t)c * (c + 1) / 2 + c] = 1.0 / F[(int64_t)c * f + c];
    for (int i = c + 1; i < ns; ++i) {
      const double* Fi = F + (int64_t)i * f;
      double s = 0;
      for (int k = c; k < i; ++k) s += Fi[k] * D[(int64_t)k * (k + 1) / 2 + c];
      D[(int64_t)i * (i + 1) / 2 + c] = -s / Fi[i];
    }
  }
}

// ---------------------------------------------------------------- solve schedule
// Forward sweep, level l (children before parents), for every level-l supernode s (z[J_s] final):
//   D outputs: y[J_s rows i0..i0+32) = D_s[rows, 0..min(i0+32, ns)) z[J_s]      (lane = row)
//   W outputs: W_s[rows i0..i0+32 of R_s, :] z[J_s] -> partial rows; reduce: z[R_s[i]] -= sum
// Backward sweep, level l (parents first), column chunk c0..c0+32 of s:
//   x[J_s cols] = D_s^T y[J_s] - W_s^T x[R_s]     (k-sequence [D part c0..ns | W part 0..nr]; lane = column)
// An output's k-sequence is cut into items of <= 128 k-steps (one TMA round each) grouped into chains of
// <= CL items that accumulate on one CTA; CL balances the level's items over chain_ctas CTAs.  An output
// covered by one chain is written directly (D, backward); otherwise each chain writes partial rows and the
// level's reduce sums them in chain order.
static void build_solve_schedule(HostPlan& P, const std::vector<std::vector<int32_t>>& byh) {
  const int L = 32, KC = 128;
  for (HostPlan::Sweep* S : {&P.fw, &P.bw}) {
    *S = HostPlan::Sweep();
    S->lvl_item.assign(1, 0);
    S->lvl_chain.assign(1, 0);
    S->lvl_red.assign(1, 0);
    S->red_ptr.assign(1, 0);
  }
  auto Dval = [&](int s, int i, int k) -> double {  // D_s[i][k], packed lower
    return k <= i ? P.D[P.doff[s] + (int64_t)i * (i + 1) / 2 + k] : 0.0;
  };
  auto Wval = [&](int s, int i, int k) -> double {  // W_s[i][k], row-major nr x ns
    return P.P[P.poff[s] + (int64_t)i * P.ssize[s] + k];
  };
  // one item: the block val(k, lane), k = 0..nk, lane = output row/col 0..31, in the fragment layout of the
  // fp64 tensor-core MMA (m8n8k4; plan.h sweep_frag_pos): k padded with zeros to a multiple of 4
  auto emit_item = [&](HostPlan::Sweep& S, int nk, int nv, int zr, int64_t zi, int nkd, int out, auto&& val) {
    const int64_t base = (int64_t)S.A.size();
    S.a_off.push_back(base);
    const int nkp = (nk + 3) & ~3;
    S.A.resize(base + (int64_t)nkp * L, 0.0);
    for (int k = 0; k < nk; ++k)
      for (int l = 0; l < nv; ++l) S.A[base + sweep_frag_pos(k, l)] = val(k, l);
    S.nk.push_back(nk);
    S.nkd.push_back(nkd);
    S.zrow.push_back(zr);
    S.zidx.push_back(zi);
    S.nvalid.push_back(nv);
    S.out.push_back(out);
  };
  // one output (nv lanes) over a k-sequence of ktot steps; src(p0, nk) -> {zrow, zidx, nkd} of the item at
  // p0; val(p, lane) = factor entry at sequence position p.  Direct (direct_row >= 0 and one chain) or
  // partial rows, whose bases (one per chain) are returned in order.
  auto emit_output = [&](HostPlan::Sweep& S, int CL, int ktot, int nv, int direct_row, int64_t& prow, auto&& src,
                         auto&& val) {
    std::vector<int64_t> bases;
    const int nit = std::max(1, (ktot + KC - 1) / KC);
    const int nch = (nit + CL - 1) / CL;
    const int per = (nit + nch - 1) / nch;  // items per chain, balanced
    const bool direct = direct_row >= 0 && nch == 1;
    for (int it = 0; it < nit; ++it) {
      int out = direct_row;
      if (it % per == 0) {
        S.chain.push_back((int32_t)S.a_off.size());
        if (!direct) {
          bases.push_back(prow);
          prow += L;
        }
      }
      if (!direct) out = -(int32_t)(bases.back() / L) - 1;
      const int p0 = it * KC, nk = std::max(0, std::min(KC, ktot - p0));
      const std::array<int64_t, 3> zs = src(p0, nk);
      emit_item(S, nk, nv, (int)zs[0], zs[1], (int)zs[2], out, [&](int k, int l) { return val(p0 + k, l); });
    }
    return bases;
  };
  constexpr int kChainNoSplit = 4;  // outputs of <= 4 items stay on one CTA in the backward sweep
  // chains only where a level has many more items than CTAs (fewer partial rows, still >= 4 items per CTA)
  auto chain_cap = [&](int64_t items) { return (int)std::max<int64_t>(1, items / (4 * (int64_t)P.chain_ctas)); };
  auto close_level = [&](HostPlan::Sweep& S, int64_t prow,
                         std::vector<std::tuple<int32_t, int32_t, std::vector<int32_t>>>& targets) {
    // targets (row, mode, partial rows in summation order), sorted by row: the level's reduce
    std::stable_sort(targets.begin(), targets.end(),
                     [](const auto& x, const auto& y) { return std::get<0>(x) < std::get<0>(y); });
    for (auto& t : targets) {
      S.red_row.push_back(std::get<0>(t));
      S.red_mode.push_back(std::get<1>(t));
      for (int32_t r : std::get<2>(t)) S.red_src.push_back(r);
      S.red_ptr.push_back((int32_t)S.red_src.size());
    }
    targets.clear();
    S.lvl_red.push_back((int32_t)S.red_row.size());
    S.lvl_item.push_back((int32_t)S.a_off.size());
    S.lvl_chain.push_back((int32_t)S.chain.size());
    S.max_partial_rows = std::max(S.max_partial_rows, prow);
  };
  std::vector<std::tuple<int32_t, int32_t, std::vector<int32_t>>> targets;
  // ---- forward
  {
    HostPlan::Sweep& S = P.fw;
    for (int lev = 0; lev < P.nlevels; ++lev) {
      int64_t items = 0;
      for (int s : byh[lev]) {
        const int ns = P.ssize[s], nr = (int)(P.rptr[s + 1] - P.rptr[s]);
        for (int i0 = 0; i0 < ns; i0 += L) items += (std::min(i0 + L, ns) + KC - 1) / KC;
        items += (int64_t)((nr + L - 1) / L) * ((ns + KC - 1) / KC);
      }
      const int CL = chain_cap(items);
      int64_t prow = 0;  // partial rows are reused level by level (the reduce consumes them first)
      std::map<int32_t, std::vector<int32_t>> wsum;  // target row -> partial rows (emission order)
      for (int s : byh[lev]) {
        const int ns = P.ssize[s], f = P.sfirst[s];
        const int nr = (int)(P.rptr[s + 1] - P.rptr[s]);
        for (int i0 = 0; i0 < ns; i0 += L) {  // D outputs
          const int kend = std::min(i0 + L, ns), nv = std::min(L, ns - i0);
          auto bases = emit_output(
              S, CL, kend, nv, f + i0, prow,
              [&](int p0, int) { return std::array<int64_t, 3>{f + p0, 0, std::min(KC, kend - p0)}; },
              [&](int p, int l) { return Dval(s, i0 + l, p); });
          if (!bases.empty())
            for (int l = 0; l < nv; ++l) {
              std::vector<int32_t> src;
              for (int64_t b : bases) src.push_back((int32_t)(b + l));
              targets.emplace_back(f + i0 + l, 0, std::move(src));
            }
        }
        for (int i0 = 0; i0 < nr; i0 += L) {  // W outputs (always partial: targets shared across supernodes)
          const int nv = std::min(L, nr - i0);
          auto bases = emit_output(
              S, CL, ns, nv, -1, prow,
              [&](int p0, int) { return std::array<int64_t, 3>{f + p0, 0, std::min(KC, ns - p0)}; },
              [&](int p, int l) { return Wval(s, i0 + l, p); });
          for (int l = 0; l < nv; ++l)
            for (int64_t b : bases) wsum[P.rows[P.rptr[s] + i0 + l]].push_back((int32_t)(b + l));
        }
      }
      for (auto& kv : wsum) targets.emplace_back(kv.first, 1, std::move(kv.second));
      close_level(S, prow, targets);
    }
  }
  // ---- backward (levels top-down; stored in that execution order: level index = H - l)
  {
    HostPlan::Sweep& S = P.bw;
    for (int lev = P.nlevels - 1; lev >= 0; --lev) {
      int64_t items = 0;
      int lmax = 1;  // longest output (items)
      for (int s : byh[lev]) {
        const int ns = P.ssize[s], nr = (int)(P.rptr[s + 1] - P.rptr[s]);
        for (int c0 = 0; c0 < ns; c0 += L) {
          const int nit = ((ns - c0) + nr + KC - 1) / KC;
          items += nit;
          lmax = std::max(lmax, nit);
        }
      }
      // chains long enough that no output of the level is split (no partial rows, no reduce launch) when the
      // longest output is short; else the balance cap
      const int CL = std::max(chain_cap(items), lmax <= kChainNoSplit ? lmax : 1);
      int64_t prow = 0;
      for (int s : byh[lev]) {
        const int ns = P.ssize[s], f = P.sfirst[s];
        const int nr = (int)(P.rptr[s + 1] - P.rptr[s]);
        for (int c0 = 0; c0 < ns; c0 += L) {
          const int nv = std::min(L, ns - c0);
          // k-sequence = [D part: rows c0..ns of D_s | W part: rows 0..nr of W_s]
          const int nd = ns - c0, ktot_c = nd + nr;
          auto bases = emit_output(
              S, CL, ktot_c, nv, f + c0, prow,
              [&](int p0, int nk) {
                return std::array<int64_t, 3>{f + c0 + p0, P.rptr[s] + std::max(0, p0 - nd),
                                              std::max(0, std::min(nk, nd - p0))};
              },
              [&](int q, int l) { return q < nd ? Dval(s, c0 + q, c0 + l) : -Wval(s, q - nd, c0 + l); });
          if (!bases.empty())
            for (int l = 0; l < nv; ++l) {
              std::vector<int32_t> src;
              for (int64_t b : bases) src.push_back((int32_t)(b + l));
              targets.emplace_back(f + c0 + l, 0, std::move(src));
            }
        }
      }
      close_level(S, prow, targets);
    }
  }
  for (HostPlan::Sweep* S : {&P.fw, &P.bw}) {
    S->chain.push_back((int32_t)S->a_off.size());  // sentinel
    // Within a level, chains are independent: lay them out longest first, so that the static round-robin
    // assignment (CTA c takes chains c, c + G, ...) gives every CTA one of the long chains before any gets a
    // second chain (balance without knowing G).  Items move with their chain; outputs are unchanged.
    {
      HostPlan::Sweep T = *S;
      T.A.clear();
      T.a_off.clear();
      T.nk.clear();
      T.nkd.clear();
      T.zrow.clear();
      T.zidx.clear();
      T.out.clear();
      T.nvalid.clear();
      T.chain.clear();
      for (int l = 0; l < P.nlevels; ++l) {
        std::vector<int32_t> order;
        for (int c = S->lvl_chain[l]; c < S->lvl_chain[l + 1]; ++c) order.push_back(c);
        std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
          return S->chain[x + 1] - S->chain[x] > S->chain[y + 1] - S->chain[y];
        });
        for (int32_t c : order) {
          T.chain.push_back((int32_t)T.a_off.size());
          for (int t = S->chain[c]; t < S->chain[c + 1]; ++t) {
            const int64_t len = (int64_t)((S->nk[t] + 3) & ~3) * L;
            T.a_off.push_back((int64_t)T.A.size());
            T.A.insert(T.A.end(), S->A.begin() + S->a_off[t], S->A.begin() + S->a_off[t] + len);
            T.nk.push_back(S->nk[t]);
            T.nkd.push_back(S->nkd[t]);
            T.zrow.push_back(S->zrow[t]);
            T.zidx.push_back(S->zidx[t]);
            T.out.push_back(S->out[t]);
            T.nvalid.push_back(S->nvalid[t]);
          }
        }
      }
      T.chain.push_back((int32_t)T.a_off.size());
      *S = std::move(T);
    }
    const size_t ni = S->a_off.size();
    S->rec.assign(ni, int4x2{});
    std::vector<uint8_t> first(ni, 0), last(ni, 0);
    for (size_t c = 0; c + 1 < S->chain.size(); ++c) {
      first[S->chain[c]] = 1;
      last[S->chain[c + 1] - 1] = 1;
    }
    for (size_t t = 0; t < ni; ++t) {
      int32_t* v = S->rec[t].v;
      v[0] = (int32_t)(S->a_off[t] / 32);
      v[1] = S->nk[t] | (S->nkd[t] << 16);
      v[2] = S->zrow[t];
      v[3] = (int32_t)S->zidx[t];
      v[4] = S->out[t];
      v[5] = S->nvalid[t] | (first[t] << 8) | (last[t] << 9);
    }
    S->lvl_kmax.assign(P.nlevels, 0);
    for (int l = 0; l < P.nlevels; ++l)
      for (int t = S->lvl_item[l]; t < S->lvl_item[l + 1]; ++t)
        S->lvl_kmax[l] = std::max(S->lvl_kmax[l], (S->nk[t] + 3) & ~3);
  }
}

// ---------------------------------------------------------------- K3 v4 schedule (warp ranges)
// Tiles of a level in stream order.  Forward, supernode s: D tiles (rows i0..i0+32 of D_s over columns
// 0..min(i0+32, ns), direct into y) then W tiles (rows i0..i0+32 of W_s over all ns columns, always partial: the
// target rows R_s are shared with other supernodes of the level; z[target] -= sum).  Backward: column tiles c0 of
// s over [D part: rows c0..ns of D_s | W part: rows 0..nr of W_s], direct into x[J_s].
static void build_warp_schedule(HostPlan& P, const std::vector<std::vector<int32_t>>& byh) {
  const int L = 32;
  auto Dval = [&](int s, int i, int k) -> double {  // D_s[i][k], packed lower
    return k <= i ? P.D[P.doff[s] + (int64_t)i * (i + 1) / 2 + k] : 0.0;
  };
  auto Wval = [&](int s, int i, int k) -> double { return P.P[P.poff[s] + (int64_t)i * P.ssize[s] + k]; };
  struct Tile {
    int s, a0, nk, nv, out, mode;  // a0: D row / W row / column start; out >= 0 direct row, -1 always partial
    int kind;                      // 0 forward D, 1 forward W, 2 backward column tile, 3 merged-root S^{-1} rows
  };
  const int root_lev = P.nlevels - 1;
  const bool merge = P.merge_root && (int)byh[root_lev].size() == 1;
  const int root = merge ? byh[root_lev][0] : -1;
  if (merge) {  // S^{-1} = D^T D over the root block (D = L_rr^{-1}, packed lower)
    const int ns = P.ssize[root];
    const double* D = P.D.data() + P.doff[root];
    P.Sinv.assign((size_t)ns * ns, 0.0);
#pragma omp parallel for schedule(dynamic, 8)
    for (int i = 0; i < ns; ++i)
      for (int j = 0; j <= i; ++j) {
        double acc = 0;
        for (int k = i; k < ns; ++k) acc += D[(int64_t)k * (k + 1) / 2 + i] * D[(int64_t)k * (k + 1) / 2 + j];
        P.Sinv[(size_t)i * ns + j] = P.Sinv[(size_t)j * ns + i] = acc;
      }
  } else {
    P.merge_root = false;
    P.Sinv.clear();
  }
  for (int fwd = 1; fwd >= 0; --fwd) {
    HostPlan::Sweep4& S = fwd ? P.fw4 : P.bw4;
    S = HostPlan::Sweep4();
    S.lvl_g.assign(1, 0);
    S.lvl_piece.assign(1, 0);
    S.lvl_warp.assign(1, 0);
    S.lvl_red.assign(1, 0);
    S.red_ptr.assign(1, 0);
    for (int li = 0; li < P.nlevels; ++li) {
      const int lev = fwd ? li : P.nlevels - 1 - li;  // backward levels in execution order (top down)
      std::vector<Tile> tiles;
      for (int s : byh[lev]) {
        const int ns = P.ssize[s], f = P.sfirst[s], nr = (int)(P.rptr[s + 1] - P.rptr[s]);
        if (s == root) {  // merged root: nothing in the forward sweep; backward rows of S^{-1}, all partial
          if (!fwd)
            for (int i0 = 0; i0 < ns; i0 += L) tiles.push_back({s, i0, ns, std::min(L, ns - i0), -1, 0, 3});
          continue;
        }
        if (fwd) {
          for (int i0 = 0; i0 < ns; i0 += L) tiles.push_back({s, i0, std::min(i0 + L, ns), std::min(L, ns - i0), f + i0, 0, 0});
          for (int i0 = 0; i0 < nr; i0 += L) tiles.push_back({s, i0, ns, std::min(L, nr - i0), -1, 1, 1});
        } else {
          for (int c0 = 0; c0 < ns; c0 += L) tiles.push_back({s, c0, (ns - c0) + nr, std::min(L, ns - c0), f + c0, 0, 2});
        }
      }
      // emit the tiles' k-groups (factor blocks + k-step source rows)
      const int g_lev = S.lvl_g.back();
      std::vector<int32_t> tile_g0(tiles.size() + 1, g_lev);
      for (size_t ti = 0; ti < tiles.size(); ++ti) {
        const Tile& T = tiles[ti];
        const int s = T.s, ns = P.ssize[s], f = P.sfirst[s];
        const int nkg = (T.nk + 3) / 4;
        const int64_t base = (int64_t)S.A.size();
        S.A.resize(base + (int64_t)nkg * 128, 0.0);
        for (int k = 0; k < nkg * 4; ++k) {
          int32_t row = -1;
          if (k < T.nk) {
            if (T.kind == 0 || T.kind == 1) row = f + k;
            else if (T.kind == 3) row = -2 - (f + k);  // z_root, read from the x buffer (source B)
            else row = k < ns - T.a0 ? f + T.a0 + k : -2 - P.rows[P.rptr[s] + (k - (ns - T.a0))];
          }
          S.krow.push_back(row);
          if (k >= T.nk) continue;
          double* blk = S.A.data() + base + (int64_t)(k / 4) * 128;
          for (int l = 0; l < T.nv; ++l) {
            double v;
            if (T.kind == 0) v = Dval(s, T.a0 + l, k);
            else if (T.kind == 1) v = Wval(s, T.a0 + l, k);
            else if (T.kind == 3) v = P.Sinv[(size_t)(T.a0 + l) * ns + k];
            else v = k < ns - T.a0 ? Dval(s, T.a0 + k, T.a0 + l) : -Wval(s, k - (ns - T.a0), T.a0 + l);
            blk[sweep_frag_pos(k & 3, l)] = v;
          }
        }
        tile_g0[ti + 1] = tile_g0[ti] + nkg;
      }
      const int G = tile_g0.back() - g_lev;
      S.lvl_g.push_back(g_lev + G);
      // equal contiguous warp ranges (>= 4 k-groups = one TMA stage per warp on average)
      const int W = std::max(1, std::min(P.k3_warps, G / 4));
      std::vector<int32_t> wb(W + 1);
      for (int w = 0; w <= W; ++w) wb[w] = g_lev + (int32_t)((int64_t)G * w / W);
      // pieces = tiles cut at the warp boundaries; partial slots numbered per level
      std::map<std::pair<int32_t, int32_t>, std::vector<int32_t>> targets;  // (mode, row) -> partial rows
      int64_t slot = 0;
      size_t ti = 0;
      const int p_lev0 = (int)S.pstart.size();
      for (int w = 0; w < W; ++w) {
        S.wg.push_back(wb[w]);
        S.wpiece.push_back((int32_t)S.pstart.size());
        int g = wb[w];
        while (g < wb[w + 1]) {
          while (tile_g0[ti + 1] <= g) ++ti;
          const Tile& T = tiles[ti];
          const int ge = std::min(wb[w + 1], tile_g0[ti + 1]);
          const bool whole = g == tile_g0[ti] && ge == tile_g0[ti + 1];
          S.pstart.push_back(g);
          S.pkg.push_back(ge - g);
          S.pnv.push_back(T.nv);
          if (whole && T.out >= 0) {
            S.pout.push_back(T.out);
          } else {
            S.pout.push_back((int32_t)(-1 - slot));
            for (int l = 0; l < T.nv; ++l) {
              const int32_t row = T.kind == 1   ? P.rows[P.rptr[T.s] + T.a0 + l]
                                  : T.kind == 3 ? P.sfirst[T.s] + T.a0 + l
                                                : T.out + l;
              targets[{T.mode, row}].push_back((int32_t)(slot * L + l));
            }
            ++slot;
          }
          g = ge;
        }
      }
      S.wg.push_back(wb[W]);
      S.wpiece.push_back((int32_t)S.pstart.size());
      S.lvl_warp.push_back((int32_t)S.wg.size());
      S.lvl_piece.push_back((int32_t)S.pstart.size());
      (void)p_lev0;
      for (auto& kv : targets) {  // sorted by (mode, row); sources in piece order
        S.red_row.push_back(kv.first.second);
        S.red_mode.push_back(kv.first.first);
        for (int32_t r : kv.second) S.red_src.push_back(r);
        S.red_ptr.push_back((int32_t)S.red_src.size());
      }
      S.lvl_red.push_back((int32_t)S.red_row.size());
      S.max_partial_rows = std::max<int64_t>(S.max_partial_rows, slot * L);
    }
  }
}

// ---------------------------------------------------------------- build
std::string build_plan(HostPlan& P, int n, int m, const double* rest, const int32_t* hex8,
                       double dx, double density, double h, const int32_t* fixed_dofs,
                       int n_fixed, double w_ref, double w_m, const double fiber[3],
                       const int32_t* contact_nodes, int n_contact, bool* numerical) {
  *numerical = false;
  if (n <= 0 || m <= 0 || !rest || !hex8) return "empty mesh";
  if (!(dx > 0) || !(h > 0)) return "dx and h must be > 0";
  P.n = n;
  P.m = m;
  P.dx = dx;
  P.h = h;
  P.w_ref = w_ref;
  P.w_m = w_m;
  P.rest.assign(rest, rest + 3 * (int64_t)n);
  P.hex8.assign(hex8, hex8 + 8 * (int64_t)m);
  // voxel check: corner a of element e sits at corner0 + dx (di, dj, dk)
  for (int e = 0; e < m; ++e) {
    const int32_t* c = hex8 + 8 * (int64_t)e;
    for (int a = 0; a < 8; ++a)
      if (c[a] < 0 || c[a] >= n) return "element " + std::to_string(e) + " has an out-of-range node";
    for (int a = 0; a < 8; ++a)
      for (int b = a + 1; b < 8; ++b)
        if (c[a] == c[b]) return "element " + std::to_string(e) + " repeats a node";
    const double* x0 = rest + 3 * (int64_t)c[0];
    for (int a = 1; a < 8; ++a) {
      const double off[3] = {double(a & 1), double((a >> 1) & 1), double((a >> 2) & 1)};
      for (int j = 0; j < 3; ++j)
        if (std::fabs(rest[3 * (int64_t)c[a] + j] - x0[j] - dx * off[j]) > 1e-9 * dx)
          return "element " + std::to_string(e) + " is not an axis-aligned voxel of edge dx";
    }
  }
  stencil(P, fiber);
  P.node_mass.assign(n, 0.0);
  for (int e = 0; e < m; ++e)
    for (int a = 0; a < 8; ++a) P.node_mass[hex8[8 * (int64_t)e + a]] += density * dx * dx * dx / 8.0;
  for (int i = 0; i < n; ++i)
    if (!(P.node_mass[i] > 0)) return "node " + std::to_string(i) + " belongs to no element";
  // fixed DoFs must cover whole nodes (A = A_s (x) I_3)
  P.fixed_node.assign(n, 0);
  {
    std::vector<uint8_t> fd(3 * (int64_t)n, 0);
    for (int k = 0; k < n_fixed; ++k) {
      if (fixed_dofs[k] < 0 || fixed_dofs[k] >= 3 * n) return "fixed DoF out of range";
      fd[fixed_dofs[k]] = 1;
    }
    for (int i = 0; i < n; ++i) {
      const int s = fd[3 * i] + fd[3 * i + 1] + fd[3 * i + 2];
      if (s != 0 && s != 3) return "fixed DoFs must fix all three axes of a node";
      P.fixed_node[i] = s == 3;
    }
  }
  // incidence (sorted by element id: the deterministic summation order of the gather)
  P.inc_ptr.assign(n + 1, 0);
  for (int e = 0; e < m; ++e)
    for (int a = 0; a < 8; ++a) P.inc_ptr[hex8[8 * (int64_t)e + a] + 1]++;
  for (int i = 0; i < n; ++i) P.inc_ptr[i + 1] += P.inc_ptr[i];
  P.inc_ec.assign(P.inc_ptr[n], 0);
  {
    std::vector<int32_t> fill(P.inc_ptr.begin(), P.inc_ptr.end() - 1);
    for (int e = 0; e < m; ++e)
      for (int a = 0; a < 8; ++a) P.inc_ec[fill[hex8[8 * (int64_t)e + a]]++] = 8 * e + a;
  }

  // ---------------- nested dissection on the lattice of free nodes
  double mn[3] = {1e300, 1e300, 1e300};
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < 3; ++j) mn[j] = std::min(mn[j], rest[3 * (int64_t)i + j]);
  std::vector<int32_t> lat(3 * (int64_t)n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < 3; ++j) lat[3 * (int64_t)i + j] = (int32_t)std::llround((rest[3 * (int64_t)i + j] - mn[j]) / dx);
  // contact candidates (P:278 the node set V): free nodes, no repeats; ordered LAST
  P.nc = n_contact;
  P.cand_of_node.assign(n, -1);
  P.cand_node.assign(contact_nodes, contact_nodes + n_contact);
  for (int j = 0; j < n_contact; ++j) {
    const int v = contact_nodes[j];
    if (v < 0 || v >= n) return "contact node out of range";
    if (P.fixed_node[v]) return "a contact candidate is a Dirichlet node";
    if (P.cand_of_node[v] >= 0) return "repeated contact candidate";
    P.cand_of_node[v] = j;
  }
  std::vector<int32_t> freeNodes;
  for (int i = 0; i < n; ++i)
    if (!P.fixed_node[i] && P.cand_of_node[i] < 0) freeNodes.push_back(i);
  P.nfree = (int)freeNodes.size() + n_contact;
  if (P.nfree == 0) return "every node is fixed";

  std::vector<std::vector<int32_t>> supNodes;  // in creation (post) order
  std::vector<int32_t> supParent;
  auto lexless = [&](int32_t a, int32_t b) {
    for (int j = 2; j >= 0; --j)
      if (lat[3 * (int64_t)a + j] != lat[3 * (int64_t)b + j]) return lat[3 * (int64_t)a + j] < lat[3 * (int64_t)b + j];
    return a < b;
  };
  const int leaf = nd_leaf(P.nfree);
  std::function<int(std::vector<int32_t>&)> nd = [&](std::vector<int32_t>& nodes) -> int {
    int lo[3] = {INT32_MAX, INT32_MAX, INT32_MAX}, hi[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
    for (int v : nodes)
      for (int j = 0; j < 3; ++j) {
        lo[j] = std::min(lo[j], lat[3 * (int64_t)v + j]);
        hi[j] = std::max(hi[j], lat[3 * (int64_t)v + j]);
      }
    int ax = 0;
    for (int j = 1; j < 3; ++j)
      if (hi[j] - lo[j] > hi[ax] - lo[ax]) ax = j;
    if ((int)nodes.size() <= leaf || hi[ax] - lo[ax] < 2) {
      std::sort(nodes.begin(), nodes.end(), lexless);
      supNodes.push_back(nodes);
      supParent.push_back(-1);
      return (int)supNodes.size() - 1;
    }
    // cut plane: the populated lattice coordinate strictly inside (lo, hi) closest to the middle
    std::vector<int> hist(hi[ax] - lo[ax] + 1, 0);
    for (int v : nodes) hist[lat[3 * (int64_t)v + ax] - lo[ax]]++;
    int c = INT32_MIN;
    const int mid = (lo[ax] + hi[ax]) / 2;
    for (int off = 0; off <= hi[ax] - lo[ax] && c == INT32_MIN; ++off)
      for (int sgn : {0, 1}) {
        const int cc = sgn ? mid + off : mid - off;
        if (cc > lo[ax] && cc < hi[ax] && hist[cc - lo[ax]] > 0) { c = cc; break; }
      }
    if (c == INT32_MIN) {  // cannot cut: dense leaf
      std::sort(nodes.begin(), nodes.end(), lexless);
      supNodes.push_back(nodes);
      supParent.push_back(-1);
      return (int)supNodes.size() - 1;
    }
    std::vector<int32_t> L, S, R;
    for (int v : nodes) {
      const int x = lat[3 * (int64_t)v + ax];
      (x < c ? L : (x == c ? S : R)).push_back(v);
    }
    std::vector<int32_t>().swap(nodes);
    std::vector<int> kids;
    if (!L.empty()) kids.push_back(nd(L));
    if (!R.empty()) kids.push_back(nd(R));
    std::sort(S.begin(), S.end(), lexless);
    supNodes.push_back(S);
    supParent.push_back(-1);
    const int s = (int)supNodes.size() - 1;
    for (int k : kids) supParent[k] = s;
    return s;
  };
  const int ndroot = freeNodes.empty() ? -1 : nd(freeNodes);
  if (n_contact > 0) {
    std::vector<int32_t> cs(contact_nodes, contact_nodes + n_contact);
    std::sort(cs.begin(), cs.end(), lexless);
    supNodes.push_back(cs);
    supParent.push_back(-1);
    P.csup = (int)supNodes.size() - 1;
    if (ndroot >= 0) supParent[ndroot] = P.csup;
  }
  P.nsup = (int)supNodes.size();
  P.sfirst.resize(P.nsup);
  P.ssize.resize(P.nsup);
  P.parent = supParent;
  P.pos_of_node.assign(n, -1);
  P.node_of_pos.resize(P.nfree);
  {
    int pos = 0;
    for (int s = 0; s < P.nsup; ++s) {
      P.sfirst[s] = pos;
      P.ssize[s] = (int)supNodes[s].size();
      for (int v : supNodes[s]) {
        P.pos_of_node[v] = pos;
        P.node_of_pos[pos] = v;
        ++pos;
      }
    }
  }
  if (P.nc > 0) {
    P.cand_loc.resize(P.nc);
    P.cand_of_loc.resize(P.nc);
    for (int j = 0; j < P.nc; ++j) {
      P.cand_loc[j] = P.pos_of_node[P.cand_node[j]] - P.sfirst[P.csup];
      P.cand_of_loc[P.cand_loc[j]] = j;
    }
  }
  std::vector<int32_t> sup_of_pos(P.nfree);
  for (int s = 0; s < P.nsup; ++s)
    for (int k = 0; k < P.ssize[s]; ++k) sup_of_pos[P.sfirst[s] + k] = s;
  for (int s = 0; s < P.nsup; ++s)
    if (P.parent[s] >= 0 && P.parent[s] <= s) return "internal: ND tree not in postorder";

  // ---------------- scalar A_s in solver order (CSR)
  {
    std::vector<std::vector<std::pair<int32_t, double>>> rowsA(P.nfree);
    for (int e = 0; e < m; ++e) {
      const int32_t* c = hex8 + 8 * (int64_t)e;
      for (int a = 0; a < 8; ++a) {
        const int pa = P.pos_of_node[c[a]];
        if (pa < 0) continue;
        for (int b = 0; b < 8; ++b) {
          const int pb = P.pos_of_node[c[b]];
          if (pb < 0) continue;
          double km = P.Km[a][b];
          if (!P.fib.empty()) {  // this element's own fiber m_e: m_e^T Tm[a][b] m_e
            const double* me = P.fib.data() + 3 * (int64_t)e;
            km = 0;
            for (int j = 0; j < 3; ++j)
              for (int k = 0; k < 3; ++k) km += me[j] * P.Tm[a][b][j][k] * me[k];
          }
          rowsA[pa].push_back({pb, w_ref * P.Kc[a][b] + w_m * km});
        }
      }
    }
    P.a_ptr.assign(P.nfree + 1, 0);
    P.a_col.clear();
    P.a_val.clear();
    for (int p = 0; p < P.nfree; ++p) {
      auto& r = rowsA[p];
      r.push_back({p, P.node_mass[P.node_of_pos[p]] / (h * h)});
      std::stable_sort(r.begin(), r.end(), [](auto& x, auto& y) { return x.first < y.first; });
      for (size_t k = 0; k < r.size();) {
        size_t k2 = k;
        double s = 0;
        while (k2 < r.size() && r[k2].first == r[k].first) s += r[k2++].second;
        P.a_col.push_back(r[k].first);
        P.a_val.push_back(s);
        k = k2;
      }
      P.a_ptr[p + 1] = (int64_t)P.a_col.size();
      std::vector<std::pair<int32_t, double>>().swap(r);
    }
  }

  // ---------------- symbolic: rows(s) = (adj(J_s) U rows(children)) beyond J_s
  std::vector<std::vector<int32_t>> kids(P.nsup);
  for (int s = 0; s < P.nsup; ++s)
    if (P.parent[s] >= 0) kids[P.parent[s]].push_back(s);
  std::vector<std::vector<int32_t>> srows(P.nsup);
  P.height.assign(P.nsup, 0);
  for (int s = 0; s < P.nsup; ++s) {
    const int last = P.sfirst[s] + P.ssize[s] - 1;
    std::vector<int32_t> r;
    for (int p = P.sfirst[s]; p <= last; ++p)
      for (int64_t k = P.a_ptr[p]; k < P.a_ptr[p + 1]; ++k)
        if (P.a_col[k] > last) r.push_back(P.a_col[k]);
    for (int c : kids[s]) {
      for (int q : srows[c])
        if (q > last) r.push_back(q);
      P.height[s] = std::max(P.height[s], P.height[c] + 1);
    }
    std::sort(r.begin(), r.end());
    r.erase(std::unique(r.begin(), r.end()), r.end());
    srows[s].swap(r);
  }
  for (int s = 0; s < P.nsup; ++s)
    if (P.parent[s] < 0 && !srows[s].empty()) return "internal: ND root with off-diagonal rows";
  P.rptr.assign(P.nsup + 1, 0);
  for (int s = 0; s < P.nsup; ++s) P.rptr[s + 1] = P.rptr[s] + (int64_t)srows[s].size();
  P.rows.resize(P.rptr[P.nsup]);
  for (int s = 0; s < P.nsup; ++s) std::copy(srows[s].begin(), srows[s].end(), P.rows.begin() + P.rptr[s]);
  P.doff.assign(P.nsup + 1, 0);
  P.poff.assign(P.nsup + 1, 0);
  for (int s = 0; s < P.nsup; ++s) {
    const int64_t ns = P.ssize[s], nr = (int64_t)srows[s].size();
    P.doff[s + 1] = P.doff[s] + ns * (ns + 1) / 2;
    P.poff[s + 1] = P.poff[s] + nr * ns;
    P.factor_flops += ns * ns * ns / 3.0 + nr * ns * ns + (double)nr * nr * ns;
  }
  P.nnzL = P.doff[P.nsup] + P.poff[P.nsup];
  P.D.assign(P.doff[P.nsup], 0.0);
  P.P.assign(P.poff[P.nsup], 0.0);

  // ---------------- numeric multifrontal factorisation, level-synchronous
  auto t0 = std::chrono::steady_clock::now();
  int H = 0;
  for (int s = 0; s < P.nsup; ++s) H = std::max(H, P.height[s]);
  std::vector<std::vector<int32_t>> byh(H + 1);
  for (int s = 0; s < P.nsup; ++s) byh[P.height[s]].push_back(s);
  std::vector<std::vector<double>> U(P.nsup);  // update matrices (nr x nr row-major lower)
  const int nthreads = omp_get_max_threads();
  bool ok = true;
  for (int lev = 0; lev <= H && ok; ++lev) {
    const auto& list = byh[lev];
    const bool outer = (int)list.size() >= 2 * nthreads;
    auto work = [&](int s, bool inner_par, std::vector<int32_t>& loc) {
      const int ns = P.ssize[s];
      const int nr = (int)(P.rptr[s + 1] - P.rptr[s]);
      const int f = ns + nr;
      const int32_t* R = P.rows.data() + P.rptr[s];
      std::vector<double> F((int64_t)f * f, 0.0);
      for (int k = 0; k < ns; ++k) loc[P.sfirst[s] + k] = k;
      for (int k = 0; k < nr; ++k) loc[R[k]] = ns + k;
      for (int k = 0; k < ns; ++k) {
        const int p = P.sfirst[s] + k;
        for (int64_t t = P.a_ptr[p]; t < P.a_ptr[p + 1]; ++t) {
          const int q = P.a_col[t];
          if (q < p) continue;
          F[(int64_t)loc[q] * f + k] += P.a_val[t];
        }
      }
      for (int c : kids[s]) {
        const int nrc = (int)(P.rptr[c + 1] - P.rptr[c]);
        const int32_t* Rc = P.rows.data() + P.rptr[c];
        const double* Uc = U[c].data();
        for (int i = 0; i < nrc; ++i) {
          const int li = loc[Rc[i]];
          for (int j = 0; j <= i; ++j) F[(int64_t)li * f + loc[Rc[j]]] += Uc[(int64_t)i * nrc + j];
        }
        std::vector<double>().swap(U[c]);
      }
      if (s == P.csup) {  // the assembled root front IS the Schur complement S_CC
        P.Scc.assign((int64_t)ns * ns, 0.0);
        for (int i = 0; i < ns; ++i)
          for (int j = 0; j <= i; ++j)
            P.Scc[(int64_t)i * ns + j] = P.Scc[(int64_t)j * ns + i] = F[(int64_t)i * f + j];
      }
      if (!partial_cholesky(F.data(), f, ns, inner_par)) return false;
      schur_update(F.data(), f, ns, inner_par);
      tri_inverse(F.data(), f, ns, P.D.data() + P.doff[s], inner_par);
      // W_s = L21 L11^{-1} (row-major nr x ns): the per-level solve operator
      double* Ws = P.P.data() + P.poff[s];
      const double* Ds = P.D.data() + P.doff[s];
#pragma omp parallel for schedule(static) if (inner_par && nr > 64)
      for (int i = 0; i < nr; ++i) {
        const double* Li = F.data() + (int64_t)(ns + i) * f;
        double* Wi = Ws + (int64_t)i * ns;
        for (int c = 0; c < ns; ++c) {
          double acc = 0;
          for (int j = c; j < ns; ++j) acc += Li[j] * Ds[(int64_t)j * (j + 1) / 2 + c];
          Wi[c] = acc;
        }
      }
      if (P.parent[s] >= 0 && nr > 0) {
        U[s].assign((int64_t)nr * nr, 0.0);
        for (int i = 0; i < nr; ++i)
          std::memcpy(U[s].data() + (int64_t)i * nr, F.data() + (int64_t)(ns + i) * f + ns, sizeof(double) * (i + 1));
      }
      return true;
    };
    if (outer) {
      int bad = 0;
#pragma omp parallel
      {
        std::vector<int32_t> loc(P.nfree, -1);
#pragma omp for schedule(dynamic, 1) reduction(+ : bad)
        for (int k = 0; k < (int)list.size(); ++k)
          if (!work(list[k], false, loc)) bad++;
      }
      ok = bad == 0;
    } else {
      std::vector<int32_t> loc(P.nfree, -1);
      for (int s : list)
        if (!work(s, true, loc)) { ok = false; break; }
    }
  }
  P.factor_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (!ok) {
    *numerical = true;
    return "A is not symmetric positive definite (non-positive pivot in the Cholesky factorisation)";
  }

  // ---------------- solve schedule (K3 v3)
  P.nlevels = H + 1;
  if (const char* e = std::getenv("PD_K3_MERGE_ROOT")) P.merge_root = std::atoi(e) != 0;
  if (P.k3_version == 4) build_warp_schedule(P, byh);
  else build_solve_schedule(P, byh);
  return "";
}

}  // namespace pdb
