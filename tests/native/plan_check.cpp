// Native check of the host plan (no GPU): solves A_s x = A_s v with the stored
// supernodal factor (D_s = L_ss^{-1}, panels P_s) by plain substitution and
// reports max |x - v| / max |v|.  Build: see tests/test_native_plan.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include "../../paper_2101_05917_b200/csrc/plan.h"
using namespace pdb;
int main(int argc, char** argv) {
  int nx = atoi(argv[1]), ny = atoi(argv[2]), nz = atoi(argv[3]);
  int fix = argc > 4 ? atoi(argv[4]) : 1;
  double dx = 0.01;
  std::vector<double> rest; std::vector<int32_t> hex;
  auto nid = [&](int i, int j, int k) { return i + (nx + 1) * (j + (ny + 1) * k); };
  for (int k = 0; k <= nz; ++k) for (int j = 0; j <= ny; ++j) for (int i = 0; i <= nx; ++i) {
    rest.push_back(i * dx); rest.push_back(j * dx); rest.push_back(k * dx); }
  for (int k = 0; k < nz; ++k) for (int j = 0; j < ny; ++j) for (int i = 0; i < nx; ++i)
    for (int c = 0; c < 8; ++c) hex.push_back(nid(i + (c & 1), j + ((c >> 1) & 1), k + ((c >> 2) & 1)));
  std::vector<int32_t> fixed;
  if (fix) for (int k = 0; k <= nz; ++k) for (int j = 0; j <= ny; ++j) for (int a = 0; a < 3; ++a) fixed.push_back(3 * nid(0, j, k) + a);
  int n = (int)rest.size() / 3, m = (int)hex.size() / 8;
  // optional 5th arg = 1: bottom-face nodes (z = 0) are contact candidates, ordered last
  int contact = argc > 5 ? atoi(argv[5]) : 0;
  std::vector<int32_t> cand;
  if (contact) for (int j = 0; j <= ny; ++j) for (int i = 0; i <= nx; ++i) if (!fix || i > 0) cand.push_back(nid(i, j, 0));
  HostPlan P; bool num; double fib[3] = {1, 0, 0};
  // PLAN_V=4: the K3 v4 warp-range schedule (PLAN_WARPS warps per level launch, default 148 x 8)
  if (const char* v = std::getenv("PLAN_V")) P.k3_version = std::atoi(v);
  if (const char* v = std::getenv("PLAN_WARPS")) P.k3_warps = std::atoi(v);
  std::string e = build_plan(P, n, m, rest.data(), hex.data(), dx, 1e3, 0.01, fixed.data(), (int)fixed.size(),
                             1e5 / 1.45, 1e5 / 1.45, fib, cand.data(), (int)cand.size(), &num);
  if (contact) {  // the candidate block is the last supernode and Scc = L_cc L_cc^T
    if (P.csup != P.nsup - 1 || P.ssize[P.csup] != (int)cand.size()) { printf("bad candidate supernode\n"); return 4; }
    const int c = P.nc; const double* D = P.D.data() + P.doff[P.csup];
    // Scc^{-1} = D^T D: check Scc (D^T D e_k) = e_k for a few k
    double worst = 0;
    for (int k = 0; k < c; k += std::max(1, c / 7)) {
      std::vector<double> t(c, 0.0), u(c, 0.0);
      for (int i = k; i < c; ++i) t[i] = D[(int64_t)i * (i + 1) / 2 + k];
      for (int j = 0; j < c; ++j) { double s = 0; for (int i = j; i < c; ++i) s += D[(int64_t)i * (i + 1) / 2 + j] * t[i]; u[j] = s; }
      for (int i = 0; i < c; ++i) { double s = 0; for (int j = 0; j < c; ++j) s += P.Scc[(int64_t)i * c + j] * u[j]; worst = std::max(worst, std::fabs(s - (i == k))); }
    }
    if (worst > 1e-9) { printf("Scc check failed %.3e\n", worst); return 5; }
  }
  if (!e.empty()) { printf("ERROR %s\n", e.c_str()); return 1; }
  int N = P.nfree;
  std::mt19937 rng(1); std::normal_distribution<double> nd;
  std::vector<double> v(N), b(N, 0.0);
  for (auto& x : v) x = nd(rng);
  for (int p = 0; p < N; ++p) for (int64_t k = P.a_ptr[p]; k < P.a_ptr[p + 1]; ++k) b[p] += P.a_val[k] * v[P.a_col[k]];
  // Emulate the device schedule exactly: per level, chains (items accumulated in order, then written to
  // their direct rows or partial rows), then the level's reduce (targets in order, sources in order).
  // Forward writes y (direct / assign) and subtracts into z; backward writes x.
  std::vector<double> z(b), y(N, 0.0), x(N, 0.0);
  auto run = [&](const HostPlan::Sweep& S, std::vector<double>& zsrc, std::vector<double>& direct,
                 std::vector<double>* zsub, bool fwd) {
    std::vector<double> part((size_t)(S.max_partial_rows + 32), 0.0);
    std::vector<int> assigned(N, 0);
    if ((int)S.lvl_chain.size() != P.nlevels + 1 || S.chain.back() != (int)S.a_off.size()) {
      printf("bad chain index\n");
      exit(12);
    }
    for (int lev = 0; lev < P.nlevels; ++lev) {
      std::vector<int> pused((size_t)(S.max_partial_rows / 32 + 1), 0);
      for (int c = S.lvl_chain[lev]; c < S.lvl_chain[lev + 1]; ++c) {
        const int t0 = S.chain[c], t1 = S.chain[c + 1];
        if (t0 < S.lvl_item[lev] || t1 > S.lvl_item[lev + 1] || t1 <= t0) { printf("chain outside its level\n"); exit(13); }
        std::vector<double> acc(32, 0.0);
        for (int t = t0; t < t1; ++t) {
          if (S.out[t] != S.out[t0] || S.nvalid[t] != S.nvalid[t0]) { printf("chain output mismatch\n"); exit(14); }
          for (int l = 0; l < S.nvalid[t]; ++l)
            for (int k = 0; k < S.nk[t]; ++k) {
              const bool contig = k < S.nkd[t];
              const int zr = contig ? S.zrow[t] + k : P.rows[S.zidx[t] + k - S.nkd[t]];
              acc[l] += S.A[S.a_off[t] + sweep_frag_pos(k, l)] * (fwd ? zsrc[zr] : (contig ? y[zr] : x[zr]));
            }
        }
        const int o = S.out[t0];
        for (int l = 0; l < S.nvalid[t0]; ++l) {
          if (o >= 0) {
            if (assigned[o + l]++) { printf("row %d written twice\n", o + l); exit(10); }
            direct[o + l] = acc[l];
          } else {
            if (l == 0 && pused[-o - 1]++) { printf("partial block %d reused in a level\n", -o - 1); exit(15); }
            part[(size_t)(-o - 1) * 32 + l] = acc[l];
          }
        }
      }
      for (int r = S.lvl_red[lev]; r < S.lvl_red[lev + 1]; ++r) {
        double acc = 0;
        for (int u = S.red_ptr[r]; u < S.red_ptr[r + 1]; ++u) acc += part[S.red_src[u]];
        if (S.red_mode[r] == 0) {
          if (assigned[S.red_row[r]]++) { printf("row %d written twice\n", S.red_row[r]); exit(10); }
          direct[S.red_row[r]] = acc;
        } else {
          (*zsub)[S.red_row[r]] -= acc;
        }
      }
    }
    for (int p = 0; p < N; ++p)
      if (assigned[p] != 1) { printf("row %d written %d times\n", p, assigned[p]); exit(11); }
  };
  if (std::getenv("PLAN_LEVELS"))  // per-level schedule statistics (developer aid)
    for (const HostPlan::Sweep* S : {&P.fw, &P.bw})
      for (int l = 0; l < P.nlevels; ++l) {
        int64_t bytes = 0;
        int lmax = 0;
        for (int c = S->lvl_chain[l]; c < S->lvl_chain[l + 1]; ++c) lmax = std::max(lmax, S->chain[c + 1] - S->chain[c]);
        for (int t = S->lvl_item[l]; t < S->lvl_item[l + 1]; ++t) bytes += (int64_t)((S->nk[t] + 3) & ~3) * 256;
        int single = 0, srcs = 0;
        for (int r = S->lvl_red[l]; r < S->lvl_red[l + 1]; ++r) {
          single += S->red_ptr[r + 1] - S->red_ptr[r] == 1;
          srcs += S->red_ptr[r + 1] - S->red_ptr[r];
        }
        printf("   single-source targets %d of %d, sources %d  ", single, S->lvl_red[l + 1] - S->lvl_red[l], srcs);
        printf("%s level %2d: items %6d chains %6d longest %2d targets %6d factor MB %7.2f\n", S == &P.fw ? "fw" : "bw", l,
               S->lvl_item[l + 1] - S->lvl_item[l], S->lvl_chain[l + 1] - S->lvl_chain[l], lmax,
               S->lvl_red[l + 1] - S->lvl_red[l], bytes / 1e6);
      }
  // v4: per level, every warp range walked piece by piece (k-groups in order, k-steps through krow), outputs to
  // direct rows or partial slots, then the level's reduce (targets in order, sources in order)
  auto run4 = [&](const HostPlan::Sweep4& S, std::vector<double>& zsrc, std::vector<double>& direct,
                  std::vector<double>* zsub, bool fwd) {
    std::vector<double> part((size_t)(S.max_partial_rows + 32), 0.0);
    std::vector<int> assigned(N, 0);
    if ((int)S.lvl_g.size() != P.nlevels + 1 || (int)S.lvl_warp.size() != P.nlevels + 1) { printf("bad v4 level index\n"); exit(20); }
    for (int lev = 0; lev < P.nlevels; ++lev) {
      const int w0 = S.lvl_warp[lev], W = S.lvl_warp[lev + 1] - w0 - 1;
      if (S.wg[w0] != S.lvl_g[lev] || S.wg[w0 + W] != S.lvl_g[lev + 1]) { printf("warp ranges do not cover level %d\n", lev); exit(21); }
      std::vector<int> pused((size_t)(S.max_partial_rows / 32 + 1), 0);
      for (int w = 0; w < W; ++w) {
        int p = S.wpiece[w0 + w];
        int g = S.wg[w0 + w];
        while (g < S.wg[w0 + w + 1]) {
          if (S.pstart[p] != g || S.pkg[p] < 1) { printf("piece %d does not start at %d\n", p, g); exit(22); }
          std::vector<double> acc(32, 0.0);
          for (int gg = g; gg < g + S.pkg[p]; ++gg)
            for (int j = 0; j < 4; ++j) {
              const int v = S.krow[4 * (int64_t)gg + j];
              if (v == -1) continue;
              const double src = fwd ? zsrc[v] : (v >= 0 ? y[v] : x[-2 - v]);
              for (int l = 0; l < 32; ++l) acc[l] += S.A[(int64_t)gg * 128 + sweep_frag_pos(j, l)] * src;
            }
          const int o = S.pout[p];
          for (int l = 0; l < S.pnv[p]; ++l) {
            if (o >= 0) {
              if (assigned[o + l]++) { printf("row %d written twice\n", o + l); exit(10); }
              direct[o + l] = acc[l];
            } else {
              if (l == 0 && pused[-o - 1]++) { printf("partial slot %d reused in a level\n", -o - 1); exit(15); }
              part[(size_t)(-o - 1) * 32 + l] = acc[l];
            }
          }
          g += S.pkg[p];
          ++p;
        }
        if (p != S.wpiece[w0 + w + 1]) { printf("warp %d piece count mismatch\n", w); exit(23); }
      }
      if (std::getenv("PLAN_STATS")) {  // per-level statistics of the v4 schedule
        int np = S.lvl_piece[lev + 1] - S.lvl_piece[lev], nd = 0;
        for (int q = S.lvl_piece[lev]; q < S.lvl_piece[lev + 1]; ++q) nd += S.pout[q] >= 0;
        long long srcs = S.red_ptr[S.lvl_red[lev + 1]] - S.red_ptr[S.lvl_red[lev]];
        int single = 0;
        for (int r = S.lvl_red[lev]; r < S.lvl_red[lev + 1]; ++r) single += S.red_ptr[r + 1] - S.red_ptr[r] == 1;
        printf("  single-source %6d ", single);
        printf("%s level %2d: kgroups %7d (%6.2f MB) warps %5d pieces %6d direct %6d reduce targets %7d sources %8lld\n",
               fwd ? "fw" : "bw", lev, S.lvl_g[lev + 1] - S.lvl_g[lev], (S.lvl_g[lev + 1] - S.lvl_g[lev]) * 1024.0 / 1e6, W,
               np, nd, S.lvl_red[lev + 1] - S.lvl_red[lev], srcs);
      }
      for (int r = S.lvl_red[lev]; r < S.lvl_red[lev + 1]; ++r) {
        double acc = 0;
        for (int u = S.red_ptr[r]; u < S.red_ptr[r + 1]; ++u) acc += part[S.red_src[u]];
        if (S.red_mode[r] == 0) {
          if (assigned[S.red_row[r]]++) { printf("row %d written twice\n", S.red_row[r]); exit(10); }
          direct[S.red_row[r]] = acc;
        } else {
          (*zsub)[S.red_row[r]] -= acc;
        }
      }
    }
    // (with the merged root the forward sweep leaves the root rows of y unwritten: the backward sweep's first
    // level computes x_root = S^{-1} z_root directly)
    const int rf = P.merge_root ? P.sfirst[P.nsup - 1] : N;
    for (int p = 0; p < N; ++p)
      if (assigned[p] != 1 && !(fwd && p >= rf && assigned[p] == 0)) {
        printf("row %d written %d times\n", p, assigned[p]);
        exit(11);
      }
  };
  if (P.k3_version == 4) {
    run4(P.fw4, z, y, &z, true);
    x = z;  // the device's z and x share one buffer: the merged root level reads z_root from it
    run4(P.bw4, y, x, nullptr, false);
    double err = 0, mx = 0;
    for (int p = 0; p < N; ++p) { err = std::max(err, std::fabs(x[p] - v[p])); mx = std::max(mx, std::fabs(v[p])); }
    int64_t pieces = (int64_t)P.fw4.pstart.size() + (int64_t)P.bw4.pstart.size();
    printf("v4 n=%d nfree=%d nsup=%d levels=%d kgroups fw=%d bw=%d pieces=%lld partial rows fw=%lld bw=%lld nnzL=%lld relerr=%.3e\n",
           n, N, P.nsup, P.nlevels, P.fw4.lvl_g.back(), P.bw4.lvl_g.back(), (long long)pieces,
           (long long)P.fw4.max_partial_rows, (long long)P.bw4.max_partial_rows, (long long)P.nnzL, err / mx);
    return err / mx < 1e-10 ? 0 : 2;
  }
  run(P.fw, z, y, &z, true);
  run(P.bw, y, x, nullptr, false);
  double err = 0, mx = 0;
  for (int p = 0; p < N; ++p) { err = std::max(err, std::fabs(x[p] - v[p])); mx = std::max(mx, std::fabs(v[p])); }
  int64_t nnzA = P.a_ptr[N];
  printf("n=%d nfree=%d nsup=%d levels=%d fitems=%zu bitems=%zu fchains=%zu bchains=%zu fstream=%zu bstream=%zu nnzA=%lld nnzL=%lld flops=%.3g factor_ms=%.1f relerr=%.3e\n",
         n, N, P.nsup, P.nlevels, P.fw.a_off.size(), P.bw.a_off.size(), P.fw.chain.size() - 1, P.bw.chain.size() - 1,
         P.fw.A.size(), P.bw.A.size(), (long long)nnzA,
         (long long)P.nnzL, P.factor_flops, P.factor_ms, err / mx);
  return err / mx < 1e-10 ? 0 : 2;
}
