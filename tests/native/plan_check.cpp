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
  // Emulate the device schedule (K3 v3) exactly: per level, items (k-major 32-lane blocks) then the
  // level's reduce; forward writes y (D) / partial rows, backward writes x / partial rows.
  std::vector<double> z(b), y(N, 0.0), x(N, 0.0);
  auto run = [&](const HostPlan::Sweep& S, std::vector<double>& zsrc, std::vector<double>& direct,
                 std::vector<double>* zsub, bool fwd) {
    // dataflow invariants of the one-launch sweep: in item order every wait is already satisfied, and
    // every countdown ends at exactly 0
    std::vector<int> cd(S.cd_init.begin(), S.cd_init.end()), grem(S.g_cnt.begin(), S.g_cnt.end());
    std::vector<int> turn(S.ntiles, 0);
    std::vector<double> part(S.max_partial_rows + 32, 0.0);
    {  // a row is the target of at most one group (no concurrent read-modify-write of the same row)
      // mode 0 (y/x assign): exactly one group per row; mode 1 (z subtract): every group of a row belongs
      // to the same tile, whose groups are serialised by their turns
      std::vector<int> hits(N, 0), tile_of(N, -1);
      for (size_t g = 0; g < S.g_cnt.size(); ++g)
        for (int r = S.g_tptr[g]; r < S.g_tptr[g + 1]; ++r) {
          const int row = S.red_row[r];
          if (S.red_mode[r] == 0) {
            if (++hits[row] > 1) { printf("row %d assigned by two groups\n", row); exit(10); }
          } else {
            if (S.g_tile[g] < 0 || (tile_of[row] >= 0 && tile_of[row] != S.g_tile[g])) {
              printf("row %d updated by groups of different tiles\n", row);
              exit(10);
            }
            tile_of[row] = S.g_tile[g];
          }
        }
    }
    for (int lev = 0; lev < P.nlevels; ++lev) {
      for (int t = S.lvl_item[lev]; t < S.lvl_item[lev + 1]; ++t) {
        const int su = S.sup[t];
        if (fwd) {
          if (cd[su] != 0) { printf("fwd item %d of s=%d runs before its inputs are final\n", t, su); exit(7); }
        } else if (S.nkd[t] < S.nk[t]) {
          for (int q = S.wl_ptr[su]; q < S.wl_ptr[su + 1]; ++q)
            if (cd[S.wl[q]] != 0) { printf("bwd item %d waits on s=%d\n", t, S.wl[q]); exit(8); }
        }
        for (int l = 0; l < S.nvalid[t]; ++l) {
          double acc = 0;
          for (int k = 0; k < S.nk[t]; ++k) {
            const bool contig = k < S.nkd[t];
            const int zr = contig ? S.zrow[t] + k : P.rows[S.zidx[t] + k - S.nkd[t]];
            acc += S.A[S.a_off[t] + sweep_frag_pos(k, l)] * (fwd ? zsrc[zr] : (contig ? y[zr] : x[zr]));
          }
          if (S.out[t] >= 0) direct[S.out[t] + l] = acc;
          else part[(int64_t)(-S.out[t] - 1) * 32 + l] = acc;
        }
        if (S.sig[t] >= 0) cd[S.sig[t]]--;
        // device semantics: the item that brings a group to zero applies the group's sums, then signals
        for (int q = S.ig_ptr[t]; q < S.ig_ptr[t + 1]; ++q) {
          const int g = S.ig[q];
          if (--grem[g] != 0) continue;
          if (S.g_tile[g] >= 0 && turn[S.g_tile[g]]++ != S.g_turn[g]) { printf("group %d out of turn\n", g); exit(11); }
          for (int r = S.g_tptr[g]; r < S.g_tptr[g + 1]; ++r) {
            double acc = 0;
            for (int u = S.red_ptr[r]; u < S.red_ptr[r + 1]; ++u) acc += part[S.red_src[u]];
            if (S.red_mode[r] == 0) direct[S.red_row[r]] = acc;
            else (*zsub)[S.red_row[r]] -= acc;
          }
          if (S.g_sig[g] >= 0) cd[S.g_sig[g]]--;
        }
      }
    }
    for (size_t g = 0; g < grem.size(); ++g)
      if (grem[g] != 0) { printf("group %zu never completes (%d left)\n", g, grem[g]); exit(6); }
    for (size_t i = 0; i < cd.size(); ++i)
      if (cd[i] != 0) { printf("countdown of s=%zu ends at %d\n", i, cd[i]); exit(9); }
  };
  run(P.fw, z, y, &z, true);
  run(P.bw, y, x, nullptr, false);
  double err = 0, mx = 0;
  for (int p = 0; p < N; ++p) { err = std::max(err, std::fabs(x[p] - v[p])); mx = std::max(mx, std::fabs(v[p])); }
  int64_t nnzA = P.a_ptr[N];
  printf("n=%d nfree=%d nsup=%d levels=%d fitems=%zu bitems=%zu fstream=%zu bstream=%zu nnzA=%lld nnzL=%lld flops=%.3g factor_ms=%.1f relerr=%.3e\n",
         n, N, P.nsup, P.nlevels, P.fw.a_off.size(), P.bw.a_off.size(), P.fw.A.size(), P.bw.A.size(), (long long)nnzA,
         (long long)P.nnzL, P.factor_flops, P.factor_ms, err / mx);
  return err / mx < 1e-10 ? 0 : 2;
}
