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
  // forward: per level, D tasks y[J_s] = D_s z[J_s]; W tasks z[anc] -= W_s z_old[J_s]
  std::vector<double> z(b), y(N, 0.0), x(N, 0.0);
  for (int lev = 0; lev < P.nlevels; ++lev) {
    std::vector<double> zold = z;
    for (int t = P.flvl_ptr[lev]; t < P.flvl_ptr[lev + 1]; ++t) {
      int s = P.ft_sup[t], r0 = P.ft_r0[t], r1 = P.ft_r1[t], f = P.sfirst[s];
      if (P.ft_type[t] == 0) {
        for (int i = r0; i < r1; ++i) { double sum = 0; for (int j = 0; j <= i; ++j) sum += P.D[P.doff[s] + (int64_t)i * (i + 1) / 2 + j] * zold[f + j]; y[f + i] = sum; }
      } else {
        for (int bk = P.ft_bptr[t]; bk < P.ft_bptr[t + 1]; ++bk) {
          int d = P.fb_s[bk], nd_ = P.ssize[d];
          for (int k = P.fb_k0[bk]; k < P.fb_k1[bk]; ++k) {
            int r = P.rows[P.rptr[d] + k];
            if (r < f + r0 || r >= f + r1) { printf("bad block row\n"); return 3; }
            double sum = 0;
            for (int j = 0; j < nd_; ++j) sum += P.P[P.poff[d] + (int64_t)k * nd_ + j] * zold[P.sfirst[d] + j];
            z[r] -= sum;
          }
        }
      }
    }
  }
  for (int lev = P.nlevels - 1; lev >= 0; --lev) {
    for (int t = P.blvl_ptr[lev]; t < P.blvl_ptr[lev + 1]; ++t) {
      int s = P.bt_sup[t], c0 = P.bt_c0[t], c1 = P.bt_c1[t], f = P.sfirst[s], ns = P.ssize[s];
      int nr = (int)(P.rptr[s + 1] - P.rptr[s]);
      for (int c = c0; c < c1; ++c) {
        double sum = 0;
        for (int i = c; i < ns; ++i) sum += P.D[P.doff[s] + (int64_t)i * (i + 1) / 2 + c] * y[f + i];
        for (int k = 0; k < nr; ++k) sum -= P.P[P.poff[s] + (int64_t)k * ns + c] * x[P.rows[P.rptr[s] + k]];
        x[f + c] = sum;
      }
    }
  }
  double err = 0, mx = 0;
  for (int p = 0; p < N; ++p) { err = std::max(err, std::fabs(x[p] - v[p])); mx = std::max(mx, std::fabs(v[p])); }
  int64_t nnzA = P.a_ptr[N];
  printf("n=%d nfree=%d nsup=%d levels=%d ftasks=%zu fblocks=%zu btasks=%zu nnzA=%lld nnzL=%lld flops=%.3g factor_ms=%.1f relerr=%.3e\n",
         n, N, P.nsup, P.nlevels, P.ft_type.size(), P.fb_s.size(), P.bt_sup.size(), (long long)nnzA, (long long)P.nnzL, P.factor_flops,
         P.factor_ms, err / mx);
  return err / mx < 1e-10 ? 0 : 2;
}
