// Dump the host-side setup (univariate matrices + generalized eigenpairs) of libls
// as JSON, so that tests/test_host_setup.py can check the C++ host logic against
// the oracle without a GPU.  Usage: host_setup_dump <n_el> <p>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "setup_host.hpp"

static void arr(const char* name, const std::vector<double>& v, bool comma = true) {
  std::printf("\"%s\": [", name);
  for (size_t i = 0; i < v.size(); ++i) std::printf("%s%.17g", i ? "," : "", v[i]);
  std::printf("]%s\n", comma ? "," : "");
}

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  const int n_el = std::atoi(argv[1]), p = std::atoi(argv[2]);
  ls::Factors s = ls::space_factors(n_el, p), t = ls::time_factors(n_el, p);
  std::vector<double> ls_, Us, lt, Ut;
  int rc1 = ls::generalized_eig(s.J, s.M, s.n, ls_, Us);
  int rc2 = ls::generalized_eig(t.K, t.M, t.n, lt, Ut);
  std::printf("{\"n_s\": %d, \"n_t\": %d, \"rc\": %d,\n", s.n, t.n, rc1 + rc2);
  arr("M", s.M); arr("K", s.K); arr("J", s.J); arr("Mt", t.M); arr("Kt", t.K);
  arr("lam_s", ls_); arr("U_s", Us); arr("lam_t", lt); arr("U_t", Ut);
  std::vector<double> gx; std::vector<long double> x, w;
  ls::gauss_legendre(p + 1, x, w);
  for (auto v : w) gx.push_back(double(v));
  arr("gauss_w", gx, false);
  std::printf("}\n");
  return 0;
}
