// matvec_demo.cpp -- C++ host usage of the B200 matvec through fdhelm_b200.hpp:
// builds an operator on seeded uniform points, applies it, and compares 64
// rows against a direct O(N) sum per row (exp(i k r) / (4 pi r)).
//   ./matvec_demo [N] [kappa] [m]
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "fdhelm_b200.hpp"

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? std::atoll(argv[1]) : 20000;
  const double kappa = argc > 2 ? std::atof(argv[2]) : 8.0;
  const int m = argc > 3 ? std::atoi(argv[3]) : 4;
  std::mt19937_64 rng(12345);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  std::vector<double> tx(n), ty(n), tz(n), sx(n), sy(n), sz(n);
  for (int64_t i = 0; i < n; ++i) {
    tx[i] = 1.0 - U(rng); ty[i] = 1.0 - U(rng); tz[i] = 1.0 - U(rng);
    sx[i] = 1.0 - U(rng); sy[i] = 1.0 - U(rng); sz[i] = 1.0 - U(rng);
  }
  std::vector<fdhelm_b200::Complex> x(n);
  for (auto& v : x) v = {2 * U(rng) - 1, 2 * U(rng) - 1};
  const double lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};
  fdhelm_b200::Params p;
  p.kappa = kappa;
  p.m = m;
  try {
    fdhelm_b200::DirectionalOperator op(tx, ty, tz, sx, sy, sz, lo, hi, p);
    // the same operator from AoS points and a box type shaped like the
    // reference's fdhelm::Point3 / fdhelm::AxisBox (geometry.hpp:13-59)
    struct P3 { double x, y, z; };
    struct Box { P3 lower, upper; };
    std::vector<P3> tp(n), sp(n);
    for (int64_t i = 0; i < n; ++i) { tp[i] = {tx[i], ty[i], tz[i]}; sp[i] = {sx[i], sy[i], sz[i]}; }
    fdhelm_b200::DirectionalOperator op_aos(std::span<const P3>(tp), std::span<const P3>(sp),
                                            Box{{0, 0, 0}, {1, 1, 1}}, p);
    if (op_aos.lplus() != op.lplus() || op_aos.tree(0) != op.tree(0)) {
      std::fprintf(stderr, "AoS and SoA operators differ\n");
      return 3;
    }
    const auto y = op.apply(x);
    double num = 0, den = 0;
    for (int64_t r = 0; r < 64; ++r) {
      const int64_t j = (r * 7919) % n;
      std::complex<double> acc = 0;
      for (int64_t k = 0; k < n; ++k) {
        const double d[3] = {tx[j] - sx[k], ty[j] - sy[k], tz[j] - sz[k]};
        const double rr = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        acc += std::polar(1.0 / (4.0 * M_PI * rr), kappa * rr) * x[k];
      }
      num += std::norm(y[j] - acc);
      den += std::norm(acc);
    }
    // two right-hand sides [x, 2x] in one batch (fdh_create_multi / fdh_apply_multi)
    fdhelm_b200::Params p2 = p;
    p2.nrhs = 2;
    fdhelm_b200::DirectionalOperator op2(tx, ty, tz, sx, sy, sz, lo, hi, p2);
    std::vector<std::complex<double>> X(2 * n), Y(2 * n);
    for (int64_t k = 0; k < n; ++k) X[k] = x[k], X[n + k] = 2.0 * x[k];
    op2.apply_multi(X, Y, 2);
    double dm = 0, dn = 0;
    for (int64_t j = 0; j < n; ++j) {
      dm += std::norm(Y[j] - y[j]) + std::norm(Y[n + j] - 2.0 * y[j]);
      dn += 5.0 * std::norm(y[j]);
    }
    if (std::sqrt(dm / dn) > 1e-12) {  // int8 M2L: the batch shares one moment scale per level
      std::fprintf(stderr, "multi-rhs apply differs from single applies: %.3e\n", std::sqrt(dm / dn));
      return 4;
    }
    const fdh_stats s = op.stats();
    std::printf("N=%lld kappa=%g m=%d: N_C=%lld N_SC=%lld nf=%.3f%% apply=%.3f ms, rel. error vs direct (64 rows) = %.3e\n",
                (long long)n, kappa, m, (long long)s.n_c, (long long)s.n_sc, s.nf_percent, s.apply_ms,
                std::sqrt(num / den));
    return std::sqrt(num / den) < 1e-3 ? 0 : 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
}
