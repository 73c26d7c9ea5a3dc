// S1-S3 of Algorithm TEP: sinc quadrature of the Newton kernel,
// long/short split, and 1D Galerkin cell averages of the Gaussians.
#include <cmath>
#include <limits>
#include <vector>

#include "rs_internal.h"

namespace rs {

// 1/r = (2/sqrt(pi)) int_0^inf exp(-r^2 t^2) dt.  With t = sinh(u)/Ls and the
// trapezoid (sinc) rule of step s on the whole u axis, terms k and -k fold together:
//   t_0 = 0, a_0 = s/(sqrt(pi) Ls);  t_k = sinh(ks)/Ls, a_k = 2 s cosh(ks)/(sqrt(pi) Ls).
// (Eq. (2); the paper leaves the node family open, "proper choice of the
// quadrature points" PAPER.md:313 -- DESIGN.md reading A6.)
static void make_rule(double s, int K, double Ls, std::vector<double>& t, std::vector<double>& a) {
  t.assign(K + 1, 0.0);
  a.assign(K + 1, 0.0);
  const double c = s / (std::sqrt(M_PI) * Ls);
  a[0] = c;
  for (int k = 1; k <= K; ++k) {
    t[k] = std::sinh(k * s) / Ls;
    a[k] = 2.0 * c * std::cosh(k * s);
  }
}

static double rule_error(const std::vector<double>& t, const std::vector<double>& a,
                         const std::vector<double>& r) {
  double worst = 0.0;
  for (double ri : r) {
    double v = 0.0;
    for (size_t k = 0; k < t.size(); ++k) {
      double x = t[k] * ri;
      if (x > 40.0) break;               // t ascending: the rest underflow
      v += a[k] * std::exp(-x * x);
    }
    double e = std::fabs(v * ri - 1.0);
    if (!(e <= worst)) worst = e;        // NaN-safe max
  }
  return worst;
}

Quadrature choose_quadrature(double eps, double rmin, double rmax, double Ls) {
  std::vector<double> r(1500), rv(8000);
  for (size_t i = 0; i < r.size(); ++i)
    r[i] = rmin * std::pow(rmax / rmin, double(i) / double(r.size() - 1));
  for (size_t i = 0; i < rv.size(); ++i)
    rv[i] = rmin * std::pow(rmax / rmin, (double(i) + 0.37) / double(rv.size()));
  Quadrature best;
  best.K = -1;
  std::vector<double> t, a;
  for (int si = 5; si <= 120; ++si) {
    const double s = 0.01 * si;
    int Kmax = int(std::floor(40.0 / s));
    make_rule(s, Kmax, Ls, t, a);
    if (rule_error(t, a, r) > eps) continue;
    int lo = 1, hi = Kmax;
    while (lo < hi) {
      int mid = (lo + hi) / 2;
      make_rule(s, mid, Ls, t, a);
      if (rule_error(t, a, r) <= eps) hi = mid; else lo = mid + 1;
    }
    if (best.K < 0 || lo < best.K) {
      best.K = lo;
      best.s = s;
    }
  }
  if (best.K < 0) return best;
  best.Ls = Ls;
  make_rule(best.s, best.K, Ls, best.t, best.a);
  best.err = rule_error(best.t, best.a, rv);
  return best;
}

// Effective support radius sqrt(ln(1/eps))/t_k compared with sigma_s ("Use the van der Waals
// distance sigma > 0 to control from below the support of long-range Gaussians",
// PAPER.md:1193; reading A7).
bool is_long_term(double t, double sigma_s, double eps_split) {
  if (t == 0.0) return true;
  return std::sqrt(std::log(1.0 / eps_split)) / t >= sigma_s;
}

// g[d] = (1/h) int_{(d-1/2)h}^{(d+1/2)h} exp(-t^2 x^2) dx, evaluated at |d| (so g[-d] == g[d]
// bitwise) with the erf difference rewritten as an erfc difference away from the origin.
double cell_average(double t, double h, long d) {
  if (t == 0.0) return 1.0;
  const double ad = double(d < 0 ? -d : d);
  const double c = std::sqrt(M_PI) / (2.0 * t * h);
  if (ad < 0.5) return c * 2.0 * std::erf(t * (ad + 0.5) * h);
  return c * (std::erfc(t * (ad - 0.5) * h) - std::erfc(t * (ad + 0.5) * h));
}

}  // namespace rs
