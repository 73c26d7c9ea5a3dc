#include "setup_linalg.h"

#include <algorithm>
#include <cmath>
#include <numeric>

namespace rs {
namespace la {

FFT::FFT(int n) : N(n) {
  logN = 0;
  while ((1 << logN) < N) ++logN;
  w.resize(N / 2 > 0 ? N / 2 : 1);
  for (int k = 0; k < N / 2; ++k) {
    double ang = -2.0 * M_PI * double(k) / double(N);
    w[k] = cplx(std::cos(ang), std::sin(ang));
  }
  rev.resize(N);
  for (int i = 0; i < N; ++i) {
    int r = 0;
    for (int b = 0; b < logN; ++b)
      if (i & (1 << b)) r |= 1 << (logN - 1 - b);
    rev[i] = r;
  }
}

static void fft_core(const FFT& f, cplx* x, bool inv) {
  const int N = f.N;
  for (int i = 0; i < N; ++i)
    if (i < f.rev[i]) std::swap(x[i], x[f.rev[i]]);
  for (int len = 2; len <= N; len <<= 1) {
    const int half = len >> 1, step = N / len;
    for (int i = 0; i < N; i += len) {
      for (int j = 0; j < half; ++j) {
        cplx wj = f.w[j * step];
        if (inv) wj = std::conj(wj);
        cplx u = x[i + j], v = x[i + j + half] * wj;
        x[i + j] = u + v;
        x[i + j + half] = u - v;
      }
    }
  }
}

void FFT::forward(cplx* x) const { fft_core(*this, x, false); }
void FFT::inverse(cplx* x) const { fft_core(*this, x, true); }

void householder_qr(double* A, int m, int n, std::vector<double>& tau) {
  tau.assign(n, 0.0);
  for (int j = 0; j < n; ++j) {
    double* a = A + (size_t)j * m;
    double norm = 0.0;
    for (int i = j; i < m; ++i) norm += a[i] * a[i];
    norm = std::sqrt(norm);
    if (norm == 0.0) { tau[j] = 0.0; continue; }
    double alpha = a[j] > 0 ? -norm : norm;
    double v0 = a[j] - alpha;
    // v = [1, a[j+1..]/v0]
    for (int i = j + 1; i < m; ++i) a[i] /= v0;
    tau[j] = -v0 / alpha;   // = (alpha - a_j)/alpha ... standard LAPACK form
    a[j] = alpha;
    // apply H = I - tau v v^T to the remaining columns
    for (int c = j + 1; c < n; ++c) {
      double* b = A + (size_t)c * m;
      double dot = b[j];
      for (int i = j + 1; i < m; ++i) dot += a[i] * b[i];
      dot *= tau[j];
      b[j] -= dot;
      for (int i = j + 1; i < m; ++i) b[i] -= dot * a[i];
    }
  }
}

void form_q(const double* A, int m, int n, const std::vector<double>& tau, double* Q) {
  std::fill(Q, Q + (size_t)m * n, 0.0);
  for (int j = 0; j < n; ++j) Q[(size_t)j * m + j] = 1.0;
  for (int j = n - 1; j >= 0; --j) {
    const double* v = A + (size_t)j * m;
    if (tau[j] == 0.0) continue;
    for (int c = j; c < n; ++c) {
      double* q = Q + (size_t)c * m;
      double dot = q[j];
      for (int i = j + 1; i < m; ++i) dot += v[i] * q[i];
      dot *= tau[j];
      q[j] -= dot;
      for (int i = j + 1; i < m; ++i) q[i] -= dot * v[i];
    }
  }
}

void jacobi_svd(double* A, int m, int n, double* s, double* V, double* U) {
  std::fill(V, V + (size_t)n * n, 0.0);
  for (int j = 0; j < n; ++j) V[(size_t)j * n + j] = 1.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n - 1; ++p) {
      for (int q = p + 1; q < n; ++q) {
        double* ap = A + (size_t)p * m;
        double* aq = A + (size_t)q * m;
        double alpha = 0, beta = 0, gamma = 0;
        for (int i = 0; i < m; ++i) {
          alpha += ap[i] * ap[i];
          beta += aq[i] * aq[i];
          gamma += ap[i] * aq[i];
        }
        if (gamma == 0.0) continue;
        double c2 = std::fabs(gamma) / std::sqrt(alpha * beta);
        if (!(c2 > 1e-15)) continue;
        off = std::max(off, c2);
        double zeta = (beta - alpha) / (2.0 * gamma);
        double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
        for (int i = 0; i < m; ++i) {
          double x = ap[i], y = aq[i];
          ap[i] = c * x - sn * y;
          aq[i] = sn * x + c * y;
        }
        double* vp = V + (size_t)p * n;
        double* vq = V + (size_t)q * n;
        for (int i = 0; i < n; ++i) {
          double x = vp[i], y = vq[i];
          vp[i] = c * x - sn * y;
          vq[i] = sn * x + c * y;
        }
      }
    }
    if (off < 1e-15) break;
  }
  std::vector<double> nrm(n);
  for (int j = 0; j < n; ++j) {
    double acc = 0;
    const double* a = A + (size_t)j * m;
    for (int i = 0; i < m; ++i) acc += a[i] * a[i];
    nrm[j] = std::sqrt(acc);
  }
  std::vector<int> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return nrm[x] > nrm[y]; });
  std::vector<double> Vc(V, V + (size_t)n * n), Ac(A, A + (size_t)m * n);
  for (int j = 0; j < n; ++j) {
    int o = ord[j];
    s[j] = nrm[o];
    std::copy(Vc.begin() + (size_t)o * n, Vc.begin() + (size_t)(o + 1) * n, V + (size_t)j * n);
    std::copy(Ac.begin() + (size_t)o * m, Ac.begin() + (size_t)(o + 1) * m, A + (size_t)j * m);
    if (U) {
      for (int i = 0; i < m; ++i)
        U[(size_t)j * m + i] = s[j] > 0 ? A[(size_t)j * m + i] / s[j] : 0.0;
    }
  }
}

void sym_eig(double* A, int n, double* w, double* V) {
  std::fill(V, V + (size_t)n * n, 0.0);
  for (int j = 0; j < n; ++j) V[(size_t)j * n + j] = 1.0;
  auto at = [&](int i, int j) -> double& { return A[(size_t)j * n + i]; };
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0, diag = 0;
    for (int i = 0; i < n; ++i) {
      diag += at(i, i) * at(i, i);
      for (int j = i + 1; j < n; ++j) off += at(i, j) * at(i, j);
    }
    if (off <= 1e-30 * diag || off == 0.0) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double apq = at(p, q);
        if (apq == 0.0) continue;
        double theta = (at(q, q) - at(p, p)) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          double akp = at(k, p), akq = at(k, q);
          at(k, p) = c * akp - s * akq;
          at(k, q) = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          double apk = at(p, k), aqk = at(q, k);
          at(p, k) = c * apk - s * aqk;
          at(q, k) = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          double vkp = V[(size_t)p * n + k], vkq = V[(size_t)q * n + k];
          V[(size_t)p * n + k] = c * vkp - s * vkq;
          V[(size_t)q * n + k] = s * vkp + c * vkq;
        }
      }
  }
  std::vector<int> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::vector<double> d(n);
  for (int i = 0; i < n; ++i) d[i] = at(i, i);
  std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return d[x] < d[y]; });
  std::vector<double> Vc(V, V + (size_t)n * n);
  for (int j = 0; j < n; ++j) {
    w[j] = d[ord[j]];
    std::copy(Vc.begin() + (size_t)ord[j] * n, Vc.begin() + (size_t)(ord[j] + 1) * n,
              V + (size_t)j * n);
  }
}

static inline uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

double normal(uint64_t seed, uint64_t i) {
  uint64_t a = splitmix(seed * 0x100000001B3ull + 2 * i);
  uint64_t b = splitmix(seed * 0x100000001B3ull + 2 * i + 1);
  double u1 = (double((a >> 11) + 1)) * (1.0 / 9007199254740993.0);
  double u2 = double(b >> 11) * (1.0 / 9007199254740992.0);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

}  // namespace la
}  // namespace rs
