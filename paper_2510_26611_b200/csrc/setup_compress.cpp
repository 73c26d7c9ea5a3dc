// S5-S7 of Algorithm TEP: the long-range part of the protein potential
//   P_l[i] = sum_m z_m sum_{k long} a_k g_k[i_0 - c_{m,0}] g_k[i_1 - c_{m,1}] g_k[i_2 - c_{m,2}]
// (shift-and-windowing sum, Eq. (5)-(6)) is a canonical tensor of rank
// M * R_l ("initial rank R' = N_M R_L").  It is never formed.  Its rank is
// reduced (TEP step 4, "canonical-Tucker-canonical transform") by
//   S5  RHOSVD: per mode, the dominant left singular subspace of the implicit, weighted side
//       matrix [g_k[. - c_{m,l}]]_{(m,k)} (n x M R_l), found by a randomized range finder whose
//       products with the side matrix are 1D convolutions (FFT) with binned charge trains;
//   S6  the exact Tucker core G = P_l x_0 U_0^T x_1 U_1^T x_2 U_2^T;
//   S7  core -> CP: the exact slice expansion (rank <= r_0 min(r_1, r_2)) when it fits in R,
//       else CP-ALS to width R initialised from the dominant slice triplets.
// Then F_l = U_l X_l (n x R), weights folded into F_0.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <vector>

#include "rs_internal.h"
#include "setup_linalg.h"

namespace rs {

using la::cplx;

namespace {

struct ConvOps {
  int n = 0, N = 0, RL = 0;
  la::FFT fft{2};
  std::vector<std::vector<double>> G;     // G[k][d], d = 0..n-1 (even kernel)
  std::vector<std::vector<cplx>> FG;      // FFT of the centred kernel, size N
  std::vector<std::vector<double>> nrm;   // windowed column norms N_k(j)
  std::vector<std::vector<double>> pre;   // prefix sums of G^2 over d = -(n-1)..(n-1)
  DeviceConv* dev = nullptr;              // RS_FLAG_DEVICE_FFT: convolutions on the device

  ConvOps(int n_, double h, const std::vector<double>& t_long) : n(n_), RL((int)t_long.size()) {
    N = 1;
    while (N < 3 * n) N <<= 1;
    fft = la::FFT(N);
    G.assign(RL, std::vector<double>(n));
    FG.assign(RL, std::vector<cplx>(N));
    nrm.assign(RL, std::vector<double>(n));
    pre.assign(RL, std::vector<double>(2 * n, 0.0));
#pragma omp parallel for schedule(dynamic)
    for (int k = 0; k < RL; ++k) {
      for (int d = 0; d < n; ++d) G[k][d] = cell_average(t_long[k], h, d);
      std::vector<cplx>& f = FG[k];
      std::fill(f.begin(), f.end(), cplx(0, 0));
      for (int m = 0; m < 2 * n - 1; ++m) f[m] = G[k][std::abs(m - (n - 1))];
      fft.forward(f.data());
      // prefix sums of G^2 over d = -(n-1)..(n-1)
      std::vector<double>& pk = pre[k];
      for (int m = 0; m < 2 * n - 1; ++m) {
        double g = G[k][std::abs(m - (n - 1))];
        pk[m + 1] = pk[m] + g * g;
      }
      // N_k(j)^2 = sum_{i=0}^{n-1} G[i-j]^2 = sum_{d=-j}^{n-1-j}; index m = d + n - 1
      for (int j = 0; j < n; ++j) nrm[k][j] = wnorm(k, j, 0, n - 1);
    }
  }

  // sqrt(sum_{i=lo}^{hi} G[i-j]^2): the column norm over the rows of a box (scheme (B))
  double wnorm(int k, int j, int lo, int hi) const {
    const int m0 = lo - j + n - 1, m1 = hi - j + n - 1;
    return std::sqrt(std::max(0.0, pre[k][m1 + 1] - pre[k][m0]));
  }

  // y_s = T_k x_s for the columns s of X (n x p column-major); Y likewise.
  void apply_one(int k, const double* X, double* Y, int p) const {
    if (dev && dev->apply(k, X, Y, p)) return;
    std::vector<cplx> buf(N);
    for (int s = 0; s < p; s += 2) {
      std::fill(buf.begin(), buf.end(), cplx(0, 0));
      const bool two = s + 1 < p;
      for (int i = 0; i < n; ++i)
        buf[i] = cplx(X[(size_t)s * n + i], two ? X[(size_t)(s + 1) * n + i] : 0.0);
      fft.forward(buf.data());
      for (int m = 0; m < N; ++m) buf[m] *= FG[k][m];
      fft.inverse(buf.data());
      const double inv = 1.0 / N;
      for (int i = 0; i < n; ++i) {
        Y[(size_t)s * n + i] = buf[i + n - 1].real() * inv;
        if (two) Y[(size_t)(s + 1) * n + i] = buf[i + n - 1].imag() * inv;
      }
    }
  }
};

// RS_SETUP_TIMING: per-phase wall times of the range finder (stderr)
struct PhaseClock {
  bool on = std::getenv("RS_SETUP_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void lap(int mode, const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[rs setup]     mode %d %-14s %7.3f s\n", mode, what,
                 std::chrono::duration<double>(now - t).count());
    t = now;
  }
};

// Thin orthonormal basis of the columns of Y (n x p) in place: CholeskyQR2 (the Gram matrix
// Y^T Y, its Cholesky factor R, Y <- Y R^-1, twice; the second pass restores orthogonality to
// rounding), OpenMP over rows; a Householder QR when a Cholesky pivot vanishes (rank-deficient
// Y, e.g. rows clipped to a box).  The result spans the same space (one basis of it).
namespace {
bool cholesky_qr_pass(std::vector<double>& Y, int n, int p) {
  // Gram matrix over 64 fixed row blocks summed in block order: bitwise independent of the
  // thread count (the setup is deterministic)
  constexpr int kBlocks = 64;
  std::vector<std::vector<double>> part(kBlocks);
#pragma omp parallel for schedule(dynamic)
  for (int blk = 0; blk < kBlocks; ++blk) {
    std::vector<double> g((size_t)p * p, 0.0);
    const int i0 = (int)((int64_t)n * blk / kBlocks), i1 = (int)((int64_t)n * (blk + 1) / kBlocks);
    for (int i = i0; i < i1; ++i)
      for (int a = 0; a < p; ++a) {
        const double ya = Y[(size_t)a * n + i];
        if (ya == 0.0) continue;
        for (int b = a; b < p; ++b) g[(size_t)a * p + b] += ya * Y[(size_t)b * n + i];
      }
    part[blk].swap(g);
  }
  std::vector<double> G((size_t)p * p, 0.0);
  for (int blk = 0; blk < kBlocks; ++blk)
    for (size_t t = 0; t < G.size(); ++t) G[t] += part[blk][t];
  // G = R^T R, R upper triangular (row-major R[a][b], a <= b)
  std::vector<double> R((size_t)p * p, 0.0);
  double dmax = 0.0;
  for (int a = 0; a < p; ++a) dmax = std::max(dmax, G[(size_t)a * p + a]);
  for (int a = 0; a < p; ++a) {
    double d = G[(size_t)a * p + a];
    for (int k = 0; k < a; ++k) d -= R[(size_t)k * p + a] * R[(size_t)k * p + a];
    if (!(d > 1e-24 * dmax)) return false;
    const double r = std::sqrt(d);
    R[(size_t)a * p + a] = r;
    for (int b = a + 1; b < p; ++b) {
      double v = G[(size_t)a * p + b];
      for (int k = 0; k < a; ++k) v -= R[(size_t)k * p + a] * R[(size_t)k * p + b];
      R[(size_t)a * p + b] = v / r;
    }
  }
  // each row y of Y: x R = y (forward substitution over the columns)
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i)
    for (int b = 0; b < p; ++b) {
      double v = Y[(size_t)b * n + i];
      for (int a = 0; a < b; ++a) v -= Y[(size_t)a * n + i] * R[(size_t)a * p + b];
      Y[(size_t)b * n + i] = v / R[(size_t)b * p + b];
    }
  return true;
}
}  // namespace

void orthonormalise(std::vector<double>& Y, int n, int p) {
  std::vector<double> keep = Y;
  if (n >= p && cholesky_qr_pass(Y, n, p) && cholesky_qr_pass(Y, n, p)) return;
  Y.swap(keep);
  std::vector<double> tau;
  std::vector<double> A = Y;
  la::householder_qr(A.data(), n, p, tau);
  la::form_q(A.data(), n, p, tau, Y.data());
}

// Mode-l RHOSVD basis.  c[k][j] = sum_{m at j} D_{mk}^2 with D_{mk} = |z_m a_k| times the
// windowed norms of the other two modes' columns (the Khatri-Rao column norms of the
// unfolding T_(l) = A_l diag(z a) (A_l'' kr A_l')^T).
struct ModeBasis {
  std::vector<double> U;      // n x r column-major
  std::vector<double> sigma;  // singular values of the weighted side matrix (p of them)
  int r = 0;
  double tail = 0;            // relative discarded energy sqrt(sum_{i>=r} s^2 / sum s^2)
};

// box (scheme (B), N3): the side matrix of this mode is restricted to the rows lo..hi of the
// box (P_box A), and the other modes' column norms to their box rows; null = the whole grid.
ModeBasis mode_basis(const ConvOps& ops, int mode, const std::vector<int32_t>& cells,
                     const std::vector<double>& z, const std::vector<double>& a_long,
                     int rank_R, double eps, int tucker_cap, uint64_t seed,
                     const int* box_lo = nullptr, const int* box_hi = nullptr) {
  const int n = ops.n, RL = ops.RL;
  const int row_lo = box_lo ? box_lo[mode] : 0, row_hi = box_hi ? box_hi[mode] : n - 1;
  auto clip_rows = [&](std::vector<double>& Y, int cols) {   // P_box
    if (!box_lo) return;
    for (int s_ = 0; s_ < cols; ++s_)
      for (int i = 0; i < n; ++i)
        if (i < row_lo || i > row_hi) Y[(size_t)s_ * n + i] = 0.0;
  };
  const int64_t M = (int64_t)z.size();
  const int l1 = (mode + 1) % 3, l2 = (mode + 2) % 3;
  std::vector<std::vector<double>> c(RL, std::vector<double>(n, 0.0));
  std::vector<char> occ(n, 0);
  for (int64_t m = 0; m < M; ++m) {
    const int j = cells[3 * m + mode];
    occ[j] = 1;
    for (int k = 0; k < RL; ++k) {
      const double n1 = box_lo ? ops.wnorm(k, cells[3 * m + l1], box_lo[l1], box_hi[l1])
                               : ops.nrm[k][cells[3 * m + l1]];
      const double n2 = box_lo ? ops.wnorm(k, cells[3 * m + l2], box_lo[l2], box_hi[l2])
                               : ops.nrm[k][cells[3 * m + l2]];
      double d = z[m] * a_long[k] * n1 * n2;
      c[k][j] += d * d;
    }
  }
  std::vector<int> occj;
  for (int j = 0; j < n; ++j)
    if (occ[j]) occj.push_back(j);

  const int pmax = std::min(row_hi - row_lo + 1, 512);
  // the largest Tucker rank this build can keep; a fixed-width build starts its sketch at the
  // 2 r_cap + 16 columns that resolve it (one range-finder pass instead of a doubling sequence)
  const int r_cap = rank_R > 0 ? (tucker_cap > 0 ? std::max(rank_R, tucker_cap) : rank_R + 8)
                               : (tucker_cap > 0 ? tucker_cap : n);
  int p = (rank_R > 0) ? std::min(pmax, std::max(2 * r_cap + 16, 48)) : std::min(pmax, 64);
  ModeBasis out;
  std::unique_ptr<RangeFinderDevice> rf;
  if (ops.dev && !box_lo) {
    rf.reset(new RangeFinderDevice(*ops.dev, c, n));
    if (!rf->ok()) rf.reset();
  }
  PhaseClock pc;
  pc.lap(mode, "weights");
  for (;;) {
    // range finder: Y = sum_k T_k (sqrt(c_k) .* Xi_k).  Per-k results are summed in k order
    // so the setup is bitwise independent of the thread count.  Device-FFT builds (no box) run
    // the sums on the device (RangeFinderDevice), the host path below otherwise.
    std::vector<double> Y((size_t)n * p, 0.0);
    std::vector<std::vector<double>> Yk(RL);
    if (!(rf && rf->sketch(p, seed, mode, occj, Y))) {
    rf.reset();
    std::fill(Y.begin(), Y.end(), 0.0);
#pragma omp parallel
    {
      std::vector<double> X((size_t)n * p);
#pragma omp for schedule(dynamic)
      for (int k = 0; k < RL; ++k) {
        std::fill(X.begin(), X.end(), 0.0);
        for (int s = 0; s < p; ++s)
          for (int j : occj)
            X[(size_t)s * n + j] = std::sqrt(c[k][j]) *
                la::normal(seed + 0x51ED27ull * (mode + 1), ((uint64_t)k * n + j) * 4096u + s);
        Yk[k].assign((size_t)n * p, 0.0);
        ops.apply_one(k, X.data(), Yk[k].data(), p);
      }
    }
    for (int k = 0; k < RL; ++k) {
      for (size_t i = 0; i < Y.size(); ++i) Y[i] += Yk[k][i];
      std::vector<double>().swap(Yk[k]);
    }
    }
    pc.lap(mode, "sketch");
    clip_rows(Y, p);
    orthonormalise(Y, n, p);
    clip_rows(Y, p);
    pc.lap(mode, "qr1");
    // one power iteration: Y = sum_k T_k (c_k .* (T_k Q))
    {
      std::vector<double> Y2((size_t)n * p, 0.0);
      if (!(rf && rf->power(Y, p, Y2))) {
      rf.reset();
      std::fill(Y2.begin(), Y2.end(), 0.0);
#pragma omp parallel
      {
        std::vector<double> Z((size_t)n * p);
#pragma omp for schedule(dynamic)
        for (int k = 0; k < RL; ++k) {
          ops.apply_one(k, Y.data(), Z.data(), p);
          for (int s = 0; s < p; ++s)
            for (int j = 0; j < n; ++j) Z[(size_t)s * n + j] *= c[k][j];
          Yk[k].assign((size_t)n * p, 0.0);
          ops.apply_one(k, Z.data(), Yk[k].data(), p);
        }
      }
      for (int k = 0; k < RL; ++k) {
        for (size_t i = 0; i < Y2.size(); ++i) Y2[i] += Yk[k][i];
        std::vector<double>().swap(Yk[k]);
      }
      }
      Y.swap(Y2);
      pc.lap(mode, "power");
      clip_rows(Y, p);
      orthonormalise(Y, n, p);
      clip_rows(Y, p);
      pc.lap(mode, "qr2");
    }
    // W^T Q, stacked over (k, occupied j): rows sqrt(c_k[j]) (T_k Q)[j, :].  Its singular values
    // and right vectors from the p x p Gram matrix sum_k sum_j c_k[j] Z_k[j,:]^T Z_k[j,:]
    // (Z_k = T_k Q; per k in parallel, summed in k order: bitwise independent of the thread
    // count), by the Jacobi eigensolver; sigma = sqrt(lambda) descending.  (Squaring costs
    // accuracy only below ~1e-8 sigma_0, far under the ranks kept.)
    std::vector<double> Gm((size_t)p * p, 0.0);
    if (!(rf && rf->gram(Y, p, Gm))) {
    rf.reset();
    std::fill(Gm.begin(), Gm.end(), 0.0);
    const int nocc = (int)occj.size();
    std::vector<std::vector<double>> Zk(RL);   // (T_k Q) at the occupied rows, nocc x p
#pragma omp parallel
    {
      std::vector<double> Z((size_t)n * p);
#pragma omp for schedule(dynamic)
      for (int k = 0; k < RL; ++k) {
        ops.apply_one(k, Y.data(), Z.data(), p);
        Zk[k].assign((size_t)nocc * p, 0.0);
        for (int jj = 0; jj < nocc; ++jj)
          for (int s = 0; s < p; ++s) Zk[k][(size_t)jj * p + s] = Z[(size_t)s * n + occj[jj]];
      }
    }
    pc.lap(mode, "WtQ apply");
    std::vector<std::vector<double>> Gk(RL);
#pragma omp parallel for schedule(dynamic)
    for (int k = 0; k < RL; ++k) {
      std::vector<double> g((size_t)p * p, 0.0);
      for (int jj = 0; jj < nocc; ++jj) {
        const double cw = c[k][occj[jj]];
        if (cw == 0.0) continue;
        const double* zr = Zk[k].data() + (size_t)jj * p;
        for (int s_ = 0; s_ < p; ++s_) {
          const double v = cw * zr[s_];
          for (int t = s_; t < p; ++t) g[(size_t)s_ * p + t] += v * zr[t];
        }
      }
      Gk[k].swap(g);
      std::vector<double>().swap(Zk[k]);
    }
    for (int k = 0; k < RL; ++k)
      for (size_t t = 0; t < Gm.size(); ++t) Gm[t] += Gk[k][t];
    for (int s_ = 0; s_ < p; ++s_)
      for (int t = s_ + 1; t < p; ++t) Gm[(size_t)t * p + s_] = Gm[(size_t)s_ * p + t];
    }
    pc.lap(mode, "WtQ gram");
    std::vector<double> lam(p), Ve((size_t)p * p);
    la::sym_eig(Gm.data(), p, lam.data(), Ve.data());   // ascending
    std::vector<double> sv(p), V((size_t)p * p);
    for (int i = 0; i < p; ++i) {
      const int src = p - 1 - i;
      sv[i] = std::sqrt(std::max(lam[src], 0.0));
      for (int s_ = 0; s_ < p; ++s_) V[(size_t)i * p + s_] = Ve[(size_t)src * p + s_];
    }
    pc.lap(mode, "svd");
    double tot = 0;
    for (double v : sv) tot += v * v;
    // rank for the tolerance
    int r_tol = p;
    {
      double tail = 0;
      for (int i = p - 1; i >= 0; --i) {
        if (std::sqrt(tail + sv[i] * sv[i]) > eps * std::sqrt(tot)) {
          r_tol = i + 1;
          break;
        }
        tail += sv[i] * sv[i];
        r_tol = i;
      }
      r_tol = std::max(r_tol, 1);
    }
    // resolved: the spectrum fell below the tolerance, or the sketch already oversamples the
    // largest rank this build can keep (r_cap) by r_cap + 16 columns (one power iteration)
    const bool resolved = sv[p - 1] <= 0.1 * eps * sv[0] || p >= pmax ||
                          p >= 2 * r_cap + 16;
    if (!resolved && r_tol >= p - 4) {
      p = std::min(pmax, 2 * p);
      continue;
    }
    int r;
    // fixed width R: Tucker rank r_tol at eps, limited to R + 8 by default or to an explicit
    // tucker_cap (a richer Tucker form for rs_restrict_box, N3); tolerance mode: r_tol
    if (rank_R > 0) r = std::max(rank_R, std::min(r_tol, tucker_cap > 0 ? tucker_cap : rank_R + 8));
    else r = r_tol;
    if (tucker_cap > 0) r = std::min(r, tucker_cap);
    r = std::min(r, std::min(p, n));
    double tail = 0;
    for (int i = r; i < p; ++i) tail += sv[i] * sv[i];
    out.r = r;
    out.tail = tot > 0 ? std::sqrt(tail / tot) : 0.0;
    out.sigma = sv;
    out.U.assign((size_t)n * r, 0.0);
    for (int a = 0; a < r; ++a)
      for (int s = 0; s < p; ++s) {
        const double v = V[(size_t)a * p + s];
        if (v == 0.0) continue;
        for (int i = 0; i < n; ++i) out.U[(size_t)a * n + i] += Y[(size_t)s * n + i] * v;
      }
    return out;
  }
}

// dense CP reconstruction error ||G - [[A,B,C]]|| (G r0 x r1 x r2 row-major, factors
// column-major r_l x R)
double cp_error(const std::vector<double>& G, int r0, int r1, int r2, const std::vector<double>& A,
                const std::vector<double>& B, const std::vector<double>& C, int R) {
  double err = 0;
  for (int a = 0; a < r0; ++a)
    for (int b = 0; b < r1; ++b)
      for (int c = 0; c < r2; ++c) {
        double v = 0;
        for (int q = 0; q < R; ++q) v += A[(size_t)q * r0 + a] * B[(size_t)q * r1 + b] * C[(size_t)q * r2 + c];
        double d = G[((size_t)a * r1 + b) * r2 + c] - v;
        err += d * d;
      }
  return std::sqrt(err);
}

// X = Mt * pinv(V) for symmetric PSD V (R x R); Mt is r x R column-major.
void solve_normal(std::vector<double>& X, const std::vector<double>& Mt, std::vector<double> V,
                  int r, int R) {
  std::vector<double> w(R), E((size_t)R * R);
  la::sym_eig(V.data(), R, w.data(), E.data());
  double wmax = 0;
  for (double v : w) wmax = std::max(wmax, std::fabs(v));
  std::vector<double> Pinv((size_t)R * R, 0.0);
  for (int e = 0; e < R; ++e) {
    if (!(w[e] > 1e-13 * wmax)) continue;
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < R; ++j)
        Pinv[(size_t)j * R + i] += E[(size_t)e * R + i] * E[(size_t)e * R + j] / w[e];
  }
  X.assign((size_t)r * R, 0.0);
  for (int q = 0; q < R; ++q)
    for (int j = 0; j < R; ++j) {
      const double pij = Pinv[(size_t)q * R + j];
      if (pij == 0.0) continue;
      for (int i = 0; i < r; ++i) X[(size_t)q * r + i] += Mt[(size_t)j * r + i] * pij;
    }
}

void gram(const std::vector<double>& A, int r, int R, std::vector<double>& out) {
  out.assign((size_t)R * R, 0.0);
  for (int p = 0; p < R; ++p)
    for (int q = 0; q < R; ++q) {
      double s = 0;
      for (int i = 0; i < r; ++i) s += A[(size_t)p * r + i] * A[(size_t)q * r + i];
      out[(size_t)q * R + p] = s;
    }
}

void cp_als(const std::vector<double>& G, int r0, int r1, int r2, int R, int sweeps,
            std::vector<double>& A, std::vector<double>& B, std::vector<double>& C) {
  double gn = 0;
  for (double v : G) gn += v * v;
  gn = std::sqrt(gn);
  double prev = cp_error(G, r0, r1, r2, A, B, C, R);
  std::vector<double> Mt, V, V2;
  for (int it = 0; it < sweeps; ++it) {
    // A <- G_(0) (C kr B) ((B^T B) * (C^T C))^+
    Mt.assign((size_t)r0 * R, 0.0);
    for (int q = 0; q < R; ++q)
      for (int a = 0; a < r0; ++a) {
        double s = 0;
        for (int b = 0; b < r1; ++b) {
          const double bq = B[(size_t)q * r1 + b];
          const double* g = &G[((size_t)a * r1 + b) * r2];
          double t = 0;
          for (int c = 0; c < r2; ++c) t += g[c] * C[(size_t)q * r2 + c];
          s += bq * t;
        }
        Mt[(size_t)q * r0 + a] = s;
      }
    gram(B, r1, R, V);
    gram(C, r2, R, V2);
    for (size_t i = 0; i < V.size(); ++i) V[i] *= V2[i];
    solve_normal(A, Mt, V, r0, R);
    // B
    Mt.assign((size_t)r1 * R, 0.0);
    for (int q = 0; q < R; ++q)
      for (int b = 0; b < r1; ++b) {
        double s = 0;
        for (int a = 0; a < r0; ++a) {
          const double aq = A[(size_t)q * r0 + a];
          const double* g = &G[((size_t)a * r1 + b) * r2];
          double t = 0;
          for (int c = 0; c < r2; ++c) t += g[c] * C[(size_t)q * r2 + c];
          s += aq * t;
        }
        Mt[(size_t)q * r1 + b] = s;
      }
    gram(A, r0, R, V);
    gram(C, r2, R, V2);
    for (size_t i = 0; i < V.size(); ++i) V[i] *= V2[i];
    solve_normal(B, Mt, V, r1, R);
    // C
    Mt.assign((size_t)r2 * R, 0.0);
    for (int q = 0; q < R; ++q) {
      std::vector<double> acc(r2, 0.0);
      for (int a = 0; a < r0; ++a)
        for (int b = 0; b < r1; ++b) {
          const double w = A[(size_t)q * r0 + a] * B[(size_t)q * r1 + b];
          if (w == 0.0) continue;
          const double* g = &G[((size_t)a * r1 + b) * r2];
          for (int c = 0; c < r2; ++c) acc[c] += w * g[c];
        }
      for (int c = 0; c < r2; ++c) Mt[(size_t)q * r2 + c] = acc[c];
    }
    gram(A, r0, R, V);
    gram(B, r1, R, V2);
    for (size_t i = 0; i < V.size(); ++i) V[i] *= V2[i];
    solve_normal(C, Mt, V, r2, R);
    // normalise B, C columns into A
    for (int q = 0; q < R; ++q) {
      double nb = 0, nc = 0;
      for (int i = 0; i < r1; ++i) nb += B[(size_t)q * r1 + i] * B[(size_t)q * r1 + i];
      for (int i = 0; i < r2; ++i) nc += C[(size_t)q * r2 + i] * C[(size_t)q * r2 + i];
      nb = std::sqrt(nb);
      nc = std::sqrt(nc);
      if (nb > 0) for (int i = 0; i < r1; ++i) B[(size_t)q * r1 + i] /= nb;
      if (nc > 0) for (int i = 0; i < r2; ++i) C[(size_t)q * r2 + i] /= nc;
      for (int i = 0; i < r0; ++i) A[(size_t)q * r0 + i] *= nb * nc;
    }
    if ((it & 7) == 7 || it == sweeps - 1) {
      double e = cp_error(G, r0, r1, r2, A, B, C, R);
      if (std::fabs(prev - e) <= 1e-12 * gn) break;
      prev = e;
    }
  }
}

}  // namespace

// S7: core G (r0 x r1 x r2) -> CP of width rank_R (0: the smallest width whose dropped slice
// singular values stay within eps of the core norm): the exact canonical expansion from the
// SVDs of the slices G[a,:,:] = sum sigma u v^T, truncated, then CP-ALS when it was truncated.
// A (R blocks of r0), B, C: term q is A[q] o B[q] o C[q].  Returns R.
int core_to_cp(const std::vector<double>& G, int r0, int r1, int r2, int rank_R, double eps,
               int als_sweeps, std::vector<double>& A, std::vector<double>& B,
               std::vector<double>& C, int* R_exact, double* rel_err) {
  double gnorm = 0;
  for (double v : G) gnorm += v * v;
  gnorm = std::sqrt(gnorm);
  struct Trip { int a; double s; std::vector<double> u, v; };
  std::vector<Trip> trips;
  const bool tr = r1 < r2;              // Jacobi SVD wants rows >= cols
  const int mr = tr ? r2 : r1, nc = tr ? r1 : r2;
  for (int a = 0; a < r0; ++a) {
    std::vector<double> S((size_t)mr * nc), V((size_t)nc * nc), U((size_t)mr * nc), sv(nc);
    for (int b = 0; b < r1; ++b)
      for (int c = 0; c < r2; ++c) {
        const double v = G[((size_t)a * r1 + b) * r2 + c];
        if (!tr) S[(size_t)c * mr + b] = v; else S[(size_t)b * mr + c] = v;
      }
    la::jacobi_svd(S.data(), mr, nc, sv.data(), V.data(), U.data());
    for (int q = 0; q < nc; ++q) {
      if (!(sv[q] > 1e-15 * gnorm)) continue;
      Trip t;
      t.a = a;
      t.s = sv[q];
      std::vector<double> uu(U.begin() + (size_t)q * mr, U.begin() + (size_t)(q + 1) * mr);
      std::vector<double> vv(V.begin() + (size_t)q * nc, V.begin() + (size_t)(q + 1) * nc);
      if (!tr) { t.u = uu; t.v = vv; } else { t.u = vv; t.v = uu; }
      trips.push_back(std::move(t));
    }
  }
  std::stable_sort(trips.begin(), trips.end(), [](const Trip& x, const Trip& y) { return x.s > y.s; });
  *R_exact = (int)trips.size();
  int R;
  size_t keep = trips.size();
  if (rank_R <= 0) {
    double tot = 0, drop = 0;
    for (auto& t : trips) tot += t.s * t.s;
    while (keep > 1 && drop + trips[keep - 1].s * trips[keep - 1].s <= eps * eps * tot) {
      drop += trips[keep - 1].s * trips[keep - 1].s;
      --keep;
    }
    R = (int)keep;
  } else {
    R = rank_R;
    keep = std::min(trips.size(), (size_t)rank_R);
  }
  A.assign((size_t)r0 * R, 0.0);
  B.assign((size_t)r1 * R, 0.0);
  C.assign((size_t)r2 * R, 0.0);
  for (size_t q = 0; q < keep; ++q) {
    A[q * r0 + trips[q].a] = trips[q].s;
    for (int i = 0; i < r1; ++i) B[q * r1 + i] = trips[q].u[i];
    for (int i = 0; i < r2; ++i) C[q * r2 + i] = trips[q].v[i];
  }
  if (rank_R > 0 && (int)trips.size() > rank_R)
    cp_als(G, r0, r1, r2, R, als_sweeps > 0 ? als_sweeps : 300, A, B, C);
  *rel_err = gnorm > 0 ? cp_error(G, r0, r1, r2, A, B, C, R) / gnorm : 0.0;
  return R;
}

void compress_long_range(int n, double h, const std::vector<int32_t>& cells,
                         const std::vector<double>& z, const std::vector<double>& t_long,
                         const std::vector<double>& a_long, int rank_R, double eps,
                         int tucker_cap, int als_sweeps, uint64_t seed,
                         std::vector<double> F[3], int* R_out, SetupReport* rep,
                         TuckerRep* tk, const int* box_lo, const int* box_hi, int device,
                         bool device_fft) {
  ConvOps ops(n, h, t_long);
  std::unique_ptr<DeviceConv> dconv;
  if (device >= 0 && device_fft) {
    dconv.reset(new DeviceConv(device, n, ops.N, ops.FG));
    if (dconv->ok()) ops.dev = dconv.get();
  }
  const int RL = ops.RL;
  const int64_t M = (int64_t)z.size();
  ModeBasis mb[3];
  for (int l = 0; l < 3; ++l)
    mb[l] = mode_basis(ops, l, cells, z, a_long, rank_R, eps, tucker_cap, seed, box_lo, box_hi);
  const int r0 = mb[0].r, r1 = mb[1].r, r2 = mb[2].r;
  for (int l = 0; l < 3; ++l) rep->tucker_r[l] = mb[l].r;
  if (std::getenv("RS_SETUP_TIMING")) std::fprintf(stderr, "[rs setup]   mode bases done at %.3f\n", std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count());
  rep->tucker_err = std::sqrt(mb[0].tail * mb[0].tail + mb[1].tail * mb[1].tail +
                              mb[2].tail * mb[2].tail);

  // S6: core G = sum_k sum_m z_m a_k (U_0^T g_k[.-c_m0]) o (U_1^T ...) o (U_2^T ...)
  std::vector<double> G((size_t)r0 * r1 * r2, 0.0);
  // on the device when the build has one (bitwise the same core, setup_device.cu)
  const int rr_[3] = {r0, r1, r2};
  std::unique_ptr<CoreDevice> cdev;
  if (device >= 0 && (double)M * r0 * r1 * r2 * RL > 1e8) {
    cdev.reset(new CoreDevice(device, n, rr_, cells, z));
    if (!cdev->ok()) cdev.reset();
  }
  double t_conv = 0, t_add = 0;
  const bool timing = std::getenv("RS_SETUP_TIMING") != nullptr;
  // device convolutions and device accumulation: every term without leaving the device (the
  // same cuFFT calls and the same accumulation as the per-term loop below, so bitwise the same)
  int k0 = 0;
  if (cdev && ops.dev) {
    std::vector<double> U3[3] = {mb[0].U, mb[1].U, mb[2].U};
    if (cdev->add_terms_device(*ops.dev, U3, a_long)) k0 = RL;
    else cdev.reset();
  }
  for (int k = k0; k < RL; ++k) {
    std::vector<double> H[3];   // row-major n x r_l
    auto tc = std::chrono::steady_clock::now();
    for (int l = 0; l < 3; ++l) {
      const int r = mb[l].r;
      std::vector<double> tmp((size_t)n * r);
      ops.apply_one(k, mb[l].U.data(), tmp.data(), r);
      H[l].assign((size_t)n * r, 0.0);
      for (int a = 0; a < r; ++a)
        for (int i = 0; i < n; ++i) H[l][(size_t)i * r + a] = tmp[(size_t)a * n + i];
    }
    if (timing) t_conv += std::chrono::duration<double>(std::chrono::steady_clock::now() - tc).count();
    if (cdev) {
      tc = std::chrono::steady_clock::now();
      const bool ok_add = cdev->add_term(a_long[k], H);
      if (timing) t_add += std::chrono::duration<double>(std::chrono::steady_clock::now() - tc).count();
      if (ok_add) continue;
      // the device failed mid-way: redo the core on the host from scratch
      cdev.reset();
      std::fill(G.begin(), G.end(), 0.0);
      k = -1;
      continue;
    }
#pragma omp parallel for schedule(dynamic)
    for (int a = 0; a < r0; ++a) {
      std::vector<double> row((size_t)r1 * r2, 0.0);
      for (int64_t m = 0; m < M; ++m) {
        const double w = z[m] * a_long[k] * H[0][(size_t)cells[3 * m] * r0 + a];
        if (w == 0.0) continue;
        const double* h1 = &H[1][(size_t)cells[3 * m + 1] * r1];
        const double* h2 = &H[2][(size_t)cells[3 * m + 2] * r2];
        for (int b = 0; b < r1; ++b) {
          const double wb = w * h1[b];
          double* dst = &row[(size_t)b * r2];
          for (int c = 0; c < r2; ++c) dst[c] += wb * h2[c];
        }
      }
      double* g = &G[(size_t)a * r1 * r2];
      for (size_t i = 0; i < row.size(); ++i) g[i] += row[i];
    }
  }
  if (cdev && !cdev->fetch(G)) {
    // could not read the device core back: the host loop (rare; keeps the build working)
    cdev.reset();
    std::fill(G.begin(), G.end(), 0.0);
    for (int k = 0; k < RL; ++k) {
      std::vector<double> H[3];
      for (int l = 0; l < 3; ++l) {
        const int r = mb[l].r;
        std::vector<double> tmp((size_t)n * r);
        ops.apply_one(k, mb[l].U.data(), tmp.data(), r);
        H[l].assign((size_t)n * r, 0.0);
        for (int a = 0; a < r; ++a)
          for (int i = 0; i < n; ++i) H[l][(size_t)i * r + a] = tmp[(size_t)a * n + i];
      }
      for (int a = 0; a < r0; ++a) {
        std::vector<double> row((size_t)r1 * r2, 0.0);
        for (int64_t m = 0; m < M; ++m) {
          const double w = z[m] * a_long[k] * H[0][(size_t)cells[3 * m] * r0 + a];
          if (w == 0.0) continue;
          const double* h1 = &H[1][(size_t)cells[3 * m + 1] * r1];
          const double* h2 = &H[2][(size_t)cells[3 * m + 2] * r2];
          for (int b = 0; b < r1; ++b) {
            const double wb = w * h1[b];
            double* dst = &row[(size_t)b * r2];
            for (int c = 0; c < r2; ++c) dst[c] += wb * h2[c];
          }
        }
        double* g = &G[(size_t)a * r1 * r2];
        for (size_t i = 0; i < row.size(); ++i) g[i] += row[i];
      }
    }
  }
  if (timing) std::fprintf(stderr, "[rs setup]     core: convolutions %.3f s, device accumulation %.3f s\n", t_conv, t_add);
  if (std::getenv("RS_SETUP_TIMING")) std::fprintf(stderr, "[rs setup]   core done at %.3f\n", std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count());
  // S7: core -> CP of width R
  std::vector<double> A, B, C;
  const int R = core_to_cp(G, r0, r1, r2, rank_R, eps, als_sweeps, A, B, C, &rep->R_exact,
                           &rep->cp_core_err);
  if (tk) {
    for (int l = 0; l < 3; ++l) { tk->r[l] = mb[l].r; tk->U[l] = mb[l].U; }
    tk->G = G;
  }

  // F_l = U_l X_l  (n x R row-major)
  const std::vector<double>* X[3] = {&A, &B, &C};
  const int rr[3] = {r0, r1, r2};
  for (int l = 0; l < 3; ++l) {
    F[l].assign((size_t)n * R, 0.0);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i)
      for (int q = 0; q < R; ++q) {
        double s = 0;
        for (int a = 0; a < rr[l]; ++a) s += mb[l].U[(size_t)a * n + i] * (*X[l])[(size_t)q * rr[l] + a];
        F[l][(size_t)i * R + q] = s;
      }
  }
  if (box_lo)                           // scheme (B): the tensor says nothing outside the box
    for (int l = 0; l < 3; ++l)
      for (int i = 0; i < n; ++i)
        if (i < box_lo[l] || i > box_hi[l])
          for (int q = 0; q < R; ++q) F[l][(size_t)i * R + q] = std::numeric_limits<double>::quiet_NaN();
  *R_out = R;
}

// ---- NEXT row N3: scheme (C), recompression inside a box ------------------
// Rows lo_l..hi_l of the Tucker bases U_l (n x r_l) of the long-range part: their SVD
// U_l[lo:hi] = Q_l diag(s_l) V_l^T gives orthonormal Q_l (m_l x r'_l) and S_l = diag(s_l) V_l^T
// (r'_l x r_l, singular values above 1e-13 s_max kept); the box's Tucker core is
// G_box = G x_0 S_0 x_1 S_1 x_2 S_2 and its CP (core_to_cp, width rank or eps) gives the box
// factors F_l = Q_l X_l in rows lo_l..hi_l.  Rows outside the box are NaN: a ligand atom outside
// the box makes the pose's energy NaN (the restricted tensor says nothing there).
int restrict_to_box(int n, const TuckerRep& tk, const int lo[3], const int hi[3], int rank,
                    double eps, int als_sweeps, std::vector<double> F[3], SetupReport* rep) {
  std::vector<double> Q[3], S[3];
  int rp[3];
  for (int l = 0; l < 3; ++l) {
    const int r = tk.r[l], m = hi[l] - lo[l] + 1;
    const bool tall = m >= r;
    const int mr = tall ? m : r, nc = tall ? r : m;
    std::vector<double> Aw((size_t)mr * nc), V((size_t)nc * nc), U((size_t)mr * nc), sv(nc);
    for (int a = 0; a < r; ++a)
      for (int i = 0; i < m; ++i) {
        const double u = tk.U[l][(size_t)a * n + lo[l] + i];
        if (tall) Aw[(size_t)a * mr + i] = u; else Aw[(size_t)i * mr + a] = u;
      }
    la::jacobi_svd(Aw.data(), mr, nc, sv.data(), V.data(), U.data());
    // tall: U_box = U diag(s) V^T;  wide: U_box^T = U diag(s) V^T, so U_box = V diag(s) U^T
    int keep = 0;
    while (keep < nc && sv[keep] > 1e-13 * sv[0]) ++keep;
    rp[l] = keep;
    Q[l].assign((size_t)m * keep, 0.0);          // column-major m x keep
    S[l].assign((size_t)keep * r, 0.0);          // row j: s_j (right vector)^T over a
    for (int j = 0; j < keep; ++j) {
      const double* left = tall ? &U[(size_t)j * mr] : &V[(size_t)j * nc];    // length m
      const double* right = tall ? &V[(size_t)j * nc] : &U[(size_t)j * mr];   // length r
      for (int i = 0; i < m; ++i) Q[l][(size_t)j * m + i] = left[i];
      for (int a = 0; a < r; ++a) S[l][(size_t)j * r + a] = sv[j] * right[a];
    }
  }
  // G_box[j0,j1,j2] = sum_abc S0[j0,a] S1[j1,b] S2[j2,c] G[a,b,c], one mode at a time
  const int r0 = tk.r[0], r1 = tk.r[1], r2 = tk.r[2];
  std::vector<double> T2((size_t)r0 * r1 * rp[2], 0.0);
  for (size_t ab = 0; ab < (size_t)r0 * r1; ++ab)
    for (int j = 0; j < rp[2]; ++j) {
      double s = 0;
      for (int c = 0; c < r2; ++c) s += tk.G[ab * r2 + c] * S[2][(size_t)j * r2 + c];
      T2[ab * rp[2] + j] = s;
    }
  std::vector<double> T1((size_t)r0 * rp[1] * rp[2], 0.0);
  for (int a = 0; a < r0; ++a)
    for (int j = 0; j < rp[1]; ++j)
      for (int b = 0; b < r1; ++b) {
        const double w = S[1][(size_t)j * r1 + b];
        const double* src = &T2[((size_t)a * r1 + b) * rp[2]];
        double* dst = &T1[((size_t)a * rp[1] + j) * rp[2]];
        for (int c = 0; c < rp[2]; ++c) dst[c] += w * src[c];
      }
  std::vector<double> Gb((size_t)rp[0] * rp[1] * rp[2], 0.0);
  const size_t slab = (size_t)rp[1] * rp[2];
  for (int j = 0; j < rp[0]; ++j)
    for (int a = 0; a < r0; ++a) {
      const double w = S[0][(size_t)j * r0 + a];
      for (size_t x = 0; x < slab; ++x) Gb[j * slab + x] += w * T1[a * slab + x];
    }
  std::vector<double> A, B, C;
  const int R = core_to_cp(Gb, rp[0], rp[1], rp[2], rank, eps, als_sweeps, A, B, C,
                           &rep->R_exact, &rep->cp_core_err);
  for (int l = 0; l < 3; ++l) rep->tucker_r[l] = rp[l];
  const std::vector<double>* X[3] = {&A, &B, &C};
  for (int l = 0; l < 3; ++l) {
    const int m = hi[l] - lo[l] + 1;
    F[l].assign((size_t)n * R, std::numeric_limits<double>::quiet_NaN());
    for (int i = 0; i < m; ++i)
      for (int q = 0; q < R; ++q) {
        double s = 0;
        for (int j = 0; j < rp[l]; ++j) s += Q[l][(size_t)j * m + i] * (*X[l])[(size_t)q * rp[l] + j];
        F[l][(size_t)(lo[l] + i) * R + q] = s;
      }
  }
  return R;
}

// ---- S9: cell lists --------------------------------------------------------------------------
void build_cell_lists(int n, double b, double h, const std::vector<double>& xyz,
                      const std::vector<int32_t>& cells, double rho, double cell_edge,
                      CoarseGrid* cg) {
  const int64_t M = (int64_t)cells.size() / 3;
  // automatic edge: about rho/4 (fewer candidates per atom: a pair list holds every atom within
  // rr of the cell's box, so the false candidates shrink with the cell), coarsened while the
  // estimated entry count M * |cube (+) ball(rr)| / c^3 exceeds kMaxEntries
  const double target = cell_edge > 0 ? cell_edge : rho / 4.0;
  int shift = 0;
  while (shift < 15 && h * double(1 << (shift + 1)) <= target * 1.4142) ++shift;
  if (cell_edge <= 0) {
    const double kMaxEntries = 64.0 * (1 << 20);
    const double r = rho + 2 * h, pi = 3.14159265358979323846;
    for (; shift < 15; ++shift) {
      const double c = h * double(1 << shift);
      const double v = c * c * c + 6 * c * c * r + 3 * pi * c * r * r + 4.0 / 3.0 * pi * r * r * r;
      if (double(M) * v / (c * c * c) <= kMaxEntries) break;
    }
  }
  cg->shift = shift;
  const int pf = (int)std::ceil((rho + 2 * h) / h) + 1;
  for (int a = 0; a < 3; ++a) {
    int mn = n, mx = -1;
    for (int64_t m = 0; m < M; ++m) {
      mn = std::min(mn, (int)cells[3 * m + a]);
      mx = std::max(mx, (int)cells[3 * m + a]);
    }
    if (M == 0) { mn = 0; mx = 0; }
    const int lo = std::max(0, mn - pf) >> shift;
    const int hi = std::min(n - 1, mx + pf) >> shift;
    cg->lo[a] = lo;
    cg->dim[a] = hi - lo + 1;
  }
  const int64_t ncell = (int64_t)cg->dim[0] * cg->dim[1] * cg->dim[2];
  std::vector<int32_t> cnt(ncell + 1, 0);
  const double cw = h * double(1 << shift);
  const double rr = rho + 2 * h, rr2 = rr * rr;
  auto visit = [&](int64_t m, auto&& fn) {
    const double* x = &xyz[3 * m];
    int c0[3], c1[3];
    for (int a = 0; a < 3; ++a) {
      int f0 = (int)std::floor((x[a] - rr + b) / h) - 1, f1 = (int)std::floor((x[a] + rr + b) / h) + 1;
      f0 = std::max(f0, 0);
      f1 = std::min(f1, n - 1);
      c0[a] = std::max(f0 >> shift, cg->lo[a]);
      c1[a] = std::min(f1 >> shift, cg->lo[a] + cg->dim[a] - 1);
    }
    for (int i = c0[0]; i <= c1[0]; ++i) {
      const double lo0 = -b + i * cw, hi0 = lo0 + cw;
      const double d0 = std::max({0.0, lo0 - x[0], x[0] - hi0});
      for (int j = c0[1]; j <= c1[1]; ++j) {
        const double lo1 = -b + j * cw, hi1 = lo1 + cw;
        const double d1 = std::max({0.0, lo1 - x[1], x[1] - hi1});
        if (d0 * d0 + d1 * d1 > rr2) continue;
        for (int k = c0[2]; k <= c1[2]; ++k) {
          const double lo2 = -b + k * cw, hi2 = lo2 + cw;
          const double d2 = std::max({0.0, lo2 - x[2], x[2] - hi2});
          if (d0 * d0 + d1 * d1 + d2 * d2 > rr2) continue;
          const int64_t cell = ((int64_t)(i - cg->lo[0]) * cg->dim[1] + (j - cg->lo[1])) * cg->dim[2] +
                               (k - cg->lo[2]);
          fn(cell);
        }
      }
    }
  };
  // counts and fill over the atoms in parallel (atomic slots), then every cell's list sorted
  // back to ascending atom index: the same lists as a serial pass over the atoms
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t m = 0; m < M; ++m)
    visit(m, [&](int64_t c) {
#pragma omp atomic
      cnt[c + 1]++;
    });
  for (int64_t c = 0; c < ncell; ++c) cnt[c + 1] += cnt[c];
  cg->off = cnt;
  cg->idx.assign(cnt[ncell], 0);
  std::vector<int32_t> pos(cnt.begin(), cnt.end() - 1);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t m = 0; m < M; ++m)
    visit(m, [&](int64_t c) {
      int32_t slot;
#pragma omp atomic capture
      slot = pos[c]++;
      cg->idx[slot] = (int32_t)m;
    });
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t c = 0; c < ncell; ++c)
    if (cnt[c + 1] - cnt[c] > 1) std::sort(cg->idx.begin() + cnt[c], cg->idx.begin() + cnt[c + 1]);
}

// ---- sampled compression error (reported; O11(iii) re-checks it independently) ---------------
void sample_compression_error(int n, double b, double h, const std::vector<double>& xyz,
                              const std::vector<int32_t>& cells, const std::vector<double>& z,
                              const std::vector<double>& t_long, const std::vector<double>& a_long,
                              const std::vector<double> F[3], int R, double r_excl,
                              const CoarseGrid& cg, int n_samples, uint64_t seed,
                              SetupReport* rep, int device) {
  const int64_t M = (int64_t)z.size();
  const int RL = (int)t_long.size();
  if (M == 0 || n_samples <= 0) return;
  std::vector<double> G((size_t)RL * n);
  for (int k = 0; k < RL; ++k)
    for (int d = 0; d < n; ++d) G[(size_t)k * n + d] = cell_average(t_long[k], h, d);
  const double inv_h = double(n) / (2.0 * b);
  auto snapc = [&](double x) {
    double u = (x + b) * inv_h;
    double c = std::ceil(u) - 1.0;
    c = std::min(std::max(c, 0.0), double(n - 1));
    return (int)c;
  };
  // sample exterior points: x = x_m + delta u, delta in [r_excl, 4 r_excl], no atom within r_excl
  std::vector<int> pts;
  uint64_t ctr = 0;
  const double rx2 = r_excl * r_excl;
  while ((int)pts.size() / 3 < n_samples && ctr < (uint64_t)n_samples * 400) {
    const double u0 = la::normal(seed ^ 0xABCDEFull, ctr * 5 + 0);
    const double u1 = la::normal(seed ^ 0xABCDEFull, ctr * 5 + 1);
    const double u2 = la::normal(seed ^ 0xABCDEFull, ctr * 5 + 2);
    const double uu = la::normal(seed ^ 0xABCDEFull, ctr * 5 + 3);
    const double vv = la::normal(seed ^ 0xABCDEFull, ctr * 5 + 4);
    ++ctr;
    const double nu = std::sqrt(u0 * u0 + u1 * u1 + u2 * u2);
    if (!(nu > 0)) continue;
    const int64_t m = (int64_t)(std::fabs(uu) * 1e6) % M;
    const double delta = r_excl * (1.0 + 3.0 * (0.5 + 0.5 * std::erf(vv / std::sqrt(2.0))));
    double x[3] = {xyz[3 * m] + delta * u0 / nu, xyz[3 * m + 1] + delta * u1 / nu,
                   xyz[3 * m + 2] + delta * u2 / nu};
    bool ok = true;
    for (int a = 0; a < 3; ++a) ok = ok && x[a] > -b + h && x[a] < b - h;
    if (!ok) continue;
    int c[3] = {snapc(x[0]), snapc(x[1]), snapc(x[2])};
    // exclusion via the cell lists (they cover every atom within rho >= r_excl)
    int cc[3];
    for (int a = 0; a < 3; ++a) cc[a] = (c[a] >> cg.shift) - cg.lo[a];
    if (cc[0] >= 0 && cc[0] < cg.dim[0] && cc[1] >= 0 && cc[1] < cg.dim[1] && cc[2] >= 0 &&
        cc[2] < cg.dim[2]) {
      const int64_t cell = ((int64_t)cc[0] * cg.dim[1] + cc[1]) * cg.dim[2] + cc[2];
      for (int32_t e = cg.off[cell]; e < cg.off[cell + 1] && ok; ++e) {
        const int32_t q = cg.idx[e];
        double d2 = 0;
        for (int a = 0; a < 3; ++a) d2 += (x[a] - xyz[3 * q + a]) * (x[a] - xyz[3 * q + a]);
        if (d2 < rx2) ok = false;
      }
    }
    if (!ok) continue;
    pts.push_back(c[0]);
    pts.push_back(c[1]);
    pts.push_back(c[2]);
  }
  const int ns = (int)pts.size() / 3;
  std::vector<double> ex(ns), cp(ns);
  // the uncompressed values: on the device when the build has one (the O(ns M R_l) sum)
  const bool on_dev = device >= 0 && exact_long_values_device(device, n, G, a_long, cells, z, pts, ex);
#pragma omp parallel for schedule(dynamic)
  for (int s = 0; s < ns; ++s) {
    const int* c = &pts[3 * s];
    double v = 0;
    for (int64_t m = 0; m < M && !on_dev; ++m) {
      const int d0 = std::abs(c[0] - cells[3 * m]), d1 = std::abs(c[1] - cells[3 * m + 1]),
                d2 = std::abs(c[2] - cells[3 * m + 2]);
      double acc = 0;
      for (int k = 0; k < RL; ++k)
        acc += a_long[k] * G[(size_t)k * n + d0] * G[(size_t)k * n + d1] * G[(size_t)k * n + d2];
      v += z[m] * acc;
    }
    if (!on_dev) ex[s] = v;
    double w = 0;
    for (int q = 0; q < R; ++q)
      w += F[0][(size_t)c[0] * R + q] * F[1][(size_t)c[1] * R + q] * F[2][(size_t)c[2] * R + q];
    cp[s] = w;
  }
  double emax = 0, vmax = 0, e2 = 0, v2 = 0;
  for (int s = 0; s < ns; ++s) {
    emax = std::max(emax, std::fabs(ex[s] - cp[s]));
    vmax = std::max(vmax, std::fabs(ex[s]));
    e2 += (ex[s] - cp[s]) * (ex[s] - cp[s]);
    v2 += ex[s] * ex[s];
  }
  rep->n_samples = ns;
  rep->sampled_max = vmax > 0 ? emax / vmax : 0.0;
  rep->sampled_rms = v2 > 0 ? std::sqrt(e2 / v2) : 0.0;
}

}  // namespace rs
