// Small dense linear-algebra and FFT helpers for the host setup (TEP step 4).
#pragma once

#include <complex>
#include <cstdint>
#include <vector>

namespace rs {
namespace la {

using cplx = std::complex<double>;

// Radix-2 complex FFT of a fixed power-of-two size.
struct FFT {
  int N = 0, logN = 0;
  std::vector<cplx> w;        // twiddles e^{-2 pi i k / N}, k < N/2
  std::vector<int> rev;
  explicit FFT(int n);
  void forward(cplx* x) const;
  void inverse(cplx* x) const;   // unscaled inverse; caller divides by N
};

// Column-major dense matrix helpers (m rows, n cols, leading dimension m).
// Householder QR in place: A (m x n, m >= n) -> R in the upper triangle; Q applied
// explicitly by form_q().  tau has n entries.
void householder_qr(double* A, int m, int n, std::vector<double>& tau);
// Form the thin Q (m x n) from the reflectors stored in A (below the diagonal).
void form_q(const double* A, int m, int n, const std::vector<double>& tau, double* Q);
// One-sided Jacobi SVD of A (m x n, m >= n): on return A holds U*diag(s) columns, V is
// n x n (column-major), s sorted descending with the columns permuted accordingly.
void jacobi_svd(double* A, int m, int n, double* s, double* V, double* U);
// Symmetric eigen-decomposition by cyclic Jacobi: A (n x n, column-major) -> w ascending,
// V eigenvectors in columns.
void sym_eig(double* A, int n, double* w, double* V);

// counter-based standard normal (splitmix64 + Box-Muller), deterministic per (seed, i)
double normal(uint64_t seed, uint64_t i);

}  // namespace la
}  // namespace rs
