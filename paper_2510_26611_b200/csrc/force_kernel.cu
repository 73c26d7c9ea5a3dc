// Forces on the rigid ligand (NEXT row N1): PAPER.md §3.3 Eq. (21) "differ_ligand"
// (finite differences of the long-range CP value on the grid) and §4
// Eqs. (24)-(25) / Lemma 4.1 (resultants on the rigid cluster).  Reading
// DESIGN.md A22; the oracle is oracle/oracle_score.c: oracle_score_forces (no shared code).
//
// One warp per pose (grid-stride), lanes over ligand atoms.  Per atom: O1-O3 as the scoring
// kernel, then four O4 values phi(i), phi(i - e_a) (a = 0, 1, 2; forward at i_a = 0) from the
// L2-resident factor rows (the shifted value reuses two of the three rows), the backward
// differences g_a = (phi(i) - phi(i - e_a)) * inv_h, F_l = -(z_l g), r_l = x'_l - t, the
// torque r_l x F_l and the radial part c r_l, c = (F_l . r_l) / |r_l|^2; per pose nine
// double-double sums (order-free, O6), reduced by xor butterflies.  Every op is an explicit
// round-to-nearest intrinsic in the oracle's order (the file is compiled with -fmad=false).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "rs_internal.h"
#include "rs_device.cuh"

namespace rs {
namespace {

using namespace dev;

constexpr int kForceThreads = 256;
#ifndef RS_FORCE_MINB
#define RS_FORCE_MINB 1          // resident blocks per SM the register budget must allow
#endif
constexpr unsigned kAll = 0xffffffffu;

// O4: rank pairs, then the pairwise halving tree (reading A20), rows from L2
template <int R>
__device__ __forceinline__ double phi_rows(const double* a, const double* b, const double* c) {
  constexpr int CH = R / 2;
  constexpr int C = CH <= 1 ? 1 : CH <= 2 ? 2 : CH <= 4 ? 4 : CH <= 8 ? 8 : 16;
  const double2* a2 = reinterpret_cast<const double2*>(a);
  const double2* b2 = reinterpret_cast<const double2*>(b);
  const double2* c2 = reinterpret_cast<const double2*>(c);
  double s[C];
#pragma unroll
  for (int j = 0; j < C; ++j) {
    s[j] = 0.0;
    if (j < CH) {
      const double2 x = __ldg(a2 + j), y = __ldg(b2 + j), z = __ldg(c2 + j);
      s[j] = __dadd_rn(__dmul_rn(__dmul_rn(x.x, y.x), z.x), __dmul_rn(__dmul_rn(x.y, y.y), z.y));
    }
  }
#pragma unroll
  for (int m = C / 2; m >= 1; m /= 2) {
#pragma unroll
    for (int j = 0; j < m; ++j) s[j] = __dadd_rn(s[j], s[j + m]);
  }
  return s[0];
}

// the same for a runtime width (odd R or widths without a compiled variant)
__device__ double phi_rows_rt(const double* a, const double* b, const double* c, int R) {
  int C = 1;
  while (2 * C < R) C *= 2;
  double st[24];
  int lg = 0;
  while ((1 << lg) < C) ++lg;
  int top = 0;
  for (int j = 0; j < C; ++j) {
    const int k = lg ? (int)(__brev((unsigned)j) >> (32 - lg)) : 0;
    double q0 = 0.0, q1 = 0.0;
    if (2 * k < R) q0 = __dmul_rn(__dmul_rn(__ldg(a + 2 * k), __ldg(b + 2 * k)), __ldg(c + 2 * k));
    if (2 * k + 1 < R)
      q1 = __dmul_rn(__dmul_rn(__ldg(a + 2 * k + 1), __ldg(b + 2 * k + 1)), __ldg(c + 2 * k + 1));
    double v = __dadd_rn(q0, q1);
    for (int t = j; t & 1; t >>= 1) v = __dadd_rn(st[--top], v);
    st[top++] = v;
  }
  return st[0];
}

// The four values phi(i), phi(i with axis 0 moved to s0), ... axis 2 -> s2 at once, chunk by
// chunk (six rows: each shifted value swaps one of the three rows), each through the same
// depth-first halving tree as phi_rows: identical arithmetic, a quarter of the live registers
// of four separate evaluations, so more warps stay resident for the L2 latency.
struct Phi4 {
  double v[4];
};

template <int C, int STRIDE, int CNT>
struct Tree4 {
  static __device__ __forceinline__ Phi4 eval(const double2* A, const double2* A2,
                                              const double2* B, const double2* B2,
                                              const double2* Cr, const double2* C2, int CH) {
    Phi4 r;
    if constexpr (CNT == 1) {
      if (C < CH) {
        const double2 a = __ldg(A + C), b = __ldg(B + C), c = __ldg(Cr + C);
        const double2 a2 = __ldg(A2 + C), b2 = __ldg(B2 + C), c2 = __ldg(C2 + C);
        const double abx = __dmul_rn(a.x, b.x), aby = __dmul_rn(a.y, b.y);
        r.v[0] = __dadd_rn(__dmul_rn(abx, c.x), __dmul_rn(aby, c.y));
        r.v[1] = __dadd_rn(__dmul_rn(__dmul_rn(a2.x, b.x), c.x), __dmul_rn(__dmul_rn(a2.y, b.y), c.y));
        r.v[2] = __dadd_rn(__dmul_rn(__dmul_rn(a.x, b2.x), c.x), __dmul_rn(__dmul_rn(a.y, b2.y), c.y));
        r.v[3] = __dadd_rn(__dmul_rn(abx, c2.x), __dmul_rn(aby, c2.y));
      } else {
        r.v[0] = r.v[1] = r.v[2] = r.v[3] = 0.0;
      }
    } else {
      const Phi4 l = Tree4<C, 2 * STRIDE, CNT / 2>::eval(A, A2, B, B2, Cr, C2, CH);
      const Phi4 h = Tree4<C + STRIDE, 2 * STRIDE, CNT / 2>::eval(A, A2, B, B2, Cr, C2, CH);
#pragma unroll
      for (int t = 0; t < 4; ++t) r.v[t] = __dadd_rn(l.v[t], h.v[t]);
    }
    return r;
  }
};

__device__ __forceinline__ double4 ld256(const double* p) {
  double4 v;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}

template <int R>
__device__ __forceinline__ Phi4 phi4_at(const ScoreArgs& a, const int* i, const int* sh) {
  constexpr int CH = R / 2;
  constexpr int C = CH <= 1 ? 1 : CH <= 2 ? 2 : CH <= 4 ? 4 : CH <= 8 ? 8 : 16;
  if constexpr (CH % 2 != 0) {
    const double2* A = reinterpret_cast<const double2*>(a.t.F[0] + (size_t)i[0] * R);
    const double2* A2 = reinterpret_cast<const double2*>(a.t.F[0] + (size_t)sh[0] * R);
    const double2* B = reinterpret_cast<const double2*>(a.t.F[1] + (size_t)i[1] * R);
    const double2* B2 = reinterpret_cast<const double2*>(a.t.F[1] + (size_t)sh[1] * R);
    const double2* Cr = reinterpret_cast<const double2*>(a.t.F[2] + (size_t)i[2] * R);
    const double2* C2 = reinterpret_cast<const double2*>(a.t.F[2] + (size_t)sh[2] * R);
    return Tree4<0, 1, C>::eval(A, A2, B, B2, Cr, C2, CH);
  } else {
    // 32-byte loads (two rank pairs per lane and request: whole L2 sectors), then the halving
    // tree level by level (same pairings as phi_rows)
    const double* A = a.t.F[0] + (size_t)i[0] * R;
    const double* A2 = a.t.F[0] + (size_t)sh[0] * R;
    const double* B = a.t.F[1] + (size_t)i[1] * R;
    const double* B2 = a.t.F[1] + (size_t)sh[1] * R;
    const double* Cr = a.t.F[2] + (size_t)i[2] * R;
    const double* C2 = a.t.F[2] + (size_t)sh[2] * R;
    double s[4][C];
#pragma unroll
    for (int j = 0; j < C; ++j) s[0][j] = s[1][j] = s[2][j] = s[3][j] = 0.0;
#pragma unroll
    for (int j = 0; j < CH / 2; ++j) {
      const double4 x = ld256(A + 4 * j), x2 = ld256(A2 + 4 * j), y = ld256(B + 4 * j);
      const double4 y2 = ld256(B2 + 4 * j), z = ld256(Cr + 4 * j), z2 = ld256(C2 + 4 * j);
      const double p0 = __dmul_rn(x.x, y.x), p1 = __dmul_rn(x.y, y.y);
      const double p2 = __dmul_rn(x.z, y.z), p3 = __dmul_rn(x.w, y.w);
      s[0][2 * j] = __dadd_rn(__dmul_rn(p0, z.x), __dmul_rn(p1, z.y));
      s[0][2 * j + 1] = __dadd_rn(__dmul_rn(p2, z.z), __dmul_rn(p3, z.w));
      s[1][2 * j] = __dadd_rn(__dmul_rn(__dmul_rn(x2.x, y.x), z.x), __dmul_rn(__dmul_rn(x2.y, y.y), z.y));
      s[1][2 * j + 1] = __dadd_rn(__dmul_rn(__dmul_rn(x2.z, y.z), z.z), __dmul_rn(__dmul_rn(x2.w, y.w), z.w));
      s[2][2 * j] = __dadd_rn(__dmul_rn(__dmul_rn(x.x, y2.x), z.x), __dmul_rn(__dmul_rn(x.y, y2.y), z.y));
      s[2][2 * j + 1] = __dadd_rn(__dmul_rn(__dmul_rn(x.z, y2.z), z.z), __dmul_rn(__dmul_rn(x.w, y2.w), z.w));
      s[3][2 * j] = __dadd_rn(__dmul_rn(p0, z2.x), __dmul_rn(p1, z2.y));
      s[3][2 * j + 1] = __dadd_rn(__dmul_rn(p2, z2.z), __dmul_rn(p3, z2.w));
    }
#pragma unroll
    for (int m = C / 2; m >= 1; m /= 2) {
#pragma unroll
      for (int j = 0; j < m; ++j) {
#pragma unroll
        for (int t = 0; t < 4; ++t) s[t][j] = __dadd_rn(s[t][j], s[t][j + m]);
      }
    }
    Phi4 r;
#pragma unroll
    for (int t = 0; t < 4; ++t) r.v[t] = s[t][0];
    return r;
  }
}

template <int R>
__device__ __forceinline__ double phi_at(const ScoreArgs& a, int i0, int i1, int i2) {
  const int r = R > 0 ? R : a.R;
  const double* f0 = a.t.F[0] + (size_t)i0 * r;
  const double* f1 = a.t.F[1] + (size_t)i1 * r;
  const double* f2 = a.t.F[2] + (size_t)i2 * r;
  if constexpr (R > 0 && (R % 2) == 0) return phi_rows<R>(f0, f1, f2);
  else return phi_rows_rt(f0, f1, f2, r);
}

template <int R>
__global__ void __launch_bounds__(kForceThreads, RS_FORCE_MINB) force_kernel(const ScoreArgs a,
                                                                             double* out) {
  const int lane = threadIdx.x & 31;
  // each block owns a contiguous pose range (its warps interleave inside it), so consecutive
  // poses of one block share translations and their factor rows stay in the SM's L1
  const int64_t p_lo = a.P * (int64_t)blockIdx.x / gridDim.x;
  const int64_t p_hi = a.P * (int64_t)(blockIdx.x + 1) / gridDim.x;
  const int64_t warp0 = p_lo + (threadIdx.x >> 5);
  constexpr int64_t nwarps = kForceThreads / 32;
  const int nm1 = a.n - 1;
  for (int64_t p = warp0; p < p_hi; p += nwarps) {
    const double* pq = a.poses + 7 * p;
    double q[7];
#pragma unroll
    for (int i = 0; i < 7; ++i) q[i] = __ldg(pq + i);
    double Rm[9];
    bool ok = quat_rot_dev(q, Rm);
    double hi[9], lo[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) hi[j] = lo[j] = 0.0;
    for (int l0 = 0; ok && l0 < a.L; l0 += 32) {
      const int l = l0 + lane;
      bool bad = false;
      if (l < a.L) {
        const double y0 = __ldg(a.yl + 3 * (int64_t)l), y1 = __ldg(a.yl + 3 * (int64_t)l + 1),
                     y2 = __ldg(a.yl + 3 * (int64_t)l + 2), z = __ldg(a.zl + l);
        double xp[3];
#pragma unroll
        for (int r = 0; r < 3; ++r)
          xp[r] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(Rm[3 * r], y0), __dmul_rn(Rm[3 * r + 1], y1)),
                                      __dmul_rn(Rm[3 * r + 2], y2)),
                            q[4 + r]);
        if (!(fabs(xp[0]) <= a.b && fabs(xp[1]) <= a.b && fabs(xp[2]) <= a.b)) {
          bad = true;
        } else {
          int i[3];
#pragma unroll
          for (int r = 0; r < 3; ++r) i[r] = snap_dev(xp[r], a.b, a.inv_h, nm1);
          // backward neighbours (forward at the lower edge)
          int sh[3];
#pragma unroll
          for (int ax = 0; ax < 3; ++ax) sh[ax] = i[ax] > 0 ? i[ax] - 1 : i[ax] + 1;
          double phi, pn[3];
          if constexpr (R > 0 && (R % 2) == 0) {
            const Phi4 f = phi4_at<R>(a, i, sh);
            phi = f.v[0];
            pn[0] = f.v[1];
            pn[1] = f.v[2];
            pn[2] = f.v[3];
          } else {
            phi = phi_at<R>(a, i[0], i[1], i[2]);
            pn[0] = phi_at<R>(a, sh[0], i[1], i[2]);
            pn[1] = phi_at<R>(a, i[0], sh[1], i[2]);
            pn[2] = phi_at<R>(a, i[0], i[1], sh[2]);
          }
          double F[3], rv[3];
#pragma unroll
          for (int ax = 0; ax < 3; ++ax) {
            const double g = i[ax] > 0 ? __dmul_rn(__dsub_rn(phi, pn[ax]), a.inv_h)
                                       : __dmul_rn(__dsub_rn(pn[ax], phi), a.inv_h);
            F[ax] = -__dmul_rn(z, g);
            rv[ax] = __dsub_rn(xp[ax], q[4 + ax]);
          }
          const double tau0 = __dsub_rn(__dmul_rn(rv[1], F[2]), __dmul_rn(rv[2], F[1]));
          const double tau1 = __dsub_rn(__dmul_rn(rv[2], F[0]), __dmul_rn(rv[0], F[2]));
          const double tau2 = __dsub_rn(__dmul_rn(rv[0], F[1]), __dmul_rn(rv[1], F[0]));
          const double rr = __dadd_rn(__dadd_rn(__dmul_rn(rv[0], rv[0]), __dmul_rn(rv[1], rv[1])),
                                      __dmul_rn(rv[2], rv[2]));
          double c = 0.0;
          if (rr > 0.0)
            c = __ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn(F[0], rv[0]), __dmul_rn(F[1], rv[1])),
                                    __dmul_rn(F[2], rv[2])),
                          rr);
#pragma unroll
          for (int ax = 0; ax < 3; ++ax) dd_acc(hi[ax], lo[ax], F[ax]);
          dd_acc(hi[3], lo[3], tau0);
          dd_acc(hi[4], lo[4], tau1);
          dd_acc(hi[5], lo[5], tau2);
#pragma unroll
          for (int ax = 0; ax < 3; ++ax) dd_acc(hi[6 + ax], lo[6 + ax], __dmul_rn(c, rv[ax]));
        }
      }
      if (__any_sync(kAll, bad)) ok = false;
    }
    double res[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
        dd_merge(hi[j], lo[j], __shfl_xor_sync(kAll, hi[j], off), __shfl_xor_sync(kAll, lo[j], off));
      res[j] = ok ? __dadd_rn(hi[j], lo[j]) : NAN;
    }
    // lanes 0..8 write one component each (coalesced 72-byte row)
    double mine = res[0];
#pragma unroll
    for (int j = 1; j < 9; ++j)
      if (lane == j) mine = res[j];
    if (lane < 9) out[9 * p + lane] = mine;
    if (!ok && lane == 0 && a.invalid) atomicAdd(a.invalid, 1ull);
  }
}

// ---- windowed variant (widths with a power-of-two number of rank pairs: R = 4, 8, 16, 32) ----
// One 512-thread block per SM owns a contiguous pose range and walks it in tiles of 32 poses
// (two per warp; measured at C3: 1 per warp 4.41 ms, 2: 4.08, 4: 4.10, 8: 4.54).  The rows a tile can touch (t +- (r_max + 2h) per axis, plus one row for the
// backward neighbour) are staged into shared memory when they are not already there (C3:
// consecutive poses share their translation, so a block restages a few times per launch), and
// a tile that straddles two translations is staged around its last pose; the six rows of each
// atom are read from shared memory, lane l taking in slot c the rank pair
// c ^ (l & 7) (conflict-free 16-byte loads; the halving tree pairs slot c with c ^ m, so the
// XOR relabelling leaves every sum bitwise unchanged, reading A20).  An atom whose rows fall
// outside the window reads them from L2 as in force_kernel.  Same arithmetic, same output.
constexpr int kWinThreads = 512;
constexpr int kWinWarps = kWinThreads / 32;
#ifndef RS_FWIN_PPW
#define RS_FWIN_PPW 2            // poses per warp per tile (one window decision per tile)
#endif
constexpr int kWinTile = kWinWarps * RS_FWIN_PPW;

// depth-first evaluation of the halving tree (as Tree4): slot C of the tree reads rank pair
// C ^ k of each row
template <int C, int STRIDE, int CNT>
struct TreeW {
  static __device__ __forceinline__ Phi4 eval(const double2* A, const double2* A2,
                                              const double2* B, const double2* B2,
                                              const double2* Cr, const double2* C2, int k) {
    Phi4 r;
    if constexpr (CNT == 1) {
      const int ch = C ^ k;
      const double2 x = A[ch], x2 = A2[ch], y = B[ch], y2 = B2[ch], z = Cr[ch], z2 = C2[ch];
      const double p0 = __dmul_rn(x.x, y.x), p1 = __dmul_rn(x.y, y.y);
      r.v[0] = __dadd_rn(__dmul_rn(p0, z.x), __dmul_rn(p1, z.y));
      r.v[1] = __dadd_rn(__dmul_rn(__dmul_rn(x2.x, y.x), z.x), __dmul_rn(__dmul_rn(x2.y, y.y), z.y));
      r.v[2] = __dadd_rn(__dmul_rn(__dmul_rn(x.x, y2.x), z.x), __dmul_rn(__dmul_rn(x.y, y2.y), z.y));
      r.v[3] = __dadd_rn(__dmul_rn(p0, z2.x), __dmul_rn(p1, z2.y));
    } else {
      const Phi4 l = TreeW<C, 2 * STRIDE, CNT / 2>::eval(A, A2, B, B2, Cr, C2, k);
      const Phi4 h = TreeW<C + STRIDE, 2 * STRIDE, CNT / 2>::eval(A, A2, B, B2, Cr, C2, k);
#pragma unroll
      for (int t = 0; t < 4; ++t) r.v[t] = __dadd_rn(l.v[t], h.v[t]);
    }
    return r;
  }
};

template <int R>
__device__ __forceinline__ Phi4 phi4_win(const double2* W0, const double2* W1, const double2* W2,
                                         const int* org, const int* i, const int* sh, int lane) {
  constexpr int CH = R / 2;
  const double2* A = W0 + (size_t)(i[0] - org[0]) * CH;
  const double2* A2 = W0 + (size_t)(sh[0] - org[0]) * CH;
  const double2* B = W1 + (size_t)(i[1] - org[1]) * CH;
  const double2* B2 = W1 + (size_t)(sh[1] - org[1]) * CH;
  const double2* Cr = W2 + (size_t)(i[2] - org[2]) * CH;
  const double2* C2 = W2 + (size_t)(sh[2] - org[2]) * CH;
  return TreeW<0, 1, CH>::eval(A, A2, B, B2, Cr, C2, lane & (CH < 8 ? CH - 1 : 7));
}

template <int R>
__global__ void __launch_bounds__(kWinThreads, 1) force_window_kernel(const ScoreArgs a,
                                                                      double* out, int cap) {
  constexpr int CH = R / 2;
  extern __shared__ __align__(16) double2 wsm[];
  double2* W[3] = {wsm, wsm + (size_t)cap * CH, wsm + (size_t)2 * cap * CH};
  __shared__ int s_org[3], s_len[3], s_tlo[3], s_thi[3], s_use;
  __shared__ double s_rmax;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nm1 = a.n - 1;
  // ligand radius about the body origin (bounds only; correctness never depends on it)
  if (threadIdx.x == 0) s_rmax = 0.0;
  __syncthreads();
  {
    double m = 0.0;
    for (int64_t l = threadIdx.x; l < a.L; l += kWinThreads) {
      const double y0 = a.yl[3 * l], y1 = a.yl[3 * l + 1], y2 = a.yl[3 * l + 2];
      m = fmax(m, sqrt(y0 * y0 + y1 * y1 + y2 * y2));
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(kAll, m, off));
    if (lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(&s_rmax),
                             (unsigned long long)__double_as_longlong(m));
  }
  if (threadIdx.x < 3) { s_org[threadIdx.x] = 0; s_len[threadIdx.x] = 0; }
  __syncthreads();
  const double reach = s_rmax * 1.000001 + 2.0 * a.h;
  const int64_t p_lo = a.P * (int64_t)blockIdx.x / gridDim.x;
  const int64_t p_hi = a.P * (int64_t)(blockIdx.x + 1) / gridDim.x;
  for (int64_t t0 = p_lo; t0 < p_hi; t0 += kWinTile) {
    // tile bounds: block min/max of the per-pose row ranges (warp 0, kWinTile / 32 poses per lane)
    if (warp == 0) {
      int lo[3] = {a.n, a.n, a.n}, hi[3] = {-1, -1, -1};
      for (int64_t p = t0 + lane; p < min(t0 + kWinTile, p_hi); p += 32) {
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
          const double t = a.poses[7 * p + 4 + ax];
          if (isfinite(t)) {
            const double ul = (t - reach + a.b) * a.inv_h, uh = (t + reach + a.b) * a.inv_h;
            lo[ax] = min(lo[ax], (int)fmax(0.0, fmin((double)nm1, floor(ul) - 2.0)));
            hi[ax] = max(hi[ax], (int)fmax(0.0, fmin((double)nm1, ceil(uh) + 2.0)));
          }
        }
      }
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          lo[ax] = min(lo[ax], __shfl_xor_sync(kAll, lo[ax], off));
          hi[ax] = max(hi[ax], __shfl_xor_sync(kAll, hi[ax], off));
        }
      }
      if (lane == 0) {
        bool inside = true, fits = true;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
          s_tlo[ax] = lo[ax];
          s_thi[ax] = hi[ax];
          if (hi[ax] < lo[ax]) continue;                       // no finite pose: nothing to stage
          inside = inside && lo[ax] >= s_org[ax] && hi[ax] < s_org[ax] + s_len[ax];
          fits = fits && hi[ax] - lo[ax] + 1 <= cap;
        }
        int use = inside ? 0 : 1;                              // 0 keep, 1 restage, 2 no window
        if (!inside && !fits) {
          // the tile straddles two translations: stage around the tile's last pose (the next
          // tiles continue there); the other poses' atoms read L2 where they miss the window
          const int64_t pl = min(t0 + kWinTile, p_hi) - 1;
          bool ok_last = true;
#pragma unroll
          for (int ax = 0; ax < 3; ++ax) {
            const double t = a.poses[7 * pl + 4 + ax];
            if (!isfinite(t)) { ok_last = false; continue; }
            const double ul = (t - reach + a.b) * a.inv_h, uh = (t + reach + a.b) * a.inv_h;
            const int l = (int)fmax(0.0, fmin((double)nm1, floor(ul) - 2.0));
            const int h = (int)fmax(0.0, fmin((double)nm1, ceil(uh) + 2.0));
            ok_last = ok_last && h - l + 1 <= cap;
            s_tlo[ax] = l;
          }
          if (!ok_last) use = 2;
        }
        s_use = use;
      }
    }
    __syncthreads();
    const int use = s_use;
    if (use == 1) {
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        const int org = s_tlo[ax];
        const int len = min(cap, a.n - org);
        const double2* src = reinterpret_cast<const double2*>(a.t.F[ax] + (size_t)org * R);
        for (int j = threadIdx.x; j < len * CH; j += kWinThreads) W[ax][j] = __ldg(src + j);
      }
      __syncthreads();
      if (threadIdx.x < 3) {
        s_org[threadIdx.x] = s_tlo[threadIdx.x];
        s_len[threadIdx.x] = min(cap, a.n - s_tlo[threadIdx.x]);
      }
      __syncthreads();
    }
    int org[3], len[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) { org[ax] = s_org[ax]; len[ax] = use == 2 ? 0 : s_len[ax]; }
    for (int64_t p = t0 + warp; p < min(t0 + kWinTile, p_hi); p += kWinWarps) {
      const double* pq = a.poses + 7 * p;
      double q[7];
#pragma unroll
      for (int i = 0; i < 7; ++i) q[i] = __ldg(pq + i);
      double Rm[9];
      bool ok = quat_rot_dev(q, Rm);
      double hi[9], lo[9];
#pragma unroll
      for (int j = 0; j < 9; ++j) hi[j] = lo[j] = 0.0;
      for (int l0 = 0; ok && l0 < a.L; l0 += 32) {
        const int l = l0 + lane;
        bool bad = false;
        if (l < a.L) {
          const double y0 = __ldg(a.yl + 3 * (int64_t)l), y1 = __ldg(a.yl + 3 * (int64_t)l + 1),
                       y2 = __ldg(a.yl + 3 * (int64_t)l + 2), z = __ldg(a.zl + l);
          double xp[3];
#pragma unroll
          for (int r = 0; r < 3; ++r)
            xp[r] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(Rm[3 * r], y0), __dmul_rn(Rm[3 * r + 1], y1)),
                                        __dmul_rn(Rm[3 * r + 2], y2)),
                              q[4 + r]);
          if (!(fabs(xp[0]) <= a.b && fabs(xp[1]) <= a.b && fabs(xp[2]) <= a.b)) {
            bad = true;
          } else {
            int i[3], sh[3];
            bool inwin = true;
#pragma unroll
            for (int r = 0; r < 3; ++r) {
              i[r] = snap_dev(xp[r], a.b, a.inv_h, nm1);
              sh[r] = i[r] > 0 ? i[r] - 1 : i[r] + 1;
              inwin = inwin && min(i[r], sh[r]) >= org[r] && max(i[r], sh[r]) < org[r] + len[r];
            }
            Phi4 f;
            RS_DCHECK(i[0] >= 0 && i[0] < a.n && i[1] >= 0 && i[1] < a.n && i[2] >= 0 && i[2] < a.n &&
                      sh[0] >= 0 && sh[0] < a.n && sh[1] >= 0 && sh[1] < a.n && sh[2] >= 0 && sh[2] < a.n);
            RS_DCHECK(!inwin || (len[0] <= cap && len[1] <= cap && len[2] <= cap));
            if (inwin) {
              f = phi4_win<R>(W[0], W[1], W[2], org, i, sh, lane);
            } else {      // rows outside the window: depth-first tree on 16-byte L2 loads
              f = Tree4<0, 1, CH>::eval(
                  reinterpret_cast<const double2*>(a.t.F[0] + (size_t)i[0] * R),
                  reinterpret_cast<const double2*>(a.t.F[0] + (size_t)sh[0] * R),
                  reinterpret_cast<const double2*>(a.t.F[1] + (size_t)i[1] * R),
                  reinterpret_cast<const double2*>(a.t.F[1] + (size_t)sh[1] * R),
                  reinterpret_cast<const double2*>(a.t.F[2] + (size_t)i[2] * R),
                  reinterpret_cast<const double2*>(a.t.F[2] + (size_t)sh[2] * R), CH);
            }
            const double phi = f.v[0];
            const double pn[3] = {f.v[1], f.v[2], f.v[3]};
            double F[3], rv[3];
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
              const double g = i[ax] > 0 ? __dmul_rn(__dsub_rn(phi, pn[ax]), a.inv_h)
                                         : __dmul_rn(__dsub_rn(pn[ax], phi), a.inv_h);
              F[ax] = -__dmul_rn(z, g);
              rv[ax] = __dsub_rn(xp[ax], q[4 + ax]);
            }
            const double tau0 = __dsub_rn(__dmul_rn(rv[1], F[2]), __dmul_rn(rv[2], F[1]));
            const double tau1 = __dsub_rn(__dmul_rn(rv[2], F[0]), __dmul_rn(rv[0], F[2]));
            const double tau2 = __dsub_rn(__dmul_rn(rv[0], F[1]), __dmul_rn(rv[1], F[0]));
            const double rr = __dadd_rn(__dadd_rn(__dmul_rn(rv[0], rv[0]), __dmul_rn(rv[1], rv[1])),
                                        __dmul_rn(rv[2], rv[2]));
            double c = 0.0;
            if (rr > 0.0)
              c = __ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn(F[0], rv[0]), __dmul_rn(F[1], rv[1])),
                                      __dmul_rn(F[2], rv[2])),
                            rr);
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) dd_acc(hi[ax], lo[ax], F[ax]);
            dd_acc(hi[3], lo[3], tau0);
            dd_acc(hi[4], lo[4], tau1);
            dd_acc(hi[5], lo[5], tau2);
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) dd_acc(hi[6 + ax], lo[6 + ax], __dmul_rn(c, rv[ax]));
          }
        }
        if (__any_sync(kAll, bad)) ok = false;
      }
      double res[9];
#pragma unroll
      for (int j = 0; j < 9; ++j) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
          dd_merge(hi[j], lo[j], __shfl_xor_sync(kAll, hi[j], off), __shfl_xor_sync(kAll, lo[j], off));
        res[j] = ok ? __dadd_rn(hi[j], lo[j]) : NAN;
      }
      double mine = res[0];
#pragma unroll
      for (int j = 1; j < 9; ++j)
        if (lane == j) mine = res[j];
      RS_DCHECK(p >= 0 && p < a.P);
      if (lane < 9) out[9 * p + lane] = mine;
      if (!ok && lane == 0 && a.invalid) atomicAdd(a.invalid, 1ull);
    }
    __syncthreads();                   // the window may be restaged by the next tile
  }
}

template <int R>
int launch_forces_window(const ScoreArgs& a, double* out, cudaStream_t st, int sms, int device) {
  int smem_max = 0;
  cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  const int row_bytes = R * 8;
  const int cap = std::min(a.n, (smem_max - 1024) / (3 * row_bytes));
  const size_t bytes = (size_t)3 * cap * row_bytes;
  const cudaError_t ae = cudaFuncSetAttribute(force_window_kernel<R>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (ae != cudaSuccess) return (int)ae;
  const int64_t blocks = std::min<int64_t>((a.P + kWinTile - 1) / kWinTile, sms);
  force_window_kernel<R><<<(int)std::max<int64_t>(blocks, 1), kWinThreads, bytes, st>>>(a, out, cap);
  return (int)cudaGetLastError();
}

template <int R>
int launch_forces_t(const ScoreArgs& a, double* out, cudaStream_t st, int sms) {
  const int64_t warps_needed = a.P;
  const int64_t blocks = std::min<int64_t>((warps_needed + 7) / 8, (int64_t)sms * 8 * RS_FORCE_MINB);
  force_kernel<R><<<(int)std::max<int64_t>(blocks, 1), kForceThreads, 0, st>>>(a, out);
  return (int)cudaGetLastError();
}

}  // namespace

int launch_forces(const ScoreArgs& a, double* out, void* stream, int device) {
  if (a.P <= 0) return 0;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaStream_t st = (cudaStream_t)stream;
#ifndef RS_FORCE_NOWIN
  switch (a.R) {
    case 4: return launch_forces_window<4>(a, out, st, sms, device);
    case 8: return launch_forces_window<8>(a, out, st, sms, device);
    case 16: return launch_forces_window<16>(a, out, st, sms, device);
    case 32: return launch_forces_window<32>(a, out, st, sms, device);
    default: break;
  }
#endif
  switch (a.R) {
    case 4: return launch_forces_t<4>(a, out, st, sms);
    case 8: return launch_forces_t<8>(a, out, st, sms);
    case 12: return launch_forces_t<12>(a, out, st, sms);
    case 16: return launch_forces_t<16>(a, out, st, sms);
    case 24: return launch_forces_t<24>(a, out, st, sms);
    case 32: return launch_forces_t<32>(a, out, st, sms);
    default: return launch_forces_t<0>(a, out, st, sms);
  }
}

}  // namespace rs
