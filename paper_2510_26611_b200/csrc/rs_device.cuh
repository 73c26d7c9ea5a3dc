// Device-side steps of the evaluation contract shared by every kernel that scores poses
// (score_kernel.cu, force_kernel.cu): one copy of each op sequence, so the kernels cannot drift
// apart (the oracle, oracle/oracle_score.c, has its own independent copy).  DESIGN.md §2:
//   O1 quaternion -> rotation (Shoemake form, s = 2 / |q|^2)
//   O3 snap of a coordinate to its cell (ties to the lower cell)
//   O4 one rank pair of the CP gather and the pairwise halving tree   PAPER.md:864-872 (A20)
//   O6 double-double accumulation (TwoProduct + TwoSum, any order)
// Every floating-point op is an explicit round-to-nearest intrinsic (the .cu files are also
// compiled with -fmad=false), in the oracle's order.
#pragma once

#include <cuda_runtime.h>

// Bounds-checked build (-DRS_DEVICE_CHECKS; tools/build_variants.py checked=-DRS_DEVICE_CHECKS):
// every shared-memory window row, local-table cell, queue slot, list entry, record, memo
// value, TMA box and output index is asserted in range (device assert: the failing
// expression, block and thread are printed and the launch fails).  The substitute for
// compute-sanitizer, which this pool does not run.
#ifdef RS_DEVICE_CHECKS
#include <cassert>
#define RS_DCHECK(x) assert(x)
#else
#define RS_DCHECK(x) ((void)0)
#endif

namespace rs {
namespace dev {

// O1: quaternion (w,x,y,z) -> R (row-major); false if |q|^2 is 0 or not finite
__device__ __forceinline__ bool quat_rot_dev(const double* q, double* R) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  const double nn = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(w, w), __dmul_rn(x, x)), __dmul_rn(y, y)),
                              __dmul_rn(z, z));
  if (!(nn > 0.0) || !isfinite(nn)) return false;
  const double s = __ddiv_rn(2.0, nn);
  const double xs = __dmul_rn(x, s), ys = __dmul_rn(y, s), zs = __dmul_rn(z, s);
  const double wx = __dmul_rn(w, xs), wy = __dmul_rn(w, ys), wz = __dmul_rn(w, zs);
  const double xx = __dmul_rn(x, xs), xy = __dmul_rn(x, ys), xz = __dmul_rn(x, zs);
  const double yy = __dmul_rn(y, ys), yz = __dmul_rn(y, zs), zz = __dmul_rn(z, zs);
  R[0] = __dsub_rn(1.0, __dadd_rn(yy, zz));
  R[1] = __dsub_rn(xy, wz);
  R[2] = __dadd_rn(xz, wy);
  R[3] = __dadd_rn(xy, wz);
  R[4] = __dsub_rn(1.0, __dadd_rn(xx, zz));
  R[5] = __dsub_rn(yz, wx);
  R[6] = __dsub_rn(xz, wy);
  R[7] = __dadd_rn(yz, wx);
  R[8] = __dsub_rn(1.0, __dadd_rn(xx, yy));
  return true;
}

// O3 cell of a valid coordinate: u = (x + b) * inv_h in [0, n(1+eps)]; i = clamp(ceil(u)-1)
__device__ __forceinline__ int snap_dev(double x, double b, double inv_h, int nm1) {
  const double u = __dmul_rn(__dadd_rn(x, b), inv_h);
  int c;
  asm("cvt.rpi.s32.f64 %0, %1;" : "=r"(c) : "d"(u));
  return min(max(c - 1, 0), nm1);
}

// O6: (hi, lo) += p exactly up to the final lo rounding (Knuth TwoSum)
__device__ __forceinline__ void dd_acc(double& hi, double& lo, double p) {
  const double s = __dadd_rn(hi, p);
  const double bb = __dsub_rn(s, hi);
  const double err = __dadd_rn(__dsub_rn(hi, __dsub_rn(s, bb)), __dsub_rn(p, bb));
  hi = s;
  lo = __dadd_rn(lo, err);
}

// O6: accumulate the exact product a*b into (hi, lo) (Dekker TwoProduct + Knuth TwoSum)
__device__ __forceinline__ void dd_add_prod(double& hi, double& lo, double a, double b) {
  const double p = __dmul_rn(a, b);
  const double e = __fma_rn(a, b, -p);
  const double s = __dadd_rn(hi, p);
  const double bb = __dsub_rn(s, hi);
  const double err = __dadd_rn(__dsub_rn(hi, __dsub_rn(s, bb)), __dsub_rn(p, bb));
  hi = s;
  lo = __dadd_rn(lo, __dadd_rn(err, e));
}

// O6: (hi, lo) += (h2, l2) exactly up to the final lo rounding (TwoSum on the high parts; its
// outputs do not depend on the operand order, so butterfly partners agree)
__device__ __forceinline__ void dd_merge(double& hi, double& lo, double h2, double l2) {
  const double s = __dadd_rn(hi, h2);
  const double bb = __dsub_rn(s, hi);
  const double e = __dadd_rn(__dsub_rn(hi, __dsub_rn(s, bb)), __dsub_rn(h2, bb));
  hi = s;
  lo = __dadd_rn(__dadd_rn(lo, l2), e);
}

// O4 one rank pair: s_c = (a0 b0) c0 + (a1 b1) c1
__device__ __forceinline__ double pair_prod(double2 a, double2 b, double2 c) {
  return __dadd_rn(__dmul_rn(__dmul_rn(a.x, b.x), c.x), __dmul_rn(__dmul_rn(a.y, b.y), c.y));
}

// O4 halving tree over NS pair sums (A20): s_c = s_c + s_{c+m}, m = NS/2 .. 1
template <int NS>
__device__ __forceinline__ double halving_tree(double* s) {
#pragma unroll
  for (int m = NS / 2; m >= 1; m /= 2) {
#pragma unroll
    for (int c = 0; c < m; ++c) s[c] = __dadd_rn(s[c], s[c + m]);
  }
  return s[0];
}

}  // namespace dev
}  // namespace rs
