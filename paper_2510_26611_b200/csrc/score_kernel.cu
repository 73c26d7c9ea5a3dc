// Fused sm_100a pose-scoring kernel: Algorithm PLIE with Lemma 3.2 /
// Eq. (18), the RS entry formula and the vdW constraint
// of Eq. (22).  Rows H1-H8 of SURVEY.md §8(a), in one pass:
//   H1 quaternion -> rotation      H2 x' = R y + t           H3 snap to the cell grid
//   H4 long-range CP gather + rank chain (rows of F_0, F_1, F_2 from a shared-memory window
//      or from L2)                  H5 short-range replicas of nearby protein atoms
//   H6 vdW min distance over the same cell-list candidates
//   H7 warp double-double reduction H8 one energy + one min distance per pose
//
// Arithmetic contract (mirrored by oracle/oracle_score.c):
// every floating-point op of H1-H5 and H7 is an explicit round-to-nearest intrinsic (no FMA
// contraction; the file is also compiled with -fmad=false), in the same order as the oracle:
//   q_k = (F0[i0][k] * F1[i1][k]) * F2[i2][k]; rank pairs s_c = q_2c + q_2c+1 summed by a
//   pairwise halving tree (reading A20)
// Per-pose sums are double-double (Dekker TwoProduct + Knuth TwoSum), so the order in which
// lanes accumulate and the reduction tree are free.
//
// Layout of the shared-memory window (design notes): a CTA scores a tile
// of poses whose atoms fall inside per-axis row ranges [lo_a, hi_a]; those rows of the three
// factor matrices are staged once per tile (reused across tiles when contained) as 16-byte
// chunks, padded or replicated to whole 128-byte bank lines.  Lane l of a warp reads the
// chunks of its own row in the rotated order (c + (l & 7)) mod CHP, so the 8 lanes of every
// quarter-warp hit 8 distinct bank groups whatever rows they gather (conflict-free LDS.128);
// the halving tree over rank pairs is invariant under that rotation, so no rotate-back is needed.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "rs_internal.h"

namespace rs {
namespace {

#ifndef RS_THREADS
#define RS_THREADS 640
#endif
constexpr int kThreads = RS_THREADS;
constexpr int kWarps = kThreads / 32;
constexpr int kTile = 8 * kWarps;        // poses per tile (upper bound)
constexpr int kLigSmem = 256;            // ligand atoms staged in shared memory
constexpr unsigned kFull = 0xffffffffu;

template <int R>
struct Geo {
  static constexpr int CH = R / 2;                                 // 16-byte chunks of a row
  static constexpr bool REP = (CH == 1 || CH == 2 || CH == 4);      // replicate to 128 B
  static constexpr int CHP = REP ? 8 : ((CH + 7) / 8) * 8;         // physical chunks per row
  static constexpr int NS = REP ? CH : CHP;                        // loads per row and lane
};

__device__ __forceinline__ double2 ldg2(const double2* p) { return __ldg(p); }

template <bool SMEM>
__device__ __forceinline__ double2 ld2(const double2* p) {
  if constexpr (SMEM) return *p;
  else return __ldg(p);
}

// O3: cell of coordinate x; -1 outside [-b, b]
__device__ __forceinline__ int snap_dev(double x, double b, double inv_h, int n) {
  if (!(x >= -b && x <= b)) return -1;
  const double u = __dmul_rn(__dadd_rn(x, b), inv_h);
  double c = __dsub_rn(ceil(u), 1.0);
  c = fmax(c, 0.0);
  c = fmin(c, (double)(n - 1));
  return (int)c;
}

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

// O6 accumulate the exact product a*b into (hi, lo)
__device__ __forceinline__ void dd_add_prod(double& hi, double& lo, double a, double b) {
  const double p = __dmul_rn(a, b);
  const double e = __fma_rn(a, b, -p);
  const double s = __dadd_rn(hi, p);
  const double bb = __dsub_rn(s, hi);
  const double err = __dadd_rn(__dsub_rn(hi, __dsub_rn(s, bb)), __dsub_rn(p, bb));
  hi = s;
  lo = __dadd_rn(lo, __dadd_rn(err, e));
}

// O4 with compile-time R, rows given as 16-byte chunk pointers (smem window or global rows)
template <int R, bool SMEM>
__device__ __forceinline__ double long_phi(const double2* r0, const double2* r1, const double2* r2,
                                           int rho) {
  using G = Geo<R>;
  double q[2 * G::NS];
#pragma unroll
  for (int c = 0; c < G::NS; ++c) {
    const int ph = (c + rho) & (G::CHP - 1);
    int src;
    bool valid;
    if constexpr (G::REP) {
      src = SMEM ? ph : (ph & (G::CH - 1));
      valid = true;
    } else {
      src = ph;
      valid = ph < G::CH;
    }
    double2 a = make_double2(0.0, 0.0), b = a, cc = a;
    if (valid) {
      a = ld2<SMEM>(r0 + src);
      b = ld2<SMEM>(r1 + src);
      cc = ld2<SMEM>(r2 + src);
    }
    q[2 * c] = __dmul_rn(__dmul_rn(a.x, b.x), cc.x);
    q[2 * c + 1] = __dmul_rn(__dmul_rn(a.y, b.y), cc.y);
  }
  // O4 (A20): s_c = q_2c + q_2c+1, then the pairwise halving tree
  // s_c = s_c + s_{c+m}, m = NS/2 .. 1.  Slot c holds pair (c + rot) mod NS; the tree pairs
  // c with c + m (mod NS) at every level, so it is bitwise invariant under that rotation and
  // the slots are summed as they were loaded.
  double s[G::NS];
#pragma unroll
  for (int c = 0; c < G::NS; ++c) s[c] = __dadd_rn(q[2 * c], q[2 * c + 1]);
#pragma unroll
  for (int m = G::NS / 2; m >= 1; m /= 2) {
#pragma unroll
    for (int c = 0; c < m; ++c) s[c] = __dadd_rn(s[c], s[c + m]);
  }
  return s[0];
}

// O4 with a runtime R (generic widths, e.g. tolerance-mode builds): rows from L2, the same
// pairwise halving tree over rank pairs.  The tree is walked depth-first: its leaves in order
// are the pairs c = bitrev(j), j = 0..C-1, merged with a binary-counter stack (depth log2 C).
__device__ __forceinline__ double long_phi_rt(const double* r0, const double* r1, const double* r2,
                                              int R) {
  int lg = 0;
  while ((2 << lg) < R) ++lg;            // C = 2^lg pairs
  const int C = 1 << lg;
  double st[24];
  int top = 0;
  for (int j = 0; j < C; ++j) {
    const int c = lg ? (int)(__brev((unsigned)j) >> (32 - lg)) : 0;
    double q0 = 0.0, q1 = 0.0;
    if (2 * c < R) q0 = __dmul_rn(__dmul_rn(__ldg(r0 + 2 * c), __ldg(r1 + 2 * c)), __ldg(r2 + 2 * c));
    if (2 * c + 1 < R)
      q1 = __dmul_rn(__dmul_rn(__ldg(r0 + 2 * c + 1), __ldg(r1 + 2 * c + 1)), __ldg(r2 + 2 * c + 1));
    double v = __dadd_rn(q0, q1);
    for (int t = j; t & 1; t >>= 1) v = __dadd_rn(st[--top], v);
    st[top++] = v;
  }
  return st[0];
}

struct Window {
  int lo[3], hi[3], base[3];   // staged rows [lo, hi] per axis, first smem row of each axis
};

// A tile's poses, decoded once by one thread each (H1): rotation, translation, validity.
struct __align__(16) PoseStage {
  double R[kTile][9];
  double t[kTile][3];
  int ok[kTile];
};

// Per-warp staging of the 32 atoms of one pass for the flattened candidate-pair rounds.
struct __align__(16) PairStage {
  double x[3][32];   // transformed coordinates x'
  double z[32];      // charges
  int4 cell[32];     // i0, i1, i2, list begin
  int off[32];       // exclusive prefix of the candidate counts
  int map[64];       // two rounds: candidate slot where an atom's segment starts -> atom lane
};

// L2 path of O4 for compile-time R, kept out of line (it is the rare path in window mode)
template <int RT>
__device__ __noinline__ double long_phi_global(const double* F0, const double* F1, const double* F2,
                                               int i0, int i1, int i2, int rho) {
  return long_phi<RT, false>((const double2*)(F0 + (size_t)i0 * RT),
                             (const double2*)(F1 + (size_t)i1 * RT),
                             (const double2*)(F2 + (size_t)i2 * RT), rho);
}

// O5 value s(D): from the dense memo (filled by the same chain) or the chain itself
__device__ __forceinline__ double short_value(const ScoreArgs& a, int e0, int e1, int e2) {
  if (a.t.short_memo) {
    const int d = a.n_sigma + 1;
    const int u0 = e0 < 0 ? -e0 : e0, u1 = e1 < 0 ? -e1 : e1, u2 = e2 < 0 ? -e2 : e2;
    return __ldg(a.t.short_memo + ((size_t)u0 * d + u1) * d + u2);
  }
  const double* s0 = a.t.S[0] + (size_t)(e0 + a.n_sigma) * a.Rs;
  const double* s1 = a.t.S[1] + (size_t)(e1 + a.n_sigma) * a.Rs;
  const double* s2 = a.t.S[2] + (size_t)(e2 + a.n_sigma) * a.Rs;
  double s = 0.0;
  for (int k = 0; k < a.Rs; ++k)
    s = __dadd_rn(s, __dmul_rn(__dmul_rn(__ldg(s0 + k), __ldg(s1 + k)), __ldg(s2 + k)));
  return s;
}

// One candidate pair (atom `ow` of the pass, list entry j): O7 distance and O5 replica term.
__device__ __forceinline__ void pair_term(const ScoreArgs& a, const PairStage& ps, int ow,
                                          int4 oc, short4 mc, double2 xy, double2 zq,
                                          int64_t ns2, double& hi, double& lo, double& best) {
  const int e0 = oc.x - mc.x, e1 = oc.y - mc.y, e2 = oc.z - mc.z;
  const int64_t dd = (int64_t)e0 * e0 + (int64_t)e1 * e1 + (int64_t)e2 * e2;
  if (dd < a.vdw_cells2) {
    const double dx0 = __dsub_rn(ps.x[0][ow], xy.x);
    const double dx1 = __dsub_rn(ps.x[1][ow], xy.y);
    const double dx2 = __dsub_rn(ps.x[2][ow], zq.x);
    const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx0, dx0), __dmul_rn(dx1, dx1)), __dmul_rn(dx2, dx2));
    best = fmin(best, d2);
  }
  if (dd <= ns2) {
    const double sv = short_value(a, e0, e1, e2);
    dd_add_prod(hi, lo, ps.z[ow], __dmul_rn(zq.y, sv));
  }
}

// Score one pose with one warp.  RT > 0: compile-time width with an optional smem window.
template <int RT>
__device__ __forceinline__ void score_pose(const ScoreArgs& a, int64_t p, const double* Rm,
                                           const double* tv, bool ok, bool use_win,
                                           const Window& W, const double2* win,
                                           const double4* s_lig, bool lig_smem, int lane,
                                           PairStage& ps) {
  double hi = 0.0, lo = 0.0, best = INFINITY;
  bool bad = !ok;
  const int rho = lane & 7;
  const int64_t ns2 = (int64_t)a.n_sigma * a.n_sigma;
  const int npass = ok ? (int)((a.L + 31) / 32) : 0;
  const double2* nrec = (const double2*)a.t.nb_rec;
  const short4* ncell = reinterpret_cast<const short4*>(a.t.nb_cell);
  for (int pass = 0; pass < npass; ++pass) {
    const int64_t l = (int64_t)pass * 32 + lane;
    int cnt = 0, beg = 0, i0 = 0, i1 = 0, i2 = 0;
    double xp[3] = {0.0, 0.0, 0.0}, z = 0.0;
    if (l < a.L) {
      double y0, y1, y2;
      if (lig_smem) {
        const double4 v = s_lig[l];
        y0 = v.x; y1 = v.y; y2 = v.z; z = v.w;
      } else {
        y0 = __ldg(a.yl + 3 * l);
        y1 = __ldg(a.yl + 3 * l + 1);
        y2 = __ldg(a.yl + 3 * l + 2);
        z = __ldg(a.zl + l);
      }
      // H2 (O2)
#pragma unroll
      for (int r = 0; r < 3; ++r)
        xp[r] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(Rm[3 * r], y0), __dmul_rn(Rm[3 * r + 1], y1)),
                                    __dmul_rn(Rm[3 * r + 2], y2)),
                          tv[r]);
      // H3 (O3)
      i0 = snap_dev(xp[0], a.b, a.inv_h, a.n);
      i1 = snap_dev(xp[1], a.b, a.inv_h, a.n);
      i2 = snap_dev(xp[2], a.b, a.inv_h, a.n);
      if ((i0 | i1 | i2) < 0) {
        bad = true;
      } else {
#if !(defined(RS_EXPERIMENT) && (RS_EXPERIMENT & 1))
        // candidate range of the coarse cell containing i (cell lists cover every protein atom
        // within max(D_cap, (n_sigma + sqrt 3) h) of any point of the cell); loads issued
        // before H4 so their latency hides behind the gathers
        const int cx = (i0 >> a.nb_shift) - a.nb_lo[0];
        const int cy = (i1 >> a.nb_shift) - a.nb_lo[1];
        const int cz = (i2 >> a.nb_shift) - a.nb_lo[2];
        if (cx >= 0 && cx < a.nb_dim[0] && cy >= 0 && cy < a.nb_dim[1] && cz >= 0 &&
            cz < a.nb_dim[2]) {
          const int64_t cell = ((int64_t)cx * a.nb_dim[1] + cy) * a.nb_dim[2] + cz;
          beg = __ldg(a.t.nb_off + cell);
          cnt = __ldg(a.t.nb_off + cell + 1) - beg;
        }
#endif
        // H4 (O4)
        double phi;
        if constexpr (RT > 0) {
          using G = Geo<RT>;
          const bool inwin = use_win && i0 >= W.lo[0] && i0 <= W.hi[0] && i1 >= W.lo[1] &&
                             i1 <= W.hi[1] && i2 >= W.lo[2] && i2 <= W.hi[2];
#if defined(RS_EXPERIMENT) && (RS_EXPERIMENT & 2)
          if (inwin) {
            phi = z;
          } else
#endif
          if (inwin) {
            phi = long_phi<RT, true>(win + (size_t)(W.base[0] + i0 - W.lo[0]) * G::CHP,
                                     win + (size_t)(W.base[1] + i1 - W.lo[1]) * G::CHP,
                                     win + (size_t)(W.base[2] + i2 - W.lo[2]) * G::CHP, rho);
          } else {
            phi = long_phi_global<RT>(a.t.F[0], a.t.F[1], a.t.F[2], i0, i1, i2, rho);
          }
        } else {
          phi = long_phi_rt(a.t.F[0] + (size_t)i0 * a.R, a.t.F[1] + (size_t)i1 * a.R,
                            a.t.F[2] + (size_t)i2 * a.R, a.R);
        }
        dd_add_prod(hi, lo, z, phi);
      }
    }
    if (__any_sync(kFull, bad)) {
      bad = true;
      break;                      // the pose is invalid: NaN outputs, skip the rest
    }
    // H5 + H6 over the pass's (atom, candidate) pairs, flattened across the warp so every lane
    // works on some pair in every round (the pose sums are order-free, O6/O7); two rounds per
    // iteration keep two independent sets of loads in flight
    int inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += v;
    }
    const int total = __shfl_sync(kFull, inc, 31);
    if (total == 0) continue;
    const int myoff = inc - cnt;
    ps.x[0][lane] = xp[0];
    ps.x[1][lane] = xp[1];
    ps.x[2][lane] = xp[2];
    ps.z[lane] = z;
    ps.cell[lane] = make_int4(i0, i1, i2, beg);
    ps.off[lane] = myoff;
    int carry = 0;
    for (int base = 0; base < total; base += 64) {
      const int rel = myoff - base;
      const bool starts = cnt > 0 && rel >= 0 && rel < 64;
      __syncwarp();
      if (starts) ps.map[rel] = lane;
      const unsigned m0 = __reduce_or_sync(kFull, (starts && rel < 32) ? (1u << rel) : 0u);
      const unsigned m1 = __reduce_or_sync(kFull, (starts && rel >= 32) ? (1u << (rel - 32)) : 0u);
      __syncwarp();
      const unsigned long long m64 = ((unsigned long long)m1 << 32) | m0;
      const unsigned long long below0 = m64 & (0xffffffffull >> (31 - lane));
      const unsigned long long below1 = m64 & (0xffffffffffffffffull >> (31 - lane));
      const int ow0 = below0 ? ps.map[63 - __clzll(below0)] : carry;
      const int ow1 = below1 ? ps.map[63 - __clzll(below1)] : carry;
      carry = __shfl_sync(kFull, ow1, 31);
      const int k0 = base + lane, k1 = base + 32 + lane;
      int4 oc0 = make_int4(0, 0, 0, 0), oc1 = oc0;
      short4 mc0 = make_short4(0, 0, 0, 0), mc1 = mc0;
      double2 xy0 = make_double2(0.0, 0.0), zq0 = xy0, xy1 = xy0, zq1 = xy0;
      if (k0 < total) {
        oc0 = ps.cell[ow0];
        const int j = oc0.w + (k0 - ps.off[ow0]);
        mc0 = __ldg(ncell + j);
        xy0 = ldg2(nrec + 2 * (size_t)j);
        zq0 = ldg2(nrec + 2 * (size_t)j + 1);
      }
      if (k1 < total) {
        oc1 = ps.cell[ow1];
        const int j = oc1.w + (k1 - ps.off[ow1]);
        mc1 = __ldg(ncell + j);
        xy1 = ldg2(nrec + 2 * (size_t)j);
        zq1 = ldg2(nrec + 2 * (size_t)j + 1);
      }
      if (k0 < total) pair_term(a, ps, ow0, oc0, mc0, xy0, zq0, ns2, hi, lo, best);
      if (k1 < total) pair_term(a, ps, ow1, oc1, mc1, xy1, zq1, ns2, hi, lo, best);
    }
    __syncwarp();
  }
  // H7
  bad = __any_sync(kFull, bad);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double h2 = __shfl_xor_sync(kFull, hi, off);
    const double l2 = __shfl_xor_sync(kFull, lo, off);
    const double s = __dadd_rn(hi, h2);
    const double bb = __dsub_rn(s, hi);
    const double e = __dadd_rn(__dsub_rn(hi, __dsub_rn(s, bb)), __dsub_rn(h2, bb));
    hi = s;
    lo = __dadd_rn(__dadd_rn(lo, l2), e);
    best = fmin(best, __shfl_xor_sync(kFull, best, off));
  }
  // H8
  if (lane == 0) {
    if (bad) {
      a.E[p] = NAN;
      a.D[p] = NAN;
      if (a.invalid) atomicAdd(a.invalid, 1ull);
    } else {
      a.E[p] = __dadd_rn(hi, lo);
      a.D[p] = best < a.dcap2 ? __dsqrt_rn(best) : INFINITY;
    }
  }
}

template <int RT>
__global__ void __launch_bounds__(kThreads, 1) score_kernel(const ScoreArgs a, int cap_rows,
                                                            int lig_smem_n) {
  // dynamic shared memory: [PairStage x warps][PoseStage][ligand][factor-row window]
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PairStage* s_ps = reinterpret_cast<PairStage*>(smem_raw);
  PoseStage& s_pose = *reinterpret_cast<PoseStage*>(s_ps + kWarps);
  double4* s_lig = reinterpret_cast<double4*>(&s_pose + 1);
  double2* win = reinterpret_cast<double2*>(s_lig + lig_smem_n);
  __shared__ double s_red[kWarps][6];
  __shared__ int s_bad[kWarps];
  __shared__ int s_win[7];       // lo[3], hi[3], fits
  __shared__ Window s_cur;
  __shared__ double s_rmax2;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool lig_smem = a.L <= lig_smem_n;
  // ligand radius (body frame) and staging
  double r2 = 0.0;
  for (int64_t l = tid; l < a.L; l += kThreads) {
    const double y0 = __ldg(a.yl + 3 * l), y1 = __ldg(a.yl + 3 * l + 1), y2 = __ldg(a.yl + 3 * l + 2);
    r2 = fmax(r2, y0 * y0 + y1 * y1 + y2 * y2);
    if (lig_smem) s_lig[l] = make_double4(y0, y1, y2, __ldg(a.zl + l));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) r2 = fmax(r2, __shfl_xor_sync(kFull, r2, off));
  if (lane == 0) s_red[warp][0] = r2;
  if (tid == 0) {
    s_cur.lo[0] = s_cur.lo[1] = s_cur.lo[2] = 1;
    s_cur.hi[0] = s_cur.hi[1] = s_cur.hi[2] = 0;   // empty
  }
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int w = 0; w < kWarps; ++w) m = fmax(m, s_red[w][0]);
    s_rmax2 = m;
  }
  __syncthreads();
  // slack: |R y| <= |y| (1 + 1e-15) plus two cells for the snap rounding and the clamp
  const double rb = sqrt(s_rmax2) * (1.0 + 1e-12) + 2.0 * a.h;
  const bool window_mode = RT > 0 && cap_rows > 0;

  const int64_t p_begin = a.P * (int64_t)blockIdx.x / gridDim.x;
  const int64_t p_end = a.P * (int64_t)(blockIdx.x + 1) / gridDim.x;
  int64_t p = p_begin;
  while (p < p_end) {
    int T = (int)(p_end - p < (int64_t)kTile ? p_end - p : (int64_t)kTile);
    // H1 for the tile: one thread per pose
    if (tid < T) {
      const double* pq = a.poses + 7 * (p + tid);
      double qv[7];
#pragma unroll
      for (int i = 0; i < 7; ++i) qv[i] = __ldg(pq + i);
      double Rm[9];
      const bool ok = quat_rot_dev(qv, Rm);
#pragma unroll
      for (int i = 0; i < 9; ++i) s_pose.R[tid][i] = Rm[i];
#pragma unroll
      for (int i = 0; i < 3; ++i) s_pose.t[tid][i] = qv[4 + i];
      s_pose.ok[tid] = ok ? 1 : 0;
    }
    bool fits = false;
    if (window_mode) {
      for (;;) {
        // block min/max of the tile's translations (staged above)
        __syncthreads();
        double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
        int badt = 0;
        if (tid < T) {
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            const double t = s_pose.t[tid][r];
            if (!isfinite(t)) badt = 1;
            mn[r] = t;
            mx[r] = t;
          }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            mn[r] = fmin(mn[r], __shfl_xor_sync(kFull, mn[r], off));
            mx[r] = fmax(mx[r], __shfl_xor_sync(kFull, mx[r], off));
          }
        }
        badt = __any_sync(kFull, badt);
        if (lane == 0) {
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            s_red[warp][r] = mn[r];
            s_red[warp][3 + r] = mx[r];
          }
          s_bad[warp] = badt;
        }
        __syncthreads();
        if (tid == 0) {
          int bad = 0, rows = 0, lo[3], hi[3];
          for (int r = 0; r < 3; ++r) {
            double m0 = INFINITY, m1 = -INFINITY;
            for (int w = 0; w < kWarps; ++w) {
              m0 = fmin(m0, s_red[w][r]);
              m1 = fmax(m1, s_red[w][3 + r]);
              bad |= s_bad[w];
            }
            const double f0 = floor((m0 - rb + a.b) * a.inv_h) - 1.0;
            const double f1 = floor((m1 + rb + a.b) * a.inv_h) + 1.0;
            lo[r] = (int)fmax(0.0, fmin(f0, (double)(a.n - 1)));
            hi[r] = (int)fmax(0.0, fmin(f1, (double)(a.n - 1)));
            rows += hi[r] - lo[r] + 1;
          }
          const int fts = (!bad && rows <= cap_rows) ? 1 : 0;
          for (int r = 0; r < 3; ++r) {
            s_win[r] = lo[r];
            s_win[3 + r] = hi[r];
          }
          s_win[6] = fts;
        }
        __syncthreads();
        fits = s_win[6] != 0;
        if (fits || T == 1) break;
        T = (T + 1) / 2;           // the staged poses [0, T) stay valid
      }
      if (fits) {
        bool contained = true;
#pragma unroll
        for (int r = 0; r < 3; ++r)
          contained = contained && s_cur.lo[r] <= s_win[r] && s_win[3 + r] <= s_cur.hi[r];
        if (!contained) {
          if (tid == 0) {
            int rows = 0;
            for (int r = 0; r < 3; ++r) rows += s_win[3 + r] - s_win[r] + 1;
            const int extra = (cap_rows - rows) / 3;
            int base = 0;
            for (int r = 0; r < 3; ++r) {
              int lo = max(0, s_win[r] - extra / 2);
              int hi = min(a.n - 1, s_win[3 + r] + (extra - extra / 2));
              s_cur.lo[r] = lo;
              s_cur.hi[r] = hi;
              s_cur.base[r] = base;
              base += hi - lo + 1;
            }
          }
          __syncthreads();
          if constexpr (RT > 0) {
            using G = Geo<RT>;
            const int rows0 = s_cur.hi[0] - s_cur.lo[0] + 1, rows1 = s_cur.hi[1] - s_cur.lo[1] + 1;
            const int total = s_cur.base[2] + s_cur.hi[2] - s_cur.lo[2] + 1;
            for (int idx = tid; idx < total * G::CHP; idx += kThreads) {
              const int row = idx / G::CHP, ph = idx - row * G::CHP;
              const int ax = row < rows0 ? 0 : (row < rows0 + rows1 ? 1 : 2);
              const int grow = s_cur.lo[ax] + row - s_cur.base[ax];
              double2 v = make_double2(0.0, 0.0);
              const int src = G::REP ? (ph & (G::CH - 1)) : ph;
              if (G::REP || ph < G::CH) v = ldg2((const double2*)(a.t.F[ax] + (size_t)grow * RT) + src);
              win[idx] = v;
            }
          }
        }
      }
    }
    __syncthreads();
    const Window W = s_cur;
    for (int s = warp; s < T; s += kWarps) {
      double Rm[9], tv[3];
#pragma unroll
      for (int i = 0; i < 9; ++i) Rm[i] = s_pose.R[s][i];
#pragma unroll
      for (int i = 0; i < 3; ++i) tv[i] = s_pose.t[s][i];
      score_pose<RT>(a, p + s, Rm, tv, s_pose.ok[s] != 0, fits, W, win, s_lig, lig_smem, lane,
                     s_ps[warp]);
    }
    __syncthreads();
    p += T;
  }
}

struct DevCache {
  int sms = 0;
  int smem_optin = 0;
  bool attr_set[8] = {false};
  int max_dyn[8] = {0};
};
DevCache g_dev[64];

template <int RT>
int launch_t(const ScoreArgs& a, cudaStream_t st, int dev, int slot, bool window_mode) {
  DevCache& dc = g_dev[dev & 63];
  if (!dc.attr_set[slot]) {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, score_kernel<RT>);
    if (e != cudaSuccess) return (int)e;
    dc.max_dyn[slot] = dc.smem_optin - (int)fa.sharedSizeBytes;
    e = cudaFuncSetAttribute(score_kernel<RT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             dc.max_dyn[slot]);
    if (e != cudaSuccess) return (int)e;
    dc.attr_set[slot] = true;
  }
  constexpr int kChp = Geo<(RT > 0 ? RT : 2)>::CHP;
  const int lig_n = (int)std::min<int64_t>(a.L, kLigSmem);
  const size_t lig_b = (size_t)lig_n * sizeof(double4) + sizeof(PairStage) * kWarps + sizeof(PoseStage);
  size_t dyn = lig_b;
  int cap_rows = 0;
  if (RT > 0 && window_mode) {
    const size_t avail = (size_t)dc.max_dyn[slot] > lig_b ? (size_t)dc.max_dyn[slot] - lig_b : 0;
    cap_rows = (int)(avail / (16 * kChp));
    if (a.rmax_hint >= 0) {
      // leave the rest of the 228 KB to L1 (cell lists, records, memo): ~1.15x what one
      // translation's window needs
      const double need = 3.0 * (2.0 * (a.rmax_hint + 2.0 * a.h) / a.h + 8.0);
      cap_rows = std::min(cap_rows, (int)std::max(64.0, 1.15 * need));
    }
    dyn = lig_b + (size_t)cap_rows * 16 * kChp;
  }
  const int64_t tiles = (a.P + kTile - 1) / kTile;
  int grid = (int)std::min<int64_t>(tiles, (int64_t)dc.sms);
  if (grid < 1) grid = 1;
  score_kernel<RT><<<grid, kThreads, dyn, st>>>(a, cap_rows, lig_n);
  return (int)cudaGetLastError();
}

__global__ void fill_short_memo_kernel(const double* __restrict__ S0, const double* __restrict__ S1,
                                       const double* __restrict__ S2, int Rs, int ns, double* out) {
  const int64_t d = ns + 1, tot = d * d * d;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int e0 = (int)(t / (d * d)), e1 = (int)((t / d) % d), e2 = (int)(t % d);
    const double* s0 = S0 + (size_t)(e0 + ns) * Rs;
    const double* s1 = S1 + (size_t)(e1 + ns) * Rs;
    const double* s2 = S2 + (size_t)(e2 + ns) * Rs;
    double s = 0.0;                    // the O5 chain, ascending k
    for (int k = 0; k < Rs; ++k) s = __dadd_rn(s, __dmul_rn(__dmul_rn(s0[k], s1[k]), s2[k]));
    out[t] = s;
  }
}

}  // namespace

int launch_fill_short_memo(const double* S0, const double* S1, const double* S2, int Rs,
                           int n_sigma, double* out, void* stream) {
  fill_short_memo_kernel<<<1024, 256, 0, (cudaStream_t)stream>>>(S0, S1, S2, Rs, n_sigma, out);
  return (int)cudaGetLastError();
}

const char* score_kernel_variant(int R) {
  switch (R) {
    case 4: return "score_kernel<4>";
    case 8: return "score_kernel<8>";
    case 12: return "score_kernel<12>";
    case 16: return "score_kernel<16>";
    case 24: return "score_kernel<24>";
    case 32: return "score_kernel<32>";
    default: return "score_kernel<0> (runtime R)";
  }
}

int launch_score(const ScoreArgs& a, void* stream, int device, int* launches) {
  if (a.P <= 0) return 0;
  DevCache& dc = g_dev[device & 63];
  if (dc.sms == 0) {
    cudaDeviceGetAttribute(&dc.sms, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&dc.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  }
  cudaStream_t st = (cudaStream_t)stream;
  // window mode unless the ligand alone spans more rows than the window can hold
  bool window_mode = true;
  if (a.rmax_hint >= 0) {
    const double rows = 3.0 * (2.0 * (a.rmax_hint + 2.0 * a.h) / a.h + 4.0);
    const double row_b = 16.0 * (a.R <= 8 ? 8 : ((a.R / 2 + 7) / 8) * 8);
    window_mode = rows * row_b <= 0.9 * double(dc.smem_optin);
  }
  int e;
  switch (a.R) {
    case 4: e = launch_t<4>(a, st, device, 1, window_mode); break;
    case 8: e = launch_t<8>(a, st, device, 2, window_mode); break;
    case 12: e = launch_t<12>(a, st, device, 3, window_mode); break;
    case 16: e = launch_t<16>(a, st, device, 4, window_mode); break;
    case 24: e = launch_t<24>(a, st, device, 5, window_mode); break;
    case 32: e = launch_t<32>(a, st, device, 6, window_mode); break;
    default: e = launch_t<0>(a, st, device, 0, false); break;
  }
  if (launches) *launches += 1;
  return e;
}

}  // namespace rs
