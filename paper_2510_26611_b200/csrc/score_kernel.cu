// Fused sm_100a pose-scoring kernel: Algorithm PLIE with Lemma 3.2 /
// Eq. (18), the RS entry formula and the vdW constraint
// of Eq. (22).  Rows H1-H8 of SURVEY.md §8(a), in one pass:
//   H1 quaternion -> rotation      H2 x' = R y + t           H3 snap to the cell grid
//   H4 long-range CP gather + rank sum (rows of F_0, F_1, F_2 from a shared-memory window
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
// lanes accumulate and the reduction tree are free.  The snap (O3) is finished in integers
// after the two fp64 ops that define it (ceil of a value in [0, n+1) is exact).
//
// Work layout: persistent CTAs (one per SM, 32 warps) take chunks of
// consecutive poses from a global counter (guided: smaller chunks over the last poses); a warp
// scores one pose at a time (lanes over ligand atoms), taking poses from a per-tile queue.
// A tile is the longest run of poses whose rows fit the shared-memory window (a block scan of
// per-pose row bounds); the window's rows of the three factor matrices arrive by TMA bulk
// copies (cp.async.bulk, mbarrier completion) from a row-padded device copy, with slack so that
// the following tiles usually reuse them.  Rows are 16-byte chunks padded (R=12, 24) or
// replicated (R=4, 8) to whole 128-byte lines; lane l reads chunk c ^ (l & 7) of its own row in
// slot c, so the 8 lanes of every quarter-warp hit 8 distinct bank groups whatever rows they
// gather (conflict-free LDS.128); the halving tree over rank pairs is invariant under that
// relabelling, so no un-permute is needed.  RS_FLAG_F32_FACTORS (reading A21) runs the same
// machinery on binary32 rows of rank quads.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
#include <vector>

#include "rs_internal.h"

namespace rs {
namespace {

#ifndef RS_THREADS
#define RS_THREADS 1024
#endif
#ifndef RS_TILE
#define RS_TILE 512
#endif
#ifndef RS_CHUNK
#define RS_CHUNK 1024
#endif
#ifndef RS_WIN_SLACK
#define RS_WIN_SLACK 1.5
#endif
constexpr int kThreads = RS_THREADS;
constexpr int kWarps = kThreads / 32;
constexpr int kTile = RS_TILE;           // poses per tile (upper bound)
constexpr int kChunk = RS_CHUNK;         // poses per unit of dynamic CTA work
#ifndef RS_TAIL_DIV
#define RS_TAIL_DIV 8
#endif
#ifndef RS_TAIL_CHUNK
#define RS_TAIL_CHUNK 128
#endif
constexpr int kTailChunk = RS_TAIL_CHUNK;  // chunk size over the last 1/RS_TAIL_DIV of the poses
static_assert(kTile <= kThreads, "one thread per pose of a tile");
constexpr unsigned kFull = 0xffffffffu;
#ifndef RS_SLOTS
#define RS_SLOTS 1
#endif
constexpr int kSlots = RS_SLOTS;         // candidate slots per lane and flattened round

template <int R>
struct Geo {
  static constexpr int CH = R / 2;                                 // 16-byte chunks of a row
  static constexpr bool REP = (CH == 1 || CH == 2 || CH == 4);      // replicate to 128 B
  static constexpr int CHP = REP ? 8 : ((CH + 7) / 8) * 8;         // physical chunks per row
  static constexpr int NS = REP ? CH : CHP;                        // loads per row and lane
};

__device__ __forceinline__ double2 ldg2(const double2* p) { return __ldg(p); }

// Read-only global loads issued only when pr holds (the predicate is inside the instruction, so
// the compiler cannot turn a guarded load into an unguarded speculative one: the address may be
// meaningless when pr is false, and untaken lanes cost no L1 tag lookups).  Result 0 if !pr.
__device__ __forceinline__ double ldg_if(const double* p, bool pr) {
  double v = 0.0;
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.global.nc.f64 %0, [%1];\n}"
      : "+d"(v) : "l"(p), "r"((int)pr));
  return v;
}
__device__ __forceinline__ double2 ldg_if(const double2* p, bool pr) {
  double2 v = make_double2(0.0, 0.0);
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n @q ld.global.nc.v2.f64 {%0, %1}, [%2];\n}"
      : "+d"(v.x), "+d"(v.y) : "l"(p), "r"((int)pr));
  return v;
}
// one 256-bit read-only load (LDG.E.ENL2.256 on sm_100): a whole 32-byte sector per lane
__device__ __forceinline__ double4 ldg256(const double4* p) {
  double4 v;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ldg256x2(const float4* p, float4& hi) {
  float4 v;
  asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w), "=f"(hi.x), "=f"(hi.y), "=f"(hi.z), "=f"(hi.w)
      : "l"(p));
  return v;
}

// one 256-bit load (LDG.E.ENL2.256 on sm_100): one L1 tag lookup for a 32-byte record
__device__ __forceinline__ double4 ldg_if(const double4* p, bool pr) {
  double4 v = make_double4(0.0, 0.0, 0.0, 0.0);
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %5, 0;\n @q ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];\n}"
      : "+d"(v.x), "+d"(v.y), "+d"(v.z), "+d"(v.w) : "l"(p), "r"((int)pr));
  return v;
}
__device__ __forceinline__ int2 ldg_if(const int2* p, bool pr) {
  int2 v = make_int2(0, 0);
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n @q ld.global.nc.v2.s32 {%0, %1}, [%2];\n}"
      : "+r"(v.x), "+r"(v.y) : "l"(p), "r"((int)pr));
  return v;
}
__device__ __forceinline__ int4 ldg_if(const int4* p, bool pr) {
  int4 v = make_int4(0, 0, 0, 0);
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %5, 0;\n @q ld.global.nc.v4.s32 {%0, %1, %2, %3}, [%4];\n}"
      : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w) : "l"(p), "r"((int)pr));
  return v;
}

// O3 cell of a valid coordinate: u = (x + b) * inv_h in [0, n(1+eps)]; i = clamp(ceil(u)-1)
__device__ __forceinline__ int snap_dev(double x, double b, double inv_h, int nm1) {
  const double u = __dmul_rn(__dadd_rn(x, b), inv_h);
  int c;
  asm("cvt.rpi.s32.f64 %0, %1;" : "=r"(c) : "d"(u));
  return min(max(c - 1, 0), nm1);
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

// One rank pair: s_c = (a0 b0) c0 + (a1 b1) c1
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

// O4 with compile-time R from the shared-memory window.  rK = byte offset of row K from the
// window base (a multiple of the row size, the base 256-B aligned).  Slot c reads physical
// chunk c ^ rho (rho = lane & 7): the 8 lanes of a quarter-warp hit 8 distinct 16-byte bank
// groups whatever rows they read.  Physical chunk p holds pair p (padded widths: zero beyond CH;
// replicated widths: pair p mod CH), so slot c holds pair (c ^ rho) mod NS, and the halving
// tree, which combines c with c ^ m at every level, is bitwise invariant under that relabelling.
// The halving tree evaluated depth-first: T(c, stride, cnt) = T(c, 2 stride, cnt/2) +
// T(c + stride, 2 stride, cnt/2), leaves = slot pair sums.  Same pairings as the level-by-level
// loop (pair c meets c + NS/2 first), but partial sums retire as soon as their chunks arrive,
// so fewer values are live while the gathers are in flight.
template <int C, int STRIDE, int CNT>
struct SmemTree {
  static __device__ __forceinline__ double eval(const char* win, unsigned r0, unsigned r1,
                                                unsigned r2) {
    if constexpr (CNT == 1) {
      constexpr unsigned o = (unsigned)C << 4;
      return pair_prod(*reinterpret_cast<const double2*>(win + (r0 ^ o)),
                       *reinterpret_cast<const double2*>(win + (r1 ^ o)),
                       *reinterpret_cast<const double2*>(win + (r2 ^ o)));
    } else {
      const double lhs = SmemTree<C, 2 * STRIDE, CNT / 2>::eval(win, r0, r1, r2);
      const double rhs = SmemTree<C + STRIDE, 2 * STRIDE, CNT / 2>::eval(win, r0, r1, r2);
      return __dadd_rn(lhs, rhs);
    }
  }
};

template <int R>
__device__ __forceinline__ double long_phi_smem(const char* win, unsigned r0, unsigned r1,
                                                unsigned r2, int rho) {
  using G = Geo<R>;
  const unsigned x = (unsigned)rho << 4;
  return SmemTree<0, 1, G::NS>::eval(win, r0 | x, r1 | x, r2 | x);
}

// O4 with compile-time R from L2 (unpadded n x R rows); slot c = pair c (no bank structure)
template <int R>
__device__ __forceinline__ double long_phi_l2(const double2* r0, const double2* r1, const double2* r2) {
  // 32-byte loads (two rank pairs, LDG.E.ENL2.256): a whole L2 sector per lane and request,
  // twice the useful bytes per sector of 16-byte loads when every lane reads its own row
  using G = Geo<R>;
  constexpr int C = G::REP ? G::CH : G::CHP;
  static_assert(G::CH % 2 == 0 || G::CH == 1, "rows are whole 32-byte sectors");
  double s[C];
#pragma unroll
  for (int c = 0; c < C; ++c) s[c] = 0.0;
  if constexpr (G::CH == 1) {
    s[0] = pair_prod(__ldg(r0), __ldg(r1), __ldg(r2));
  } else {
    const double4* q0 = reinterpret_cast<const double4*>(r0);
    const double4* q1 = reinterpret_cast<const double4*>(r1);
    const double4* q2 = reinterpret_cast<const double4*>(r2);
#pragma unroll
    for (int c = 0; c < G::CH / 2; ++c) {
      const double4 a = ldg256(q0 + c), b = ldg256(q1 + c), cc = ldg256(q2 + c);
      s[2 * c] = pair_prod(make_double2(a.x, a.y), make_double2(b.x, b.y), make_double2(cc.x, cc.y));
      s[2 * c + 1] = pair_prod(make_double2(a.z, a.w), make_double2(b.z, b.w), make_double2(cc.z, cc.w));
    }
  }
  return halving_tree<C>(s);
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

// L2 path of O4 for compile-time R, kept out of line (it is the rare path in window mode)
template <int RT>
__device__ __noinline__ double long_phi_global(const double* F0, const double* F1, const double* F2,
                                               int i0, int i1, int i2) {
  return long_phi_l2<RT>((const double2*)(F0 + (size_t)i0 * RT), (const double2*)(F1 + (size_t)i1 * RT),
                         (const double2*)(F2 + (size_t)i2 * RT));
}

// ---- the binary32-factor variant (reading A21) -----------------------------------
// Rows of R floats as 16-byte quads of ranks: CHA = smallest power of two >= ceil(R/4) quads,
// zero-padded, replicated to 8 chunks (128 B) when CHA < 8.
template <int R>
struct Geo32 {
  static constexpr int CH = (R + 3) / 4;
  static constexpr int CHA = CH <= 1 ? 1 : CH <= 2 ? 2 : CH <= 4 ? 4 : CH <= 8 ? 8 : 16;
  static constexpr int CHP = CHA < 8 ? 8 : CHA;
  static constexpr int NS = CHA;
};

// One rank quad: s_c = ((a0 b0) c0 + (a1 b1) c1) + ((a2 b2) c2 + (a3 b3) c3), binary32
__device__ __forceinline__ float quad_prod(float4 a, float4 b, float4 c) {
  const float q0 = __fmul_rn(__fmul_rn(a.x, b.x), c.x), q1 = __fmul_rn(__fmul_rn(a.y, b.y), c.y);
  const float q2 = __fmul_rn(__fmul_rn(a.z, b.z), c.z), q3 = __fmul_rn(__fmul_rn(a.w, b.w), c.w);
  return __fadd_rn(__fadd_rn(q0, q1), __fadd_rn(q2, q3));
}

// The quad halving tree, depth-first, from the shared-memory window (XOR chunk order as in
// the binary64 path: the tree is invariant under the relabelling)
template <int C, int STRIDE, int CNT>
struct SmemTree32 {
  static __device__ __forceinline__ float eval(const char* win, unsigned r0, unsigned r1,
                                               unsigned r2) {
    if constexpr (CNT == 1) {
      constexpr unsigned o = (unsigned)C << 4;
      return quad_prod(*reinterpret_cast<const float4*>(win + (r0 ^ o)),
                       *reinterpret_cast<const float4*>(win + (r1 ^ o)),
                       *reinterpret_cast<const float4*>(win + (r2 ^ o)));
    } else {
      const float lhs = SmemTree32<C, 2 * STRIDE, CNT / 2>::eval(win, r0, r1, r2);
      const float rhs = SmemTree32<C + STRIDE, 2 * STRIDE, CNT / 2>::eval(win, r0, r1, r2);
      return __fadd_rn(lhs, rhs);
    }
  }
};

// L2 path of O4-f32: rows of the packed binary32 copy, quads in natural order
template <int R>
__device__ __noinline__ double long_phi_global32(const float4* F0, const float4* F1,
                                                 const float4* F2, int i0, int i1, int i2) {
  using G = Geo32<R>;
  const float4* r0 = F0 + (size_t)i0 * G::CHP;
  const float4* r1 = F1 + (size_t)i1 * G::CHP;
  const float4* r2 = F2 + (size_t)i2 * G::CHP;
  float s[G::NS];
  if constexpr (G::NS == 1) {
    s[0] = quad_prod(__ldg(r0), __ldg(r1), __ldg(r2));
  } else {
    // 32-byte loads: two quads per lane and request, only the CH quads that hold ranks (the
    // zero padding up to NS quads contributes s_c = +0 exactly, so it is not read: R = 24
    // reads 96 of the row's 128 bytes)
#pragma unroll
    for (int c = 0; c < G::NS; c += 2) {
      if (c + 1 < G::CH) {
        float4 a1, b1, c1;
        const float4 a0 = ldg256x2(r0 + c, a1), b0 = ldg256x2(r1 + c, b1), c0 = ldg256x2(r2 + c, c1);
        s[c] = quad_prod(a0, b0, c0);
        s[c + 1] = quad_prod(a1, b1, c1);
      } else if (c < G::CH) {
        s[c] = quad_prod(__ldg(r0 + c), __ldg(r1 + c), __ldg(r2 + c));
        s[c + 1] = 0.0f;
      } else {
        s[c] = 0.0f;
        s[c + 1] = 0.0f;
      }
    }
  }
#pragma unroll
  for (int m = G::NS / 2; m >= 1; m /= 2) {
#pragma unroll
    for (int c = 0; c < m; ++c) s[c] = __fadd_rn(s[c], s[c + m]);
  }
  return (double)s[0];
}

struct ChunkPlan {             // dynamic schedule: nbig chunks of `big` poses, then `tail`-pose chunks
  int64_t nbig;
  int big, tail;
};

struct Window {
  int lo[3], hi[3], off[3];    // staged rows [lo, hi] per axis; smem row of row i = i + off
};


struct __align__(16) PoseRec {  // H1 output of one pose: R (row-major) and t
  double m[12];
};

// Per-warp staging of the 32 atoms of one pass for the flattened candidate-pair rounds.
template <int NA>
struct __align__(16) PairStage {
  double2 x01[32 * NA]; // x'_0, x'_1 of slot 32 u + lane (written only for atoms with candidates)
  double2 x2z[32 * NA]; // x'_2, charge
  int4 cb[32 * NA];     // i0, i1, i2, (list begin - start of the atom's candidate segment)
  int map[32 * kSlots]; // candidate slot where an atom's segment starts -> atom slot
};

// ---- TMA bulk copy + mbarrier (window staging) ---------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// O5 value s(D): from the dense memo (filled by the same chain) or the chain itself
__device__ __forceinline__ double short_value(const ScoreArgs& a, int e0, int e1, int e2) {
  if (a.t.short_memo) {
    const int d = a.n_sigma + 1;
    return ldg_if(a.t.short_memo + (abs(e0) * d + abs(e1)) * d + abs(e2), true);
  }
  const double* s0 = a.t.S[0] + (size_t)(e0 + a.n_sigma) * a.Rs;
  const double* s1 = a.t.S[1] + (size_t)(e1 + a.n_sigma) * a.Rs;
  const double* s2 = a.t.S[2] + (size_t)(e2 + a.n_sigma) * a.Rs;
  double s = 0.0;
  for (int k = 0; k < a.Rs; ++k)
    s = __dadd_rn(s, __dmul_rn(__dmul_rn(__ldg(s0 + k), __ldg(s1 + k)), __ldg(s2 + k)));
  return s;
}

// One candidate pair: an atom of the pass (cell oc, coordinates and charge ox) and a list entry
// en = (i0 | i1 << 16, i2, sorted atom k).  O7 distance when the integer prefilter admits it,
// O5 replica term inside the n_sigma ball.  Cells are < 2^15, so the squared integer offsets sum
// exactly in 32 unsigned bits.
__device__ __forceinline__ unsigned pair_dd(const int4 oc, const int4 en) {
  const int e0 = oc.x - (en.x & 0xffff), e1 = oc.y - (int)((unsigned)en.x >> 16), e2 = oc.z - en.y;
  return (unsigned)(e0 * e0) + (unsigned)(e1 * e1) + (unsigned)(e2 * e2);
}
__device__ __forceinline__ void pair_term(const ScoreArgs& a, const double4 ox, unsigned dd,
                                          double sv, double2 xy, double2 zq, double& hi, double& lo,
                                          double& best) {
  if (dd < a.vdw_cells2) {
    const double dx0 = __dsub_rn(ox.x, xy.x);
    const double dx1 = __dsub_rn(ox.y, xy.y);
    const double dx2 = __dsub_rn(ox.z, zq.x);
    const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx0, dx0), __dmul_rn(dx1, dx1)), __dmul_rn(dx2, dx2));
    best = fmin(best, d2);
  }
  if (dd <= a.ns2) dd_add_prod(hi, lo, ox.w, __dmul_rn(zq.y, sv));
}

// O5 value for a pair inside the n_sigma ball (issued as soon as the offset is known)
__device__ __forceinline__ double pair_short(const ScoreArgs& a, const int4 oc, const int4 en) {
#if defined(RS_EXPERIMENT) && (RS_EXPERIMENT & 8)
  return 1.0;
#else
  return short_value(a, oc.x - (en.x & 0xffff), oc.y - (int)((unsigned)en.x >> 16), oc.z - en.y);
#endif
}

// Per-atom state of one pass slot (H2/H3 output and the atom's candidate-list range)
struct AtomState {
  double x0, x1, x2, z;
  int i0, i1, i2, beg, cnt;
  bool go;                     // a real ligand atom (l < L) inside the box
};

// H2, H3 and the candidate-range lookup for ligand atom l of one pose.  bad is set if the atom
// leaves the box (O8).  Lanes past the ligand's end (l >= L) run them on atom L-1 and get
// go = false, z = 0 (branch-free; they contribute nothing).
template <bool LIG_SMEM>
__device__ __forceinline__ void atom_stage(const ScoreArgs& a, int l, const double* Rm,
                                           const double* tv, const double2* s_lig, int lig_n,
                                           AtomState& st,
                                           bool& bad) {
  const bool act = l < a.L;
  const int lc = act ? l : a.L - 1;
  double y0, y1, y2, z;
  if constexpr (LIG_SMEM) {
    // ligand staged structure-of-arrays: (y0, y1) then (y2, z), conflict-free 16-byte loads
    const double2 v0 = s_lig[lc], v1 = s_lig[lig_n + lc];
    y0 = v0.x; y1 = v0.y; y2 = v1.x; z = v1.y;
  } else {
    y0 = __ldg(a.yl + 3 * (int64_t)lc);
    y1 = __ldg(a.yl + 3 * (int64_t)lc + 1);
    y2 = __ldg(a.yl + 3 * (int64_t)lc + 2);
    z = __ldg(a.zl + lc);
  }
  st.z = act ? z : 0.0;
  // H2 (O2)
  st.x0 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(Rm[0], y0), __dmul_rn(Rm[1], y1)), __dmul_rn(Rm[2], y2)), tv[0]);
  st.x1 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(Rm[3], y0), __dmul_rn(Rm[4], y1)), __dmul_rn(Rm[5], y2)), tv[1]);
  st.x2 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(Rm[6], y0), __dmul_rn(Rm[7], y1)), __dmul_rn(Rm[8], y2)), tv[2]);
  // H3 (O3): valid iff -b <= x'_a <= b on every axis (false for NaN)
  const bool ok = fabs(st.x0) <= a.b && fabs(st.x1) <= a.b && fabs(st.x2) <= a.b;
  bad = bad || (act && !ok);
  st.go = act && ok;
  const int nm1 = a.n - 1;
  st.i0 = snap_dev(st.x0, a.b, a.inv_h, nm1);
  st.i1 = snap_dev(st.x1, a.b, a.inv_h, nm1);
  st.i2 = snap_dev(st.x2, a.b, a.inv_h, nm1);
  st.beg = 0;
  st.cnt = 0;
#if !(defined(RS_EXPERIMENT) && (RS_EXPERIMENT & 1))
  // candidate range of the coarse cell containing i (cell lists cover every protein atom that can
  // matter to H5/H6 for any point of the cell); loaded before H4 so its latency hides behind it
  const unsigned cx = (unsigned)((st.i0 >> a.nb_shift) - a.nb_lo[0]);
  const unsigned cy = (unsigned)((st.i1 >> a.nb_shift) - a.nb_lo[1]);
  const unsigned cz = (unsigned)((st.i2 >> a.nb_shift) - a.nb_lo[2]);
  {
    const bool in = st.go && cx < (unsigned)a.nb_dim[0] && cy < (unsigned)a.nb_dim[1] && cz < (unsigned)a.nb_dim[2];
    const int2 bc = ldg_if(a.t.nb_range + (cx * a.nb_dim[1] + cy) * a.nb_dim[2] + cz, in);
    st.beg = bc.x;
    st.cnt = bc.y;
  }
#endif
}

// H4 (O4) for the NA atoms of a lane: atoms whose rows are staged read the window, real atoms
// outside it (rare) read L2, lanes past the ligand's end skip it (phi = 0, weight z = 0).
// F32: O4-f32 from the binary32 rows (A21).
template <int RT, int NA, bool F32>
__device__ __forceinline__ void long_range_stage(const ScoreArgs& a, const AtomState* st,
                                                 bool use_win, const Window& W, const char* win,
                                                 int rho, double* hi, double* lo) {
  double phi[NA];
#pragma unroll
  for (int u = 0; u < NA; ++u) phi[u] = 0.0;
  if constexpr (RT > 0) {
    constexpr int kChp = F32 ? Geo32<RT>::CHP : Geo<RT>::CHP;
    constexpr unsigned kRow = 16u * kChp;
    bool l2[NA];
    unsigned r0[NA], r1[NA], r2[NA];
#pragma unroll
    for (int u = 0; u < NA; ++u) {
      const bool inwin = use_win && (unsigned)(st[u].i0 - W.lo[0]) <= (unsigned)(W.hi[0] - W.lo[0]) &&
                         (unsigned)(st[u].i1 - W.lo[1]) <= (unsigned)(W.hi[1] - W.lo[1]) &&
                         (unsigned)(st[u].i2 - W.lo[2]) <= (unsigned)(W.hi[2] - W.lo[2]);
      l2[u] = st[u].go && !inwin;
      const bool w = st[u].go && inwin;
      r0[u] = w ? (unsigned)(st[u].i0 + W.off[0]) * kRow : 0u;
      r1[u] = w ? (unsigned)(st[u].i1 + W.off[1]) * kRow : 0u;
      r2[u] = w ? (unsigned)(st[u].i2 + W.off[2]) * kRow : 0u;
    }
    if (use_win) {
#pragma unroll
      for (int u = 0; u < NA; ++u) {
#if defined(RS_EXPERIMENT) && (RS_EXPERIMENT & 2)
        phi[u] = st[u].z;
#else
        if (st[u].go && !l2[u]) {
          if constexpr (F32) {
            const unsigned x = (unsigned)rho << 4;
            phi[u] = (double)SmemTree32<0, 1, Geo32<RT>::NS>::eval(win, r0[u] | x, r1[u] | x, r2[u] | x);
          } else {
            phi[u] = long_phi_smem<RT>(win, r0[u], r1[u], r2[u], rho);
          }
        }
#endif
      }
    }
#pragma unroll
    for (int u = 0; u < NA; ++u)
      if (l2[u]) {
        if constexpr (F32)
          phi[u] = long_phi_global32<RT>(a.t.Fw32[0], a.t.Fw32[1], a.t.Fw32[2], st[u].i0, st[u].i1, st[u].i2);
        else
          phi[u] = long_phi_global<RT>(a.t.F[0], a.t.F[1], a.t.F[2], st[u].i0, st[u].i1, st[u].i2);
      }
  } else {
#pragma unroll
    for (int u = 0; u < NA; ++u) {
      if (st[u].go)
        phi[u] = long_phi_rt(a.t.F[0] + (size_t)st[u].i0 * a.R, a.t.F[1] + (size_t)st[u].i1 * a.R,
                             a.t.F[2] + (size_t)st[u].i2 * a.R, a.R);
    }
  }
#pragma unroll
  for (int u = 0; u < NA; ++u) dd_add_prod(hi[u], lo[u], st[u].z, phi[u]);
}

// (hi, lo) += (h2, l2) exactly up to the final lo rounding (TwoSum on the high parts)
__device__ __forceinline__ void dd_merge(double& hi, double& lo, double h2, double l2) {
  const double s = __dadd_rn(hi, h2);
  const double bb = __dsub_rn(s, hi);
  const double e = __dadd_rn(__dsub_rn(hi, __dsub_rn(s, bb)), __dsub_rn(h2, bb));
  hi = s;
  lo = __dadd_rn(__dadd_rn(lo, l2), e);
}

__device__ __forceinline__ void load_pose(const PoseRec& pr, double* Rm, double* tv) {
  const double2* m2 = reinterpret_cast<const double2*>(pr.m);
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const double2 v = m2[i];
    const int k0 = 2 * i, k1 = 2 * i + 1;
    if (k0 < 9) Rm[k0] = v.x; else tv[k0 - 9] = v.x;
    if (k1 < 9) Rm[k1] = v.y; else tv[k1 - 9] = v.y;
  }
}

// Score one pose with one warp: lanes over ligand atoms, NA atoms per lane and pass (NA = 2
// gives every lane two independent dependency chains and halves the per-pass overheads).
template <int RT, int NA, bool F32>
__device__ __forceinline__ void score_pose(const ScoreArgs& a, int64_t p, const PoseRec& pr,
                                           bool ok, bool use_win, const Window& W,
                                           const char* win, const double2* s_lig, int lig_smem_n,
                                           int lane, PairStage<NA>& ps,
                                           double2& out) {
  double hi[NA], lo[NA], best = INFINITY;
#pragma unroll
  for (int u = 0; u < NA; ++u) hi[u] = lo[u] = 0.0;
  bool bad = !ok;
  const int rho = lane & 7;
  const bool lig_all_smem = a.L <= lig_smem_n;
  const int L = ok ? a.L : 0;
  const unsigned lanemask_le = 0xffffffffu >> (31 - lane);
  for (int l0 = 0; l0 < L; l0 += 32 * NA) {
    // the pose's R and t, re-read from shared memory (broadcast) each pass: they are live only
    // during H2, which keeps registers for more resident warps
    double Rm[9], tv[3];
    load_pose(pr, Rm, tv);
    AtomState st[NA];
#pragma unroll
    for (int u = 0; u < NA; ++u) {
      if (lig_all_smem) atom_stage<true>(a, l0 + 32 * u + lane, Rm, tv, s_lig, lig_smem_n, st[u], bad);
      else atom_stage<false>(a, l0 + 32 * u + lane, Rm, tv, s_lig, lig_smem_n, st[u], bad);
    }
    long_range_stage<RT, NA, F32>(a, st, use_win, W, win, rho, hi, lo);
    if (__any_sync(kFull, bad)) {
      bad = true;
      break;                      // the pose is invalid: NaN outputs, skip the rest
    }
    // H5 + H6 over the pass's (atom, candidate) pairs, flattened across the warp so every lane
    // works on some pair in every round (the pose sums are order-free, O6/O7); two slots per
    // lane and round keep two independent sets of loads in flight
    int cl = 0;
#pragma unroll
    for (int u = 0; u < NA; ++u) cl += st[u].cnt;
    if (__ballot_sync(kFull, cl > 0) == 0) continue;
    int inc = cl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += v;
    }
    const int total = __shfl_sync(kFull, inc, 31);
    int seg[NA];
    {
      int s0 = inc - cl;
#pragma unroll
      for (int u = 0; u < NA; ++u) {
        seg[u] = s0;
        if (st[u].cnt > 0) {        // only atoms with candidates are ever read back
          ps.x01[32 * u + lane] = make_double2(st[u].x0, st[u].x1);
          ps.x2z[32 * u + lane] = make_double2(st[u].x2, st[u].z);
          ps.cb[32 * u + lane] = make_int4(st[u].i0, st[u].i1, st[u].i2, st[u].beg - s0);
        }
        s0 += st[u].cnt;
      }
    }
    int carry = 0;
    for (int base = 0; base < total; base += 32 * kSlots) {
      unsigned m[kSlots];
#pragma unroll
      for (int q = 0; q < kSlots; ++q) m[q] = 0;
      __syncwarp();
#pragma unroll
      for (int u = 0; u < NA; ++u) {
        const int rel = seg[u] - base;
        if (st[u].cnt > 0 && rel >= 0 && rel < 32 * kSlots) {
          ps.map[rel] = 32 * u + lane;
#pragma unroll
          for (int q = 0; q < kSlots; ++q)
            if ((rel >> 5) == q) m[q] |= 1u << (rel & 31);
        }
      }
#pragma unroll
      for (int q = 0; q < kSlots; ++q) m[q] = __reduce_or_sync(kFull, m[q]);
      __syncwarp();
      // owner of slot base + 32 q + lane: the last segment starting at or before it
      int ow[kSlots];
      {
        int prev = carry;
#pragma unroll
        for (int q = 0; q < kSlots; ++q) {
          const unsigned bq = m[q] & lanemask_le;
          ow[q] = bq ? ps.map[32 * q + 31 - __clz(bq)] : prev;
          if (q + 1 < kSlots) prev = m[q] ? ps.map[32 * q + 31 - __clz(m[q])] : prev;
        }
      }
      carry = __shfl_sync(kFull, ow[kSlots - 1], 31);
      int4 oc[kSlots], en[kSlots];
      unsigned dd[kSlots];
      bool sr[kSlots], nr[kSlots];
      double sv[kSlots];
      double2 xy[kSlots], zq[kSlots];
#pragma unroll
      for (int q = 0; q < kSlots; ++q) {
        const int k = base + 32 * q + lane;
        oc[q] = make_int4(0, 0, 0, 0);
        en[q] = oc[q];
        if (k < total) oc[q] = ps.cb[ow[q]];
        en[q] = ldg_if(a.t.nb_ent + oc[q].w + k, k < total);
        dd[q] = k < total ? pair_dd(oc[q], en[q]) : 0xffffffffu;
        sr[q] = dd[q] <= a.ns2;
        nr[q] = sr[q] || dd[q] < a.vdw_cells2;
      }
      // loads of this round, all independent: memo values, then records
#pragma unroll
      for (int q = 0; q < kSlots; ++q) sv[q] = sr[q] ? pair_short(a, oc[q], en[q]) : 0.0;
#pragma unroll
      for (int q = 0; q < kSlots; ++q) {
        xy[q] = make_double2(0.0, 0.0);
        zq[q] = xy[q];
        const double4 r4 = ldg_if(a.t.prec + en[q].z, nr[q]);
        xy[q] = make_double2(r4.x, r4.y);
        zq[q] = make_double2(r4.z, r4.w);
      }
#pragma unroll
      for (int q = 0; q < kSlots; ++q)
        if (nr[q]) {
          const double2 o01 = ps.x01[ow[q]], o2z = ps.x2z[ow[q]];
          pair_term(a, make_double4(o01.x, o01.y, o2z.x, o2z.y), dd[q], sv[q], xy[q], zq[q],
                    hi[q % NA], lo[q % NA], best);
        }
    }
    __syncwarp();
  }
  // H7: double-double butterfly (TwoSum is exact, so all lanes agree); min of d^2 >= +0 by its
  // bit pattern (non-negative doubles order like their unsigned bits)
  bad = __any_sync(kFull, bad);
  double H = 0.0, Lo = 0.0;
  unsigned mhi = 0, mlo = 0;
  if (!bad) {
    H = hi[0];
    Lo = lo[0];
#pragma unroll
    for (int u = 1; u < NA; ++u) dd_merge(H, Lo, hi[u], lo[u]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double h2 = __shfl_xor_sync(kFull, H, off);
      const double l2 = __shfl_xor_sync(kFull, Lo, off);
      dd_merge(H, Lo, h2, l2);
    }
    const unsigned long long bb = (unsigned long long)__double_as_longlong(best);
    const unsigned bhi = (unsigned)(bb >> 32);
    mhi = __reduce_min_sync(kFull, bhi);
    mlo = __reduce_min_sync(kFull, bhi == mhi ? (unsigned)bb : 0xffffffffu);
  }
  // H8 is finished per tile (one thread per pose, coalesced stores): keep E and min d^2
  if (lane == 0) {
    out.x = bad ? NAN : __dadd_rn(H, Lo);
    out.y = bad ? NAN : __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
    if (bad && a.invalid) atomicAdd(a.invalid, 1ull);
  }
}

template <int NA>
__host__ __device__ constexpr size_t win_offset() {
  return ((sizeof(PoseRec) * kTile + sizeof(PairStage<NA>) * kWarps) + 255) / 256 * 256;
}

template <int RT, int NA, bool F32>
__global__ void __launch_bounds__(kThreads, 1) score_kernel(const ScoreArgs a, int cap_rows,
                                                            int lig_smem_n, const ChunkPlan cp) {
  // dynamic shared memory (256-B aligned base; every offset but the ligand's is a compile-time
  // constant, so addresses are immediates rather than recomputed values):
  //   [PoseRec x kTile][PairStage x warps][factor-row window, 256-B aligned][ligand 2 x double2 x n]
  extern __shared__ __align__(256) unsigned char smem_raw[];
  constexpr int kChp = F32 ? Geo32<(RT > 0 ? RT : 4)>::CHP : Geo<(RT > 0 ? RT : 2)>::CHP;
  PoseRec* s_pose = reinterpret_cast<PoseRec*>(smem_raw);
  PairStage<NA>* s_ps = reinterpret_cast<PairStage<NA>*>(smem_raw + sizeof(PoseRec) * kTile);
  double2* win = reinterpret_cast<double2*>(smem_raw + win_offset<NA>());
  double2* s_lig = reinterpret_cast<double2*>(smem_raw + win_offset<NA>() + (size_t)cap_rows * kChp * 16);
  __shared__ int s_ok[kTile];
  __shared__ double2 s_out[kTile];    // per pose of the tile: (E, min d^2), NaN if invalid
  __shared__ int s_wred[kWarps][8];
  __shared__ Window s_cur;
  __shared__ int s_next, s_restaged, s_chunk;
  __shared__ double s_rmax2[kWarps];
  __shared__ __align__(8) uint64_t s_bar;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ligand radius (body frame) and staging
  double r2 = 0.0;
  for (int l = tid; l < a.L; l += kThreads) {
    const double y0 = __ldg(a.yl + 3 * (int64_t)l), y1 = __ldg(a.yl + 3 * (int64_t)l + 1),
                 y2 = __ldg(a.yl + 3 * (int64_t)l + 2);
    r2 = fmax(r2, y0 * y0 + y1 * y1 + y2 * y2);
    if (l < lig_smem_n) {
      s_lig[l] = make_double2(y0, y1);
      s_lig[lig_smem_n + l] = make_double2(y2, __ldg(a.zl + l));
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) r2 = fmax(r2, __shfl_xor_sync(kFull, r2, off));
  if (lane == 0) s_rmax2[warp] = r2;
  if (tid == 0) {
    s_cur.lo[0] = s_cur.lo[1] = s_cur.lo[2] = 1;
    s_cur.hi[0] = s_cur.hi[1] = s_cur.hi[2] = 0;   // empty
    s_cur.off[0] = s_cur.off[1] = s_cur.off[2] = 0;
    mbar_init(&s_bar);
  }
  __syncthreads();
  double rmax2 = 0.0;
  for (int w = 0; w < kWarps; ++w) rmax2 = fmax(rmax2, s_rmax2[w]);
  // slack: |R y| <= |y| (1 + 1e-15) plus two cells for the snap rounding and the clamp
  const double rb = sqrt(rmax2) * (1.0 + 1e-12) + 2.0 * a.h;
  const bool window_mode = RT > 0 && cap_rows > 0;
  unsigned phase = 0;

  // dynamic chunks of kChunk consecutive poses (a global work counter): the neighbour work per
  // pose varies by an order of magnitude between translations, so static ranges leave the
  // busiest SM 2-3x behind the mean
  for (;;) {
    if (tid == 0) s_chunk = atomicAdd(a.work, 1);
    __syncthreads();
    // guided schedule (host-computed, ChunkPlan): nbig chunks of `big` poses, then chunks of
    // `tail` poses so that the CTAs finish together
    const int64_t nbig = cp.nbig;
    const int64_t c0 = s_chunk < nbig ? (int64_t)s_chunk * cp.big
                                      : nbig * cp.big + (int64_t)(s_chunk - nbig) * cp.tail;
    if (c0 >= a.P) break;
    const int64_t csz = s_chunk < nbig ? cp.big : cp.tail;
    const int64_t p_end = c0 + csz < a.P ? c0 + csz : a.P;
    if (a.arrive) {
      // streamed launch: wait until the copy chunk holding the work chunk's last pose landed
      // (copies land in order); chunk boundaries are 128-byte aligned in the pose array, so no
      // cache line mixes landed and pending poses
      if (tid == 0) {
        int c = 0;
        while (c + 1 < a.n_cb && a.cb[c + 1] <= p_end - 1) ++c;
        unsigned v = 0;
        for (long long spin = 0;; ++spin) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.arrive + c) : "memory");
          if (v != 0) break;
          if (spin > (1ll << 26)) { atomicExch(a.stall, 1u); break; }
          __nanosleep(256);
        }
      }
      __syncthreads();
    }
    int64_t p = c0;
    while (p < p_end) {
      int T = (int)(p_end - p < (int64_t)kTile ? p_end - p : (int64_t)kTile);
      // H1 for the tile: one thread per pose; per-pose window row bounds
      int wlo[3] = {INT_MAX, INT_MAX, INT_MAX}, whi[3] = {INT_MIN, INT_MIN, INT_MIN}, wbad = 0;
      if (tid < T) {
        const double* pq = a.poses + 7 * (p + tid);
        double qv[7];
#pragma unroll
        for (int i = 0; i < 7; ++i) qv[i] = __ldg(pq + i);
        double Rm[9];
        const bool ok = quat_rot_dev(qv, Rm);
        PoseRec& pr = s_pose[tid];
#pragma unroll
        for (int i = 0; i < 9; ++i) pr.m[i] = Rm[i];
#pragma unroll
        for (int i = 0; i < 3; ++i) pr.m[9 + i] = qv[4 + i];
        s_ok[tid] = ok ? 1 : 0;
        if (window_mode) {
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            const double t = qv[4 + r];
            if (!isfinite(t)) wbad = 1;
            const double f0 = floor((t - rb + a.b) * a.inv_h) - 1.0;
            const double f1 = floor((t + rb + a.b) * a.inv_h) + 1.0;
            wlo[r] = (int)fmax(0.0, fmin(f0, (double)(a.n - 1)));
            whi[r] = (int)fmax(0.0, fmin(f1, (double)(a.n - 1)));
          }
        }
      }
      bool fits = false;
      if (window_mode) {
        // inclusive block scan of the row bounds over the tile's poses: the tile becomes the
        // longest prefix whose cumulative window fits cap_rows
        if (warp * 32 < T) {             // warps without poses only join the barriers
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            int v[7];
#pragma unroll
            for (int r = 0; r < 3; ++r) {
              v[r] = __shfl_up_sync(kFull, wlo[r], o);
              v[3 + r] = __shfl_up_sync(kFull, whi[r], o);
            }
            v[6] = __shfl_up_sync(kFull, wbad, o);
            if (lane >= o) {
#pragma unroll
              for (int r = 0; r < 3; ++r) {
                wlo[r] = min(wlo[r], v[r]);
                whi[r] = max(whi[r], v[3 + r]);
              }
              wbad |= v[6];
            }
          }
          if (lane == 31) {
#pragma unroll
            for (int r = 0; r < 3; ++r) {
              s_wred[warp][r] = wlo[r];
              s_wred[warp][3 + r] = whi[r];
            }
            s_wred[warp][6] = wbad;
          }
        }
        __syncthreads();
        for (int w = 0; w < warp && warp * 32 < T; ++w) {
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            wlo[r] = min(wlo[r], s_wred[w][r]);
            whi[r] = max(whi[r], s_wred[w][3 + r]);
          }
          wbad |= s_wred[w][6];
        }
        int rows = 0;
#pragma unroll
        for (int r = 0; r < 3; ++r) rows += whi[r] - wlo[r] + 1;
        const bool fit_me = tid < T && !wbad && rows <= cap_rows;
        // fit_me is monotone in tid (cumulative bounds), so the first Tfit poses form the tile
        const int Tfit = __syncthreads_count(fit_me);
        fits = Tfit > 0;
        T = fits ? Tfit : 1;         // a single pose whose rows do not fit takes the L2 path
        // the tile's last thread owns the tile's bounds: it restages the window if needed
        if (tid == T - 1) {
          int rs = 0;
          bool contained = true;
#pragma unroll
          for (int r = 0; r < 3; ++r) contained = contained && s_cur.lo[r] <= wlo[r] && whi[r] <= s_cur.hi[r];
          if (fits && !contained) {
            const int extra = (cap_rows - rows) / 3;
            int row0 = 0;
            unsigned bytes = 0;
            int lo_[3], hi_[3];
#pragma unroll
            const bool all = cap_rows >= 3 * a.n;     // the whole factor set fits
            for (int r = 0; r < 3; ++r) {
              lo_[r] = all ? 0 : max(0, wlo[r] - extra / 2);
              hi_[r] = all ? a.n - 1 : min(a.n - 1, whi[r] + (extra - extra / 2));
              bytes += (unsigned)(hi_[r] - lo_[r] + 1) * kChp * 16;
            }
            // the window was last read through the generic proxy, before the previous barrier
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&s_bar, bytes);
#pragma unroll
            for (int r = 0; r < 3; ++r) {
              s_cur.lo[r] = lo_[r];
              s_cur.hi[r] = hi_[r];
              s_cur.off[r] = row0 - lo_[r];
              const void* src = F32 ? (const void*)(a.t.Fw32[r] + (size_t)lo_[r] * kChp)
                                    : (const void*)(a.t.Fw[r] + (size_t)lo_[r] * kChp);
              tma_load_1d(win + (size_t)row0 * kChp, src,
                          (unsigned)(hi_[r] - lo_[r] + 1) * kChp * 16, &s_bar);
              row0 += hi_[r] - lo_[r] + 1;
            }
            rs = 1;
          }
          s_restaged = rs;
          s_next = 0;
        }
      } else {
        if (tid == 0) {
          s_restaged = 0;
          s_next = 0;
        }
      }
      __syncthreads();
      if (s_restaged) {
        mbar_wait(&s_bar, phase);
        phase ^= 1;
      }
      const Window W = s_cur;
      for (;;) {
        int s = 0;
        if (lane == 0) s = atomicAdd(&s_next, 1);
        s = __shfl_sync(kFull, s, 0);
        if (s >= T) break;
        score_pose<RT, NA, F32>(a, p + s, s_pose[s], s_ok[s] != 0, fits, W, (const char*)win, s_lig, lig_smem_n,
                           lane, s_ps[warp], s_out[s]);
      }
      __syncthreads();
      // H8: d = sqrt(min d^2) below D_cap^2, else +inf; NaN for invalid poses (O8)
      if (tid < T) {
        const double2 o = s_out[tid];
        a.E[p + tid] = o.x;
        a.D[p + tid] = isnan(o.y) ? NAN : (o.y < a.dcap2 ? __dsqrt_rn(o.y) : INFINITY);
      }
      if (a.done) {
        // release the tile's outputs to the copy stream that waits on done[chunk]
        __threadfence();
        __syncthreads();
        if (tid == 0) {
          int c = 0;
          while (c + 1 < a.n_cb && a.cb[c + 1] <= p) ++c;
          int64_t q = p;
          while (q < p + T) {
            const int64_t e = min((int64_t)a.cb[c + 1], p + (int64_t)T);
            atomicAdd(a.done + c, (unsigned)(e - q));
            q = e;
            ++c;
          }
        }
      }
      p += T;
    }
  }
}

struct DevCache {
  int sms = 0;
  int smem_optin = 0;
  bool attr_set[24] = {false};
  int max_dyn[24] = {0};
};
DevCache g_dev[64];

template <int RT, int NA, bool F32>
int launch_t(const ScoreArgs& a, cudaStream_t st, int dev, int slot, bool window_mode) {
  DevCache& dc = g_dev[dev & 63];
  if (!dc.attr_set[slot]) {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, score_kernel<RT, NA, F32>);
    if (e != cudaSuccess) return (int)e;
    dc.max_dyn[slot] = dc.smem_optin - (int)fa.sharedSizeBytes;
    e = cudaFuncSetAttribute(score_kernel<RT, NA, F32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             dc.max_dyn[slot]);
    if (e != cudaSuccess) return (int)e;
    dc.attr_set[slot] = true;
  }
  constexpr int kChp = F32 ? Geo32<(RT > 0 ? RT : 4)>::CHP : Geo<(RT > 0 ? RT : 2)>::CHP;
  const size_t fixed = win_offset<NA>();
  const size_t avail = (size_t)dc.max_dyn[slot] > fixed ? (size_t)dc.max_dyn[slot] - fixed : 0;
  const size_t lig_res = std::min<size_t>(avail, (size_t)std::min<int64_t>(a.L, 256) * sizeof(double4));
  int cap_rows = 0;
  if (RT > 0 && window_mode && (F32 ? (const void*)a.t.Fw32[0] : (const void*)a.t.Fw[0])) {
    cap_rows = (int)std::min<size_t>((avail - lig_res) / (16 * kChp), (1u << 20) / (16 * kChp) - 1);
    if (3 * a.n <= cap_rows) {
      // the whole factor set fits (small grids, e.g. C1): stage it once, every tile fits
      cap_rows = 3 * a.n;
    } else if (a.rmax_hint >= 0) {
      // leave the rest of the 228 KB to L1 (cell lists, records, memo): what one
      // translation's window needs plus RS_WIN_SLACK; no window at all when even one
      // translation's rows do not fit (every pose would be its own tile with its own restage:
      // the L2 path is faster then)
      const double need = 3.0 * (2.0 * (a.rmax_hint + 2.0 * a.h) / a.h + 8.0);
      if (need > cap_rows) cap_rows = 0;
      else cap_rows = std::min(cap_rows, (int)std::max(64.0, RS_WIN_SLACK * need));
    }
  }
  const size_t win_b = (size_t)cap_rows * 16 * kChp;
  const int64_t lig_fit = (int64_t)((avail - std::min(avail, win_b)) / sizeof(double4));
  const int lig_n = (int)std::min<int64_t>(a.L, cap_rows > 0 ? std::min<int64_t>(lig_fit, 256) : lig_fit);
  const size_t dyn = fixed + win_b + (size_t)lig_n * sizeof(double4);
  // chunk plan: big chunks for the first (1 - 1/RS_TAIL_DIV) of the poses, then tail chunks of
  // at most kTailChunk poses, small enough that every SM gets work when P is small
  // (big chunks also shrink with P: at least ~4 per SM, so one chunk never dominates a launch)
  ChunkPlan cp;
  cp.big = (int)std::max<int64_t>(kTailChunk, std::min<int64_t>(kChunk, a.P / (4 * (int64_t)dc.sms)));
  cp.nbig = (a.P - a.P / RS_TAIL_DIV) / cp.big;
  const int64_t rest = a.P - cp.nbig * cp.big;
  cp.tail = (int)std::max<int64_t>(1, std::min<int64_t>(kTailChunk, (rest + 2 * dc.sms - 1) / (2 * dc.sms)));
  const int64_t chunks = cp.nbig + (rest + cp.tail - 1) / cp.tail;
  int grid = (int)std::min<int64_t>(chunks, (int64_t)dc.sms);
  if (grid < 1) grid = 1;
  score_kernel<RT, NA, F32><<<grid, kThreads, dyn, st>>>(a, cap_rows, lig_n, cp);
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
    case 4: return "score_kernel<4, NA>";
    case 8: return "score_kernel<8, NA>";
    case 12: return "score_kernel<12, NA>";
    case 16: return "score_kernel<16, NA>";
    case 24: return "score_kernel<24, NA>";
    case 32: return "score_kernel<32, NA>";
    default: return "score_kernel<0, NA> (runtime R)";
  }
}

int window_row_chunks(int R) {
  switch (R) {
    case 4: return Geo<4>::CHP;
    case 8: return Geo<8>::CHP;
    case 12: return Geo<12>::CHP;
    case 16: return Geo<16>::CHP;
    case 24: return Geo<24>::CHP;
    case 32: return Geo<32>::CHP;
    default: return 0;
  }
}

void pack_window_rows(const std::vector<double>& F, int n, int R, std::vector<double>& out) {
  const int chp = window_row_chunks(R);
  out.assign((size_t)n * chp * 2, 0.0);
  if (chp == 0) return;
  const int ch = R / 2;
  const bool rep = (ch == 1 || ch == 2 || ch == 4);   // replicated widths repeat the row
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < chp; ++c) {
      const int src = rep ? (c % ch) : c;
      if (src >= ch) continue;                           // padded widths: zero chunks
      out[((size_t)i * chp + c) * 2] = F[(size_t)i * R + 2 * src];
      out[((size_t)i * chp + c) * 2 + 1] = F[(size_t)i * R + 2 * src + 1];
    }
}

int window_row_chunks32(int R) {
  switch (R) {
    case 4: return Geo32<4>::CHP;
    case 8: return Geo32<8>::CHP;
    case 12: return Geo32<12>::CHP;
    case 16: return Geo32<16>::CHP;
    case 24: return Geo32<24>::CHP;
    case 32: return Geo32<32>::CHP;
    default: return 0;
  }
}

void pack_window_rows32(const std::vector<double>& F, int n, int R, std::vector<float>& out) {
  const int chp = window_row_chunks32(R);
  out.assign((size_t)n * chp * 4, 0.0f);
  if (chp == 0) return;
  int cha = 1;
  while (4 * cha < R) cha *= 2;                       // quads incl. zero padding (A21)
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < chp; ++c)
      for (int t = 0; t < 4; ++t) {
        const int k = 4 * (c % cha) + t;              // replicated when cha < chp
        out[((size_t)i * chp + c) * 4 + t] = k < R ? (float)F[(size_t)i * R + k] : 0.0f;
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
    const double row_b = a.f32 ? 128.0 : 16.0 * (a.R <= 8 ? 8 : ((a.R / 2 + 7) / 8) * 8);
    window_mode = rows * row_b <= 0.75 * double(dc.smem_optin);
  }
  // one atom per lane and pass (NA = 2, two independent chains per lane, needs the registers
  // of a 512-thread CTA and measured slower than 32 resident warps with NA = 1)
#ifdef RS_FORCE_NA
  const int na = RS_FORCE_NA, sl = na == 2 ? 8 : 0;
#else
  const int na = (kThreads <= 512 && a.L > 32) ? 2 : 1, sl = na == 2 ? 8 : 0;
#endif
  int e;
  if (a.f32) {
    // binary32 factors (A21): compiled widths only (the build refuses others)
    switch (a.R) {
      case 4: e = launch_t<4, 1, true>(a, st, device, 17, window_mode); break;
      case 8: e = launch_t<8, 1, true>(a, st, device, 18, window_mode); break;
      case 12: e = launch_t<12, 1, true>(a, st, device, 19, window_mode); break;
      case 16: e = launch_t<16, 1, true>(a, st, device, 20, window_mode); break;
      case 24: e = launch_t<24, 1, true>(a, st, device, 21, window_mode); break;
      case 32: e = launch_t<32, 1, true>(a, st, device, 22, window_mode); break;
      default: return (int)cudaErrorInvalidValue;
    }
  } else if (kThreads <= 512 && na == 2) {
    switch (a.R) {
      case 4: e = launch_t<4, 2, false>(a, st, device, 9, window_mode); break;
      case 8: e = launch_t<8, 2, false>(a, st, device, 10, window_mode); break;
      case 12: e = launch_t<12, 2, false>(a, st, device, 11, window_mode); break;
      case 16: e = launch_t<16, 2, false>(a, st, device, 12, window_mode); break;
      case 24: e = launch_t<24, 2, false>(a, st, device, 13, window_mode); break;
      case 32: e = launch_t<32, 2, false>(a, st, device, 14, window_mode); break;
      default: e = launch_t<0, 2, false>(a, st, device, 8, false); break;
    }
  } else {
    switch (a.R) {
      case 4: e = launch_t<4, 1, false>(a, st, device, 1, window_mode); break;
      case 8: e = launch_t<8, 1, false>(a, st, device, 2, window_mode); break;
      case 12: e = launch_t<12, 1, false>(a, st, device, 3, window_mode); break;
      case 16: e = launch_t<16, 1, false>(a, st, device, 4, window_mode); break;
      case 24: e = launch_t<24, 1, false>(a, st, device, 5, window_mode); break;
      case 32: e = launch_t<32, 1, false>(a, st, device, 6, window_mode); break;
      default: e = launch_t<0, 1, false>(a, st, device, 0, false); break;
    }
  }
  if (launches) *launches += 1;
  return e;
}

}  // namespace rs
