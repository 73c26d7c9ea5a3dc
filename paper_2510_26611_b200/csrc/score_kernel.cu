// Fused sm_100a pose-scoring kernel: Algorithm PLIE with Lemma 3.2 /
// Eq. (18), the RS entry formula and the vdW constraint
// of Eq. (22).  Rows H1-H8 of SURVEY.md §8(a), in one pass:
//   H1 quaternion -> rotation      H2 x' = R y + t           H3 snap to the cell grid
//   H4 long-range CP gather + rank sum (rows of F_0, F_1, F_2 from a shared-memory window
//      or from L2)                  H5 short-range replicas of nearby protein atoms
//   H6 vdW min distance over the same cell-list candidates
//   H7 double-double reduction      H8 one energy + one min distance per pose
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
// Work layout: persistent CTAs (one per SM) take chunks of consecutive poses
// from a global counter (guided: smaller chunks over the last poses).  A tile is the longest
// run of a chunk's poses whose factor rows fit the shared-memory window (a block scan of
// per-pose row bounds); the window's rows of the three factor matrices arrive by TMA bulk
// copies (cp.async.bulk, mbarrier completion) from a row-padded device copy, and the tile's
// coarse cells of the neighbour lists are copied into a local range table next to it.
// Warps take UNITS of the tile's poses: G poses (a power of two <= 32, guided so that the
// warps finish a tile together) with S = 32/G lanes per pose; a lane keeps its pose's R and t
// in registers and walks the ligand atoms l = sub, sub + S, ... (sub = lane mod S) through
// H2-H6, so a full unit (G = 32) is one pose per lane and needs no cross-lane reduction.
// Rows are 16-byte chunks padded (R=12, 24) or replicated (R=4, 8) to whole 128-byte lines;
// lane l reads chunk c ^ (l & 7) of its own row in slot c, so the 8 lanes of every
// quarter-warp hit 8 distinct bank groups whatever rows they gather (conflict-free LDS.128);
// the halving tree over rank pairs is invariant under that relabelling, so no un-permute is
// needed.  RS_FLAG_F32_FACTORS (reading A21) runs the same machinery on binary32 rank quads.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

#include "rs_internal.h"
#include "rs_device.cuh"

namespace rs {
namespace {

using namespace dev;

#ifndef RS_THREADS
#define RS_THREADS 512
#endif
#ifndef RS_CHUNK
#define RS_CHUNK 2048
#endif
#ifndef RS_WIN_SLACK
#define RS_WIN_SLACK 1.5
#endif
#ifndef RS_LOC_CELLS
#define RS_LOC_CELLS 10240
#endif
#ifndef RS_L2_CG
#define RS_L2_CG 1     // L2-path launches gather rows with ld.global.cg (L2 only)
#endif
constexpr int kThreads = RS_THREADS;
constexpr int kWarps = kThreads / 32;
constexpr int kTile = 2 * kThreads;      // poses per tile (upper bound): two per thread in the scan
constexpr int kChunk = RS_CHUNK;         // poses per unit of dynamic CTA work
#ifndef RS_TAIL_DIV
#define RS_TAIL_DIV 8
#endif
#ifndef RS_TAIL_CHUNK
#define RS_TAIL_CHUNK 256
#endif
constexpr int kMinBig = 128;               // smallest big chunk (small batches: C5's 10^5 poses)
constexpr int kTailChunk = RS_TAIL_CHUNK;  // chunk size over the last 1/RS_TAIL_DIV of the poses
constexpr unsigned kFull = 0xffffffffu;

template <int R>
struct Geo {
  static constexpr int CH = R / 2;                                 // 16-byte chunks of a row
  static constexpr bool REP = (CH == 1 || CH == 2 || CH == 4);      // replicate to 128 B
  static constexpr int CHP = REP ? 8 : ((CH + 7) / 8) * 8;         // physical chunks per row
  static constexpr int NS = REP ? CH : CHP;                        // loads per row and lane
};

// Read-only global loads issued only when pr holds (the predicate is inside the instruction, so
// the compiler cannot turn a guarded load into an unguarded speculative one: the address may be
// meaningless when pr is false, and untaken lanes cost no L1 tag lookups).  Result 0 if !pr.
__device__ __forceinline__ double ldg_if(const double* p, bool pr) {
  double v = 0.0;
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.global.nc.f64 %0, [%1];\n}"
      : "+d"(v) : "l"(p), "r"((int)pr));
  return v;
}
// one 256-bit load of a factor row sector on the L2 path (a whole 32-byte sector per lane).
// CG: ld.global.cg, cached in L2 only (rows of random cells miss L1 anyway: 1-4 % hit rate at
// C4/C5; the L2-only gather measures 13 % faster, tools/microbench); else ld.global.nc
// (LDG.E.ENL2.256.CONSTANT, L1-allocating: the window kernels' rare out-of-window poses)
template <bool CG>
__device__ __forceinline__ double4 ldg256(const double4* p) {
  double4 v;
  if constexpr (CG)
    asm("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  else
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
template <bool CG = false>
__device__ __forceinline__ float4 ldg256x2(const float4* p, float4& hi) {
  float4 v;
  if constexpr (CG)
    asm("ld.global.cg.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w), "=f"(hi.x), "=f"(hi.y), "=f"(hi.z), "=f"(hi.w)
        : "l"(p));
  else
    asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w), "=f"(hi.x), "=f"(hi.y), "=f"(hi.z), "=f"(hi.w)
        : "l"(p));
  return v;
}
// a scalar / 16-byte L2-path load: ld.global.cg when CG (L2 only), else the read-only path
template <bool CG>
__device__ __forceinline__ double ldg_l2(const double* p) {
  double v;
  if constexpr (CG) asm("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else v = __ldg(p);
  return v;
}
template <bool CG>
__device__ __forceinline__ float4 ldg_l2(const float4* p) {
  float4 v;
  if constexpr (CG)
    asm("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  else v = __ldg(p);
  return v;
}
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
// two consecutive 16-byte list entries (a 32-byte aligned pair) in one 256-bit load
__device__ __forceinline__ void ldg_pair_if(const int4* p, bool pr, int4& e0, int4& e1) {
  e0 = make_int4(0, 0, 0, 0);
  e1 = e0;
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %9, 0;\n"
      " @q ld.global.nc.v8.s32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n}"
      : "+r"(e0.x), "+r"(e0.y), "+r"(e0.z), "+r"(e0.w), "+r"(e1.x), "+r"(e1.y), "+r"(e1.z), "+r"(e1.w)
      : "l"(p), "r"((int)pr));
}
// Predicated loads whose outputs are left undefined when the predicate is off (the caller
// never reads them then): no zero-initialisation instructions on the hot neighbour path
#ifndef RS_ENT_CG
#define RS_ENT_CG 1    // list entries with ld.global.cg (L2 only: measured 1.3 % faster at C3)
#endif
#ifndef RS_MEMO_CG
#define RS_MEMO_CG 1   // short-range memo values with ld.global.cg (L2 only)
#endif
__device__ __forceinline__ void ldg_pair_p(const int4* p, bool pr, int4& e0, int4& e1) {
#if RS_ENT_CG
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %9, 0;\n"
      " @q ld.global.cg.v8.s32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n}"
      : "=r"(e0.x), "=r"(e0.y), "=r"(e0.z), "=r"(e0.w), "=r"(e1.x), "=r"(e1.y), "=r"(e1.z), "=r"(e1.w)
      : "l"(p), "r"((int)pr));
#else
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %9, 0;\n"
      " @q ld.global.nc.v8.s32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n}"
      : "=r"(e0.x), "=r"(e0.y), "=r"(e0.z), "=r"(e0.w), "=r"(e1.x), "=r"(e1.y), "=r"(e1.z), "=r"(e1.w)
      : "l"(p), "r"((int)pr));
#endif
}
__device__ __forceinline__ int4 ldg_int4_p(const int4* p, bool pr) {
  int4 v;
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %5, 0;\n @q ld.global.nc.v4.s32 {%0, %1, %2, %3}, [%4];\n}"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "r"((int)pr));
  return v;
}
#ifndef RS_REC_CG
#define RS_REC_CG 0    // protein records with ld.global.cg (L2 only)
#endif
__device__ __forceinline__ double4 ldg_d4_p(const double4* p, bool pr) {
  double4 v;
#if RS_REC_CG
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %5, 0;\n @q ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];\n}"
      : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p), "r"((int)pr));
#else
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %5, 0;\n @q ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];\n}"
      : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p), "r"((int)pr));
#endif
  return v;
}
__device__ __forceinline__ double ldg_d_p(const double* p, bool pr) {
  double v;
#if RS_MEMO_CG
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.global.cg.f64 %0, [%1];\n}"
      : "=d"(v) : "l"(p), "r"((int)pr));
#else
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.global.nc.f64 %0, [%1];\n}"
      : "=d"(v) : "l"(p), "r"((int)pr));
#endif
  return v;
}
// 16 bytes from shared memory at a 32-bit shared-window address
__device__ __forceinline__ double2 lds2(unsigned addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ float4 lds4f(unsigned addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ unsigned lds_u32(unsigned addr) {
  unsigned v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// O4 with compile-time R from the shared-memory window.  rK = shared address of row K with the
// lane's XOR offset rho << 4 already in bits 4.. (rows are 128/256-byte aligned, so XOR with
// c << 4 selects physical chunk c ^ rho of the row).  Physical chunk p holds pair p (padded
// widths: zero beyond CH; replicated widths: pair p mod CH), so slot c holds pair (c ^ rho)
// mod NS, and the halving tree, which combines c with c ^ m at every level, is bitwise
// invariant under that relabelling.  Evaluated depth-first: T(c, stride, cnt) = T(c, 2 stride,
// cnt/2) + T(c + stride, 2 stride, cnt/2), leaves = slot pair sums (the pairings of the
// level-by-level loop: pair c meets c + NS/2 first), so partial sums retire as their chunks
// arrive and fewer values are live while the gathers are in flight.
template <int C, int STRIDE, int CNT>
struct SmemTree {
  static __device__ __forceinline__ double eval(unsigned r0, unsigned r1, unsigned r2) {
    if constexpr (CNT == 1) {
      constexpr unsigned o = (unsigned)C << 4;
      return pair_prod(lds2(r0 ^ o), lds2(r1 ^ o), lds2(r2 ^ o));
    } else {
      const double lhs = SmemTree<C, 2 * STRIDE, CNT / 2>::eval(r0, r1, r2);
      const double rhs = SmemTree<C + STRIDE, 2 * STRIDE, CNT / 2>::eval(r0, r1, r2);
      return __dadd_rn(lhs, rhs);
    }
  }
};

// O4 with compile-time R from L2 (unpadded n x R rows); slot c = pair c (no bank structure)
template <int R, bool CG = false>
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
      const double4 a = ldg256<CG>(q0 + c), b = ldg256<CG>(q1 + c), cc = ldg256<CG>(q2 + c);
      s[2 * c] = pair_prod(make_double2(a.x, a.y), make_double2(b.x, b.y), make_double2(cc.x, cc.y));
      s[2 * c + 1] = pair_prod(make_double2(a.z, a.w), make_double2(b.z, b.w), make_double2(cc.z, cc.w));
    }
  }
  return halving_tree<C>(s);
}

// O4 with a runtime R (generic widths, e.g. tolerance-mode builds): rows from L2, the same
// pairwise halving tree over rank pairs.  The tree is walked depth-first: its leaves in order
// are the pairs c = bitrev(j), j = 0..C-1, merged with a binary-counter stack (depth log2 C).
template <bool CG = false>
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
    if (2 * c < R)
      q0 = __dmul_rn(__dmul_rn(ldg_l2<CG>(r0 + 2 * c), ldg_l2<CG>(r1 + 2 * c)), ldg_l2<CG>(r2 + 2 * c));
    if (2 * c + 1 < R)
      q1 = __dmul_rn(__dmul_rn(ldg_l2<CG>(r0 + 2 * c + 1), ldg_l2<CG>(r1 + 2 * c + 1)), ldg_l2<CG>(r2 + 2 * c + 1));
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
  static __device__ __forceinline__ float eval(unsigned r0, unsigned r1, unsigned r2) {
    if constexpr (CNT == 1) {
      constexpr unsigned o = (unsigned)C << 4;
      return quad_prod(lds4f(r0 ^ o), lds4f(r1 ^ o), lds4f(r2 ^ o));
    } else {
      const float lhs = SmemTree32<C, 2 * STRIDE, CNT / 2>::eval(r0, r1, r2);
      const float rhs = SmemTree32<C + STRIDE, 2 * STRIDE, CNT / 2>::eval(r0, r1, r2);
      return __fadd_rn(lhs, rhs);
    }
  }
};

// L2 path of O4-f32: rows of the packed binary32 copy, quads in natural order
template <int R, bool CG = false>
__device__ __forceinline__ double long_phi_l2_32(const float4* F0, const float4* F1,
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
        const float4 a0 = ldg256x2<CG>(r0 + c, a1), b0 = ldg256x2<CG>(r1 + c, b1), c0 = ldg256x2<CG>(r2 + c, c1);
        s[c] = quad_prod(a0, b0, c0);
        s[c + 1] = quad_prod(a1, b1, c1);
      } else if (c < G::CH) {
        s[c] = quad_prod(ldg_l2<CG>(r0 + c), ldg_l2<CG>(r1 + c), ldg_l2<CG>(r2 + c));
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
template <int R>
__device__ __noinline__ double long_phi_global32(const float4* F0, const float4* F1,
                                                 const float4* F2, int i0, int i1, int i2) {
  return long_phi_l2_32<R>(F0, F1, F2, i0, i1, i2);
}

// O4-T (NEXT row N5, reading A26): phi = sum_a u0[a] (sum_b u1[b] (sum_c G[a][b][c] u2[c])),
// each sum an ascending chain of rounded products and sums (the oracle's order), u_l the rows
// of the RHOSVD bases at the atom's cells (from L2), G from shared memory; r_l <= 32 (u2 held
// in registers, the c loop unrolled and predicated)
constexpr int kTkMax = 32;
__device__ __noinline__ double tucker_phi(const ScoreArgs& a, int i0, int i1, int i2, const double* G) {
  const int r0 = a.tr[0], r1 = a.tr[1], r2 = a.tr[2];
  const double* u0 = a.t.Ut[0] + (size_t)i0 * r0;
  const double* u1 = a.t.Ut[1] + (size_t)i1 * r1;
  const double* u2 = a.t.Ut[2] + (size_t)i2 * r2;
  double w[kTkMax];
#pragma unroll
  for (int c = 0; c < kTkMax; ++c) w[c] = c < r2 ? __ldg(u2 + c) : 0.0;
  double phi = 0.0;
  for (int x = 0; x < r0; ++x) {
    double t = 0.0;
    for (int y = 0; y < r1; ++y) {
      const double* g = G + ((size_t)x * r1 + y) * r2;
      double v = 0.0;
#pragma unroll
      for (int c = 0; c < kTkMax; ++c)
        if (c < r2) v = __dadd_rn(v, __dmul_rn(g[c], w[c]));
      t = __dadd_rn(t, __dmul_rn(__ldg(u1 + y), v));
    }
    phi = __dadd_rn(phi, __dmul_rn(__ldg(u0 + x), t));
  }
  return phi;
}

struct ChunkPlan {             // dynamic schedule: nbig chunks of `big` poses, then `tail`-pose chunks
  int64_t nbig;
  int big, tail;
};

struct Window {
  int lo[3], hi[3], off[3];    // staged rows [lo, hi] per axis; smem row of row i = i + off
};
struct LocalBox {              // coarse cells [lo, lo + dim) per axis copied into s_loc; dim 0: none
  int lo[3], dim[3];
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
__device__ __forceinline__ void tma_load_1d(unsigned dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
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

// O5 value s(D) from the dense memo s(|D0|,|D1|,|D2|), which the handle fills on the device with
// the O5 chain itself (ascending k) for every |D_a| <= n_sigma; loaded only when pr holds
__device__ __forceinline__ double short_value(const ScoreArgs& a, int e0, int e1, int e2, bool pr) {
  const unsigned d = (unsigned)a.n_sigma + 1u;
  const unsigned idx = ((unsigned)abs(e0) * d + (unsigned)abs(e1)) * d + (unsigned)abs(e2);
  RS_DCHECK(!pr || (abs(e0) <= a.n_sigma && abs(e1) <= a.n_sigma && abs(e2) <= a.n_sigma && idx < d * d * d));
  return ldg_d_p(reinterpret_cast<const double*>(reinterpret_cast<uintptr_t>(a.t.short_memo) +
                                                 (uint64_t)idx * 8u), pr);
}

// One candidate list entry en = (i0 | i1 << 15 | (k & 3) << 30, i2 | (k >> 2) << 15, q) against
// the atom's cell (c0, c1, c2): the squared integer offset (cells are < 2^15, so it sums
// exactly in 32 bits)
__device__ __forceinline__ unsigned entry_dd(int c0, int c1, int c2, const int4 en, int& e0, int& e1,
                                             int& e2) {
  e0 = c0 - (en.x & 0x7fff);
  e1 = c1 - (int)(((unsigned)en.x >> 15) & 0x7fffu);
  e2 = c2 - (en.y & 0x7fff);
  return (unsigned)(e0 * e0) + (unsigned)(e1 * e1) + (unsigned)(e2 * e2);
}
__device__ __forceinline__ unsigned entry_k(const int4 en) {   // the sorted atom index
  return (((unsigned)en.y >> 15) << 2) | ((unsigned)en.x >> 30);
}
__device__ __forceinline__ double entry_q(const int4 en) {     // the atom's charge z_m
  return __hiloint2double(en.w, en.z);
}

// H6 for one candidate with record r (loaded iff hit): O7 distance, keep the minimum
__device__ __forceinline__ void pair_hit(double x0, double x1, double x2, const double4 r, bool hit,
                                         double& best) {
  const double dx0 = __dsub_rn(x0, r.x);
  const double dx1 = __dsub_rn(x1, r.y);
  const double dx2 = __dsub_rn(x2, r.z);
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx0, dx0), __dmul_rn(dx1, dx1)), __dmul_rn(dx2, dx2));
  best = (hit && d2 < best) ? d2 : best;
}

// The integer prefilter of H6 tightened to the lane's running minimum: a pair with
// |x_l - x_m|^2 < best has |D| <= |x_l - x_m| inv_h + sqrt 3 cells, so only entries with
// |D|^2 below ceil((sqrt(best) inv_h + sqrt 3 + 2)^2) (the static bound's 2-cell margin) can
// lower it; capped at the static bound vdw_cells2 (D_cap).  The minimum is order-free (O7), so
// skipping the others changes no result.
#ifndef RS_DYN_THR
#define RS_DYN_THR 2   // 0: static D_cap bound only; 1: fp64 sqrt; 2: binary32 bound (rounded up)
#endif
__device__ __forceinline__ unsigned vdw_thr(const ScoreArgs& a, double best) {
#if RS_DYN_THR == 1
  const double t = __dadd_rn(__dmul_rn(__dsqrt_rn(best), a.inv_h), 3.7320508075688772);
  const double t2 = __dmul_rn(t, t);
  return t2 < (double)a.vdw_cells2 ? (unsigned)ceil(t2) + 1u : a.vdw_cells2;
#else
  // (sqrt(best) inv_h + sqrt 3 + 2)^2 <= thr_a best + thr_b (host: AM-GM, rounded up), in
  // binary32 with every step rounded up: no square root on the hot path
  const float t2 = __fadd_ru(__fmul_ru(__double2float_ru(best), a.thr_a), a.thr_b);
  return t2 < (float)a.vdw_cells2 ? (unsigned)t2 + 2u : a.vdw_cells2;
#endif
}

#ifndef RS_EARLY_STOP
#define RS_EARLY_STOP 1
#endif
// Early end of a candidate walk.  Every list is sorted by key = |2 i_m - C|^2 (half cells, C
// the coarse cell's centre; rs_build_protein).  With rho^2 = max(ns2, vthr), A = 2 a - C for
// the atom's cell a (|A_r| <= 2^s - 1) and delta = |A|, an entry the walk still needs
// (|i_m - a| <= rho) has key <= (2 rho + delta)^2: the walk ends at the first entry with
// key - 4 rho^2 - delta^2 > 4 rho delta, tested exactly in integers (both sides squared).  The
// atom's own offset from the centre instead of the worst case (2^s - 1) sqrt 3 cuts the walked
// entries by about a fifth at C3.  stop_key returns 4 rho^2 (saturated: no early end when it
// does not fit 32 bits).
__device__ __forceinline__ unsigned stop_key(const ScoreArgs& a, unsigned vthr) {
  const unsigned m = max(a.ns2, vthr);
  // (coarse cells of more than 2^12 cells would overflow the 64-bit product of the test)
  return (m < 0x40000000u && a.nb_shift <= 12) ? 4u * m : 0xffffffffu;
}

#ifndef RS_DEFER_BALL
#define RS_DEFER_BALL 0
#endif
#ifndef RS_VOTE_MASK
#define RS_VOTE_MASK 1
#endif
#ifndef RS_TILE_OVERLAP
#define RS_TILE_OVERLAP 1
#endif
#ifndef RS_LIG_CALL
#define RS_LIG_CALL 1   // 1: ligand atoms beyond the staged ones through an out-of-line load
#endif
// O5 terms of a round whose memo values are still in flight: added one round later
struct BallPending {
  double q0, q1, sv0, sv1, z;
  int f;   // bit 0 / 1: entry 0 / 1 is inside the n_sigma ball
};
__device__ __forceinline__ void ball_flush(BallPending& pd, double& hi, double& lo) {
  if (pd.f & 1) dd_add_prod(hi, lo, pd.z, __dmul_rn(pd.q0, pd.sv0));
  if (pd.f & 2) dd_add_prod(hi, lo, pd.z, __dmul_rn(pd.q1, pd.sv1));
  pd.f = 0;
}

// H5 + H6 for two candidate list entries of one ligand atom (cell c0..c2, coordinates
// x0..x2, charge z); a0/a1: the entries are real candidates.  The integer prefilter on the
// cell offset decides whether the memo value (O5 replica term inside the n_sigma ball, with
// the charge from the entry) and the protein record (O7 distance, only while the pair can
// still lower the lane's minimum: vthr) are loaded at all.
__device__ __forceinline__ void nbr_pair(const ScoreArgs& a, double x0, double x1, double x2,
                                         double z, int c0, int c1, int c2, const int4 en0,
                                         const int4 en1, bool a0, bool a1, double& hi, double& lo,
                                         double& best, unsigned vthr, unsigned stopk, bool& end,
                                         BallPending& pd) {
  int e00, e01, e02, e10, e11, e12;
  unsigned dd0 = entry_dd(c0, c1, c2, en0, e00, e01, e02);
  unsigned dd1 = entry_dd(c0, c1, c2, en1, e10, e11, e12);
#if RS_EARLY_STOP
  {
    const int msk = (1 << a.nb_shift) - 1;
    const int A0 = 2 * (c0 & msk) - msk, A1 = 2 * (c1 & msk) - msk, A2 = 2 * (c2 & msk) - msk;
    const int k0 = A0 - 2 * e10, k1 = A1 - 2 * e11, k2 = A2 - 2 * e12;   // 2 i_m - C
    const unsigned key = (unsigned)(k0 * k0) + (unsigned)(k1 * k1) + (unsigned)(k2 * k2);
    const unsigned d2 = (unsigned)(A0 * A0) + (unsigned)(A1 * A1) + (unsigned)(A2 * A2);
    const unsigned t = key - stopk, u = t - d2;
    end = a1 && key > stopk && t > d2 &&
          (unsigned long long)u * u > (((unsigned long long)stopk * d2) << 2);
  }
#else
  end = false;
#endif
  dd0 = a0 ? dd0 : 0xffffffffu;
  dd1 = a1 ? dd1 : 0xffffffffu;
  const bool sr0 = dd0 <= a.ns2, sr1 = dd1 <= a.ns2;
  const bool v0 = dd0 < vthr, v1 = dd1 < vthr;
  RS_DCHECK(!v0 || entry_k(en0) < (unsigned)a.n_prot);
  RS_DCHECK(!v1 || entry_k(en1) < (unsigned)a.n_prot);
  const double4 rc0 = ldg_d4_p(a.t.prec + entry_k(en0), v0);
  const double4 rc1 = ldg_d4_p(a.t.prec + entry_k(en1), v1);
  const double sv0 = short_value(a, e00, e01, e02, sr0);
  const double sv1 = short_value(a, e10, e11, e12, sr1);
  pair_hit(x0, x1, x2, rc0, v0, best);
  pair_hit(x0, x1, x2, rc1, v1, best);
#if RS_DEFER_BALL
  // the O5 terms wait for the next round (their memo values land behind the atom step)
  pd.q0 = entry_q(en0); pd.q1 = entry_q(en1); pd.sv0 = sv0; pd.sv1 = sv1; pd.z = z;
  pd.f = (sr0 ? 1 : 0) | (sr1 ? 2 : 0);
#else
  if (sr0) dd_add_prod(hi, lo, z, __dmul_rn(entry_q(en0), sv0));
  if (sr1) dd_add_prod(hi, lo, z, __dmul_rn(entry_q(en1), sv1));
#endif
}

#ifndef RS_NQ
#define RS_NQ 3
#endif
constexpr int kNQ = RS_NQ;   // per-lane stack of atoms waiting for their candidate walk

#ifndef RS_QCOMPACT
#define RS_QCOMPACT 0
#endif
#ifndef RS_LIG_OUTER
#define RS_LIG_OUTER 1
#endif
// Per-warp neighbour queues: atoms whose candidates a lane has not started yet
#if RS_QCOMPACT
// (atom, first entry, end entry): x' and the cell are recomputed from the lane's pose when the
// atom is popped (the same H2/H3 op sequence, so bitwise the values the atom step had)
struct __align__(16) NbrQueue {
  int4 cb[kNQ][32];
};
#else
struct __align__(16) NbrQueue {
  double2 x01[kNQ][32];   // x'_0, x'_1
  double2 x2z[kNQ][32];   // x'_2, charge
  int4 cb[kNQ][32];       // i0 | i1 << 16, i2, first entry, end entry
};
#endif


constexpr size_t kQueueBytes = sizeof(NbrQueue) * kWarps;   // dynamic shared memory

// ligand atom lc from global memory (atoms beyond the shared-memory staging): out of line, so the
// staged case pays one branch instead of the predicated-off loads
__device__ __noinline__ double4 lig_atom_global(const double* __restrict__ yl,
                                                const double* __restrict__ zl, int lc) {
  return make_double4(__ldg(yl + 3 * (int64_t)lc), __ldg(yl + 3 * (int64_t)lc + 1),
                      __ldg(yl + 3 * (int64_t)lc + 2), __ldg(zl + lc));
}

__device__ __forceinline__ int pow2_floor(int v) {   // v >= 1
  return 1 << (31 - __clz(v));
}

// ---- the fused kernel ---------------------------------------------------------------------
//
// RT: compiled CP width (0 = runtime width, L2 rows).  F32: binary32 rows (A21).  WIN: the
// shared-memory window is used (else every atom reads its rows from L2).
template <int RT, bool F32, bool WIN>
__global__ void __launch_bounds__(kThreads, 1) score_kernel(const ScoreArgs a, int cap_rows,
                                                            int lig_smem_n, int loc_cap,
                                                            const ChunkPlan cp,
                                                            const __grid_constant__ CUtensorMap tmap,
                                                            int loc_cd) {
  // dynamic shared memory: [factor-row window, 256-B aligned][local range table][ligand]
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  constexpr int kChp = F32 ? Geo32<(RT > 0 ? RT : 4)>::CHP : Geo<(RT > 0 ? RT : 2)>::CHP;
  constexpr unsigned kRow = 16u * kChp;
  const unsigned raw_u32 = smem_u32(smem_raw);
  const unsigned win_u32 = (raw_u32 + 255u) & ~255u;
  const unsigned loc_u32 = win_u32 + (unsigned)cap_rows * kRow;
  unsigned char* loc_g = smem_raw + (loc_u32 - raw_u32);
  unsigned* s_loc = reinterpret_cast<unsigned*>(loc_g);   // per coarse cell: begin | count << 24
  NbrQueue* s_nq = reinterpret_cast<NbrQueue*>(loc_g + (size_t)loc_cap * sizeof(unsigned));
  double2* s_lig = reinterpret_cast<double2*>(loc_g + (size_t)loc_cap * sizeof(unsigned) + kQueueBytes);
  __shared__ int s_wred[kWarps][8];
  __shared__ Window s_cur;
  __shared__ LocalBox s_lb;
  __shared__ int s_next, s_restaged, s_chunk;
  __shared__ double s_rmax2[kWarps];
  __shared__ __align__(8) uint64_t s_bar;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ligand radius (body frame) and staging: (y0, y1) then (y2, z), structure-of-arrays
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
#if RS_LIG_OUTER
  // atoms in descending |y| (ties: lower index first): the outer atoms, which meet the protein,
  // come first, so their queued candidate walks overlap the inner atoms' steps instead of a
  // drain after the last atom (the O6 sums are order-free)
  if (a.L > 1 && a.L <= lig_smem_n && a.L <= kThreads) {
    __syncthreads();
    double4* tmp = reinterpret_cast<double4*>(s_nq);   // the queues are unused until the units
    if (tid < a.L) {
      const double2 v0 = s_lig[tid], v1 = s_lig[lig_smem_n + tid];
      const double r = v0.x * v0.x + v0.y * v0.y + v1.x * v1.x;
      int rk = 0;
      for (int j = 0; j < (int)a.L; ++j) {
        const double2 w0 = s_lig[j], w1 = s_lig[lig_smem_n + j];
        const double rj = w0.x * w0.x + w0.y * w0.y + w1.x * w1.x;
        rk += (rj > r || (rj == r && j < tid)) ? 1 : 0;
      }
      tmp[rk] = make_double4(v0.x, v0.y, v1.x, v1.y);
    }
    __syncthreads();
    if (tid < a.L) {
      const double4 v = tmp[tid];
      s_lig[tid] = make_double2(v.x, v.y);
      s_lig[lig_smem_n + tid] = make_double2(v.z, v.w);
    }
  }
#endif
  if (tid == 0) {
    s_cur.lo[0] = s_cur.lo[1] = s_cur.lo[2] = 1;
    s_cur.hi[0] = s_cur.hi[1] = s_cur.hi[2] = 0;   // empty
    s_cur.off[0] = s_cur.off[1] = s_cur.off[2] = 0;
    s_lb.dim[0] = s_lb.dim[1] = s_lb.dim[2] = 0;
    s_lb.lo[0] = s_lb.lo[1] = s_lb.lo[2] = 0;
    mbar_init(&s_bar);
  }
  // N5 (RT < 0): the Tucker core in shared memory behind the ligand (every lane reads the same
  // core entry at the same step: broadcast loads)
  double* s_tg = reinterpret_cast<double*>(s_lig + 2 * (size_t)lig_smem_n);
  if constexpr (RT < 0) {
    const int ng = a.tr[0] * a.tr[1] * a.tr[2];
    for (int t = tid; t < ng; t += kThreads) s_tg[t] = __ldg(a.t.TG + t);
  }
  __syncthreads();
  double rmax2 = 0.0;
  for (int w = 0; w < kWarps; ++w) rmax2 = fmax(rmax2, s_rmax2[w]);
  // slack: |R y| <= |y| (1 + 1e-15) plus two cells for the snap rounding and the clamp
  const double rb = sqrt(rmax2) * (1.0 + 1e-12) + 2.0 * a.h;
  const bool window_mode = WIN && RT > 0 && cap_rows > 0;
  const int L = (int)a.L;
  const bool lig_all_smem = L <= lig_smem_n;
  // smallest unit of a tile's tail: at most ~L/6 lanes per pose, so a lane keeps >= ~6 atoms
  // (C3's 60 and C2's 50 atoms: units of >= 4 poses; C5's 5,000-atom partner: down to single
  // poses).  Smaller units lose more in H1 and the drain of their walks than idle warps cost:
  // lowering the floor for tiles too small to give every warp a unit measured +2.4 % at C3
  const int min_unit = 32 / pow2_floor(max(1, min(32, L / 6)));
  const int nm1 = a.n - 1;
  const unsigned rho16 = (unsigned)(lane & 7) << 4;
  unsigned phase = 0;

  // dynamic chunks of consecutive poses (a global work counter): the neighbour work per pose
  // varies by an order of magnitude between translations, so static ranges leave the busiest
  // SM 2-3x behind the mean
  for (;;) {
    if (tid == 0) s_chunk = atomicAdd(a.work, 1);
    __syncthreads();
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
        // bounded by wall time (%globaltimer, ns): if the copy engine does not run beside the
        // kernel (MPS, a sanitizer, a busy engine) the launch gives up once, flags the stall
        // and the host recomputes the batch without streaming
        unsigned v = 0;
        unsigned long long t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (;;) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.arrive + c) : "memory");
          if (v != 0) break;
          if (*(volatile const unsigned*)a.stall != 0u) break;   // another CTA gave up already
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
          if (t - t0 > 2000000000ull) { atomicExch(a.stall, 1u); break; }
          __nanosleep(256);
        }
      }
      __syncthreads();
    }
    int64_t p = c0;
    while (p < p_end) {
      int T = (int)(p_end - p < (int64_t)kTile ? p_end - p : (int64_t)kTile);
      bool fits = false;
      if (window_mode) {
        // per-pose window row bounds t +- rb (thread tid: poses 2 tid, 2 tid + 1), then an
        // inclusive block scan over the tile's poses: the tile becomes the longest prefix whose
        // cumulative bounds fit cap_rows
        int blo[2][3], bhi[2][3], bbad[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int q = 2 * tid + u;
          bbad[u] = 0;
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            blo[u][r] = INT_MAX;
            bhi[u][r] = INT_MIN;
          }
          if (q < T) {
            const double* pq = a.poses + 7 * (p + q);
#pragma unroll
            for (int r = 0; r < 3; ++r) {
              const double t = __ldg(pq + 4 + r);
              if (!isfinite(t)) bbad[u] = 1;
              const double f0 = floor((t - rb + a.b) * a.inv_h) - 1.0;
              const double f1 = floor((t + rb + a.b) * a.inv_h) + 1.0;
              blo[u][r] = (int)fmax(0.0, fmin(f0, (double)(a.n - 1)));
              bhi[u][r] = (int)fmax(0.0, fmin(f1, (double)(a.n - 1)));
            }
          }
        }
        // the thread's pair combined, then scanned over threads (exclusive prefix kept)
        int wlo[3], whi[3], wbad = bbad[0] | bbad[1];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          wlo[r] = min(blo[0][r], blo[1][r]);
          whi[r] = max(bhi[0][r], bhi[1][r]);
        }
        if (warp * 64 < T) {             // warps without poses only join the barriers
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
        for (int w = 0; w < warp && warp * 64 < T; ++w) {
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            wlo[r] = min(wlo[r], s_wred[w][r]);
            whi[r] = max(whi[r], s_wred[w][3 + r]);
          }
          wbad |= s_wred[w][6];
        }
        // cumulative bounds through pose 2 tid: the inclusive scan minus this thread's second pose
        // (exclusive prefix = the previous lane's inclusive value, or the previous warps' total)
        int plo[3], phi_[3], pbad;
        {
          int v[7];
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            v[r] = __shfl_up_sync(kFull, wlo[r], 1);
            v[3 + r] = __shfl_up_sync(kFull, whi[r], 1);
          }
          v[6] = __shfl_up_sync(kFull, wbad, 1);
          if (lane == 0) {
#pragma unroll
            for (int r = 0; r < 3; ++r) {
              v[r] = INT_MAX;
              v[3 + r] = INT_MIN;
            }
            v[6] = 0;
            for (int w = 0; w < warp && warp * 64 < T; ++w) {
#pragma unroll
              for (int r = 0; r < 3; ++r) {
                v[r] = min(v[r], s_wred[w][r]);
                v[3 + r] = max(v[3 + r], s_wred[w][3 + r]);
              }
              v[6] |= s_wred[w][6];
            }
          }
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            plo[r] = min(v[r], blo[0][r]);
            phi_[r] = max(v[3 + r], bhi[0][r]);
          }
          pbad = v[6] | bbad[0];
        }
        int rows0 = 0, rows1 = 0;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          rows0 += phi_[r] - plo[r] + 1;
          rows1 += whi[r] - wlo[r] + 1;
        }
        const bool fit0 = 2 * tid < T && !pbad && rows0 <= cap_rows;
        const bool fit1 = 2 * tid + 1 < T && !wbad && rows1 <= cap_rows;
        // the fit flags are monotone in the pose index (cumulative bounds), so the first Tfit
        // poses form the tile
        const int Tfit = __syncthreads_count(fit0) + __syncthreads_count(fit1);
        fits = Tfit > 0;
        T = fits ? Tfit : 1;         // a single pose whose rows do not fit takes the L2 path
        // the owner of the tile's last pose holds the tile's cumulative bounds
        const int rows = ((T - 1) & 1) ? rows1 : rows0;
        if (!((T - 1) & 1)) {
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            wlo[r] = plo[r];
            whi[r] = phi_[r];
          }
        }
        // the tile's last thread owns the tile's bounds: it restages the window if needed and
        // picks the coarse-cell box of the local range table
        if (tid == (T - 1) >> 1) {
          int rs = 0, reloc = 0;
          unsigned win_bytes = 0;
          bool contained = true;
#pragma unroll
          for (int r = 0; r < 3; ++r) contained = contained && s_cur.lo[r] <= wlo[r] && whi[r] <= s_cur.hi[r];
          if (fits && !contained) {
            const int extra = (cap_rows - rows) / 3;
            int row0 = 0;
            unsigned bytes = 0;
            int lo_[3], hi_[3];
            const bool all = cap_rows >= 3 * a.n;     // the whole factor set fits
#pragma unroll
            for (int r = 0; r < 3; ++r) {
              lo_[r] = all ? 0 : max(0, wlo[r] - extra / 2);
              hi_[r] = all ? a.n - 1 : min(a.n - 1, whi[r] + (extra - extra / 2));
              bytes += (unsigned)(hi_[r] - lo_[r] + 1) * kRow;
            }
            // the window was last read through the generic proxy, before the previous barrier
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            win_bytes = bytes;
#pragma unroll
            for (int r = 0; r < 3; ++r) {
              s_cur.lo[r] = lo_[r];
              s_cur.hi[r] = hi_[r];
              s_cur.off[r] = row0 - lo_[r];
              row0 += hi_[r] - lo_[r] + 1;
            }
            rs = 1;
          }
          if (fits && loc_cd > 0) {
            // the local range table: a loc_cd x loc_cd x (loc_cd + 4) box of the packed ranges
            // around the tile's coarse cells (every atom's cell lies within [wlo, whi]), copied
            // by one TMA tensor copy whose z origin is a multiple of 4 cells (16-byte aligned rows;
            // cells outside the global grid arrive as zero counts)
            const int ext[3] = {loc_cd, loc_cd, loc_cd + 4};
            int clo[3], chi[3];
            bool inside = s_lb.dim[0] > 0, fit_box = true;
#pragma unroll
            for (int r = 0; r < 3; ++r) {
              clo[r] = wlo[r] >> a.nb_shift;
              chi[r] = whi[r] >> a.nb_shift;
              inside = inside && s_lb.lo[r] <= clo[r] && chi[r] < s_lb.lo[r] + ext[r];
              // the packed table starts kPackPad cells below the grid (TMA coordinates are >= 0)
              fit_box = fit_box && clo[r] - a.nb_lo[r] + kPackPad >= 4;
            }
            clo[2] -= (clo[2] - a.nb_lo[2] + kPackPad) & 3;
#pragma unroll
            for (int r = 0; r < 3; ++r) fit_box = fit_box && chi[r] - clo[r] < ext[r];
            if (!inside) {
              if (fit_box) {
                if (!rs) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
                for (int r = 0; r < 3; ++r) {
                  s_lb.lo[r] = clo[r];
                  s_lb.dim[r] = ext[r];
                }
                reloc = 1;
              } else {
                s_lb.dim[0] = s_lb.dim[1] = s_lb.dim[2] = 0;   // global lookups for this tile
              }
            }
          }
          if (rs || reloc) {
            const unsigned tbytes = reloc ? (unsigned)(loc_cd * loc_cd * (loc_cd + 4)) * 4u : 0u;
            mbar_expect_tx(&s_bar, win_bytes + tbytes);
            if (win_bytes) {
#pragma unroll
              for (int r = 0; r < 3; ++r) {
                const int lo_r = s_cur.lo[r], len = s_cur.hi[r] - lo_r + 1;
                RS_DCHECK(lo_r >= 0 && len > 0 && lo_r + len <= a.n && s_cur.off[r] + lo_r >= 0 &&
                          s_cur.off[r] + lo_r + len <= cap_rows);
                const void* src = F32 ? (const void*)(a.t.Fw32[r] + (size_t)lo_r * kChp)
                                      : (const void*)(a.t.Fw[r] + (size_t)lo_r * kChp);
                tma_load_1d(win_u32 + (unsigned)(s_cur.off[r] + lo_r) * kRow, src, (unsigned)len * kRow, &s_bar);
              }
            }
            if (reloc) {
              const int c0 = s_lb.lo[2] - a.nb_lo[2] + kPackPad, c1 = s_lb.lo[1] - a.nb_lo[1] + kPackPad,
                        c2 = s_lb.lo[0] - a.nb_lo[0] + kPackPad;
              RS_DCHECK(c0 >= 0 && c1 >= 0 && c2 >= 0 && (c0 & 3) == 0);
              asm volatile(
                  "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                  " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(loc_u32),
                  "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(&s_bar))
                  : "memory");
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
      const bool use_win = window_mode && fits;
      // per-lane window row bases (shared addresses, with the lane's XOR offset in bits 4..)
      unsigned wb0, wb1, wb2;
      {
        const Window W = s_cur;
        wb0 = win_u32 + (unsigned)W.off[0] * kRow + rho16;
        wb1 = win_u32 + (unsigned)W.off[1] * kRow + rho16;
        wb2 = win_u32 + (unsigned)W.off[2] * kRow + rho16;
      }
      // local range table: address of coarse cell (cx, cy, cz) = loc_org + ((cx d1 + cy) d2 + cz) 4
      unsigned loc_org = 0;
      int ld1 = 0, ld2 = 0;
      bool use_loc = false;
      {
        const LocalBox LB = s_lb;
        use_loc = use_win && LB.dim[0] > 0;
        ld1 = LB.dim[1];
        ld2 = LB.dim[2];
        loc_org = loc_u32 - (unsigned)((LB.lo[0] * ld1 + LB.lo[1]) * ld2 + LB.lo[2]) * 4u;
      }
      // ---- units of the tile -----------------------------------------------------------
      for (;;) {
        int s = 0, g = 32;
        if (lane == 0) {
          const int r = T - *(volatile int*)&s_next;       // a hint only: ranges come from the atomic
          // the tile's last units shrink (a power of two >= min_unit poses, S lanes per pose) so
          // that the warps finish together; smaller units pay more per pose in H1 and the drain
          // of their candidate walks than they gain in balance
          if (r < 32 * kWarps) g = min(32, pow2_floor(max(min_unit, r / kWarps)));
          s = atomicAdd(&s_next, g);
        }
        s = __shfl_sync(kFull, s, 0);
        g = __shfl_sync(kFull, g, 0);
        if (s >= T) break;
        const int lgS = 5 - (31 - __clz(g));               // S = 32 / g lanes per pose
        const int S = 1 << lgS;
        const int sub = lane & (S - 1);
        const int sp = s + (lane >> lgS);
        const bool has = sp < T;
        const int64_t pp = p + (has ? sp : s);
        // H1 (O1) in registers: each lane holds its pose's R and t
        double Rm[9], tv[3];
        bool ok;
        {
          double qv[7];
          const double* pq = a.poses + 7 * pp;
#pragma unroll
          for (int i = 0; i < 7; ++i) qv[i] = __ldg(pq + i);
          ok = quat_rot_dev(qv, Rm);
          if (!ok) {
#pragma unroll
            for (int i = 0; i < 9; ++i) Rm[i] = 0.0;   // x' = t: a cell inside the tile's window
          }
#pragma unroll
          for (int i = 0; i < 3; ++i) tv[i] = qv[4 + i];
        }
        const bool live = has && ok;
        bool bad = has && !ok;
        double hi = 0.0, lo = 0.0, best = INFINITY;
        unsigned vthr = a.vdw_cells2;
        unsigned stopk = stop_key(a, vthr);
        double bthr = INFINITY;   // the minimum the bounds were computed from
        BallPending bp;
        bp.f = 0;
        const int nsteps = (L + S - 1) >> lgS;
        // H5 + H6 as a per-lane queue: a lane walks the candidate list of one atom at a time, two
        // entries per atom step, while later atoms with candidates wait on its stack; the entry
        // pair a lane walks next is loaded one atom step ahead, behind that step's H4 gathers
        double q0 = 0.0, q1 = 0.0, q2 = 0.0, qz = 0.0;
        int qc01 = 0, qc2 = 0, qpos = 0, qend = 0, qfc = 0;
        int4 pf0 = make_int4(0, 0, 0, 0), pf1 = pf0;
        NbrQueue& nq = s_nq[warp];
        // the ligand atom lc (body frame y, charge z), from shared memory when staged
        auto lig_atom = [&](int lc, double& y0, double& y1, double& y2, double& z) {
          if (lig_all_smem) {
            RS_DCHECK(lc >= 0 && lc < lig_smem_n);
            const double2 v0 = s_lig[lc], v1 = s_lig[lig_smem_n + lc];
            y0 = v0.x; y1 = v0.y; y2 = v1.x; z = v1.y;
          } else {
            // window launches stage up to 256 atoms, so this is their rare case: out of line
            // (one branch instead of predicated-off loads in every atom step); L2 launches
            // with a ligand beyond shared memory (C5's 5,000-atom partner) take it every step
            if constexpr (WIN && RS_LIG_CALL) {
              const double4 v = lig_atom_global(a.yl, a.zl, lc);
              y0 = v.x; y1 = v.y; y2 = v.z; z = v.w;
            } else {
              y0 = __ldg(a.yl + 3 * (int64_t)lc);
              y1 = __ldg(a.yl + 3 * (int64_t)lc + 1);
              y2 = __ldg(a.yl + 3 * (int64_t)lc + 2);
              z = __ldg(a.zl + lc);
            }
          }
        };
        // H2 (O2): x' = R y + t, the pose's R and t in registers
        auto h2 = [&](double y0, double y1, double y2, double& x0, double& x1, double& x2) {
          x0 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(Rm[0], y0), __dmul_rn(Rm[1], y1)), __dmul_rn(Rm[2], y2)), tv[0]);
          x1 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(Rm[3], y0), __dmul_rn(Rm[4], y1)), __dmul_rn(Rm[5], y2)), tv[1]);
          x2 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(Rm[6], y0), __dmul_rn(Rm[7], y1)), __dmul_rn(Rm[8], y2)), tv[2]);
        };
#if RS_VOTE_MASK
        unsigned am = 0;   // lanes with a walk in progress (kept across the loop: one ballot per
                           // round and per atom step instead of a vote before every decision)
#endif
        auto nbr_step = [&]() {
          const bool act = qpos < qend;
#if RS_VOTE_MASK
          if (am) {
#else
          if (__any_sync(kFull, act)) {
#endif
#if RS_DYN_THR
            // the bounds follow the lane's minimum lazily: it may have moved in the previous
            // round, whose record loads have landed behind the atom step since (a branch on this
            // round's records would stall the warp before its H4 gathers)
            if (best < bthr) {
              bthr = best;
              vthr = vdw_thr(a, best);
              stopk = stop_key(a, vthr);
            }
#endif
            bool end;
#if RS_DEFER_BALL
            ball_flush(bp, hi, lo);
#endif
            nbr_pair(a, q0, q1, q2, qz, qc01 & 0xffff, (int)((unsigned)qc01 >> 16), qc2, pf0, pf1, act,
                     qpos + 1 < qend, hi, lo, best, vthr, stopk, end, bp);
            qpos = end ? qend : qpos + 2;
            if (act && qpos >= qend && qfc > 0) {
              --qfc;
#if RS_QCOMPACT
              const int4 cb = nq.cb[qfc][lane];
              double y0, y1, y2;
              lig_atom(cb.x, y0, y1, y2, qz);
              h2(y0, y1, y2, q0, q1, q2);
              qc01 = snap_dev(q0, a.b, a.inv_h, nm1) | (snap_dev(q1, a.b, a.inv_h, nm1) << 16);
              qc2 = snap_dev(q2, a.b, a.inv_h, nm1);
              qpos = cb.y; qend = cb.z;
#else
              const double2 v01 = nq.x01[qfc][lane], v2z = nq.x2z[qfc][lane];
              const int4 cb = nq.cb[qfc][lane];
              q0 = v01.x; q1 = v01.y; q2 = v2z.x; qz = v2z.y;
              qc01 = cb.x; qc2 = cb.y; qpos = cb.z; qend = cb.w;
#endif
            }
            const bool more = qpos < qend;
            RS_DCHECK(!more || (qpos >= 0 && qpos + 2 <= a.n_ent));
#if RS_VOTE_MASK
            am = __ballot_sync(kFull, more);
            if (am) ldg_pair_p(a.t.nb_ent + qpos, more, pf0, pf1);
#else
            if (__any_sync(kFull, more)) ldg_pair_p(a.t.nb_ent + qpos, more, pf0, pf1);
#endif
          }
        };
        // one candidate round per pass; an atom step only when every lane can take its atom
        // (idle, or room on its stack); after the last atom, walk until every lane is done
        for (int it = 0;;) {
          nbr_step();
#if RS_VOTE_MASK
          if (am && __any_sync(kFull, qfc == kNQ && qpos < qend)) continue;
          if (it >= nsteps) {
            if (am) continue;
            break;
          }
#else
          if (__any_sync(kFull, qfc == kNQ && qpos < qend)) continue;
          if (it >= nsteps) {
            if (__any_sync(kFull, qpos < qend)) continue;
            break;
          }
#endif
          const int l = (it++ << lgS) + sub;
          const bool act = live && l < L;
          const int lc = l < L ? l : L - 1;
          double y0, y1, y2, z;
          lig_atom(lc, y0, y1, y2, z);
          // H2 (O2)
          double x0, x1, x2;
          h2(y0, y1, y2, x0, x1, x2);
          // H3 (O3): valid iff -b <= x'_a <= b on every axis (false for NaN)
          const bool inb = fabs(x0) <= a.b && fabs(x1) <= a.b && fabs(x2) <= a.b;
          bad = bad || (act && !inb);
          const bool go = act && inb;
          const int i0 = snap_dev(x0, a.b, a.inv_h, nm1);
          const int i1 = snap_dev(x1, a.b, a.inv_h, nm1);
          const int i2 = snap_dev(x2, a.b, a.inv_h, nm1);
          // candidate range of the coarse cell containing i (the lists hold every protein atom
          // that can matter to H5/H6 for any point of the cell); issued before H4 so its latency
          // hides behind the gathers
          int beg = 0, cnt = 0;
#if !(defined(RS_EXPERIMENT) && (RS_EXPERIMENT & 1))
          {
            const int cx = i0 >> a.nb_shift, cy = i1 >> a.nb_shift, cz = i2 >> a.nb_shift;
            int2 bc;
            if (use_loc) {
              // every atom of a fitting tile (and every lane's stand-in atom) has its coarse cell
              // inside the tile's box (the row bounds t +- rb contain the atom's cell)
              RS_DCHECK(cx >= s_lb.lo[0] && cx < s_lb.lo[0] + s_lb.dim[0] && cy >= s_lb.lo[1] &&
                        cy < s_lb.lo[1] + s_lb.dim[1] && cz >= s_lb.lo[2] && cz < s_lb.lo[2] + s_lb.dim[2]);
              const unsigned v = lds_u32(loc_org + (unsigned)((cx * ld1 + cy) * ld2 + cz) * 4u);
              bc = make_int2((int)(v & 0xffffffu), (int)(v >> 24));
            } else {
              const unsigned gx = (unsigned)(cx - a.nb_lo[0]), gy = (unsigned)(cy - a.nb_lo[1]),
                             gz = (unsigned)(cz - a.nb_lo[2]);
              const bool in = go && gx < (unsigned)a.nb_dim[0] && gy < (unsigned)a.nb_dim[1] &&
                              gz < (unsigned)a.nb_dim[2];
              bc = ldg_if(a.t.nb_range + (gx * a.nb_dim[1] + gy) * a.nb_dim[2] + gz, in);
            }
            beg = bc.x;
            cnt = go ? bc.y : 0;
          }
#endif
          // enqueue this atom's candidates: walk them next if the lane is idle, else stack them
          // (the pass loop guarantees room); the first entry pair loads behind this step's H4
          RS_DCHECK(cnt <= 0 || (beg >= 0 && beg + cnt <= a.n_ent));
          if (cnt > 0) {
            if (qpos >= qend) {
              q0 = x0; q1 = x1; q2 = x2; qz = z;
              qc01 = i0 | (i1 << 16); qc2 = i2; qpos = beg; qend = beg + cnt;
              ldg_pair_p(a.t.nb_ent + beg, true, pf0, pf1);
            } else {
              RS_DCHECK(qfc < kNQ);
#if RS_QCOMPACT
              nq.cb[qfc][lane] = make_int4(lc, beg, beg + cnt, 0);
#else
              nq.x01[qfc][lane] = make_double2(x0, x1);
              nq.x2z[qfc][lane] = make_double2(x2, z);
              nq.cb[qfc][lane] = make_int4(i0 | (i1 << 16), i2, beg, beg + cnt);
#endif
              ++qfc;
            }
          }
#if RS_VOTE_MASK
          am = __ballot_sync(kFull, qpos < qend);
#endif
          // H4 (O4)
          double phi = 0.0;
          if constexpr (RT > 0) {
            if (use_win) {
              // every row of a fitting tile is staged (the tile's bounds contain t +- rb, and
              // lanes without a real atom stand in with an atom of a pose of the tile)
              RS_DCHECK(i0 >= s_cur.lo[0] && i0 <= s_cur.hi[0] && i1 >= s_cur.lo[1] && i1 <= s_cur.hi[1] &&
                        i2 >= s_cur.lo[2] && i2 <= s_cur.hi[2]);
              const unsigned r0 = wb0 + (unsigned)i0 * kRow;
              const unsigned r1 = wb1 + (unsigned)i1 * kRow;
              const unsigned r2 = wb2 + (unsigned)i2 * kRow;
#if defined(RS_EXPERIMENT) && (RS_EXPERIMENT & 2)
              double v = z;
#else
              double v;
              if constexpr (F32) v = (double)SmemTree32<0, 1, Geo32<RT>::NS>::eval(r0, r1, r2);
              else v = SmemTree<0, 1, Geo<RT>::NS>::eval(r0, r1, r2);
#endif
              phi = go ? v : 0.0;
            } else if (go) {
              RS_DCHECK(i0 >= 0 && i0 < a.n && i1 >= 0 && i1 < a.n && i2 >= 0 && i2 < a.n);
              if constexpr (WIN) {       // a single pose whose rows do not fit: out of line
                if constexpr (F32) phi = long_phi_global32<RT>(a.t.Fw32[0], a.t.Fw32[1], a.t.Fw32[2], i0, i1, i2);
                else phi = long_phi_global<RT>(a.t.F[0], a.t.F[1], a.t.F[2], i0, i1, i2);
              } else if constexpr (F32) {
                phi = long_phi_l2_32<RT, RS_L2_CG != 0>(a.t.Fw32[0], a.t.Fw32[1], a.t.Fw32[2], i0, i1, i2);
              } else {
                phi = long_phi_l2<RT, RS_L2_CG != 0>((const double2*)(a.t.F[0] + (size_t)i0 * RT),
                                      (const double2*)(a.t.F[1] + (size_t)i1 * RT),
                                      (const double2*)(a.t.F[2] + (size_t)i2 * RT));
              }
            }
          } else if constexpr (RT == 0) {
            if (go)
              phi = long_phi_rt<RS_L2_CG != 0>(a.t.F[0] + (size_t)i0 * a.R, a.t.F[1] + (size_t)i1 * a.R,
                                a.t.F[2] + (size_t)i2 * a.R, a.R);
          } else {
            // N5: the long range from the Tucker form, core staged in shared memory
            if (go) phi = tucker_phi(a, i0, i1, i2, s_tg);
          }
          const double zg = go ? z : 0.0;
          dd_add_prod(hi, lo, zg, phi);
        }
        // after the last atom, walk until every lane is done: the pose's R and t are dead here,
        // so a drain round takes two entry pairs (both loaded a round ahead) against one record
        // latency, where the atom-step rounds take one
#if RS_DEFER_BALL
        ball_flush(bp, hi, lo);
#endif
        // H7: merge the S lanes of each pose (xor butterfly within aligned groups of S lanes;
        // TwoSum is exact, so partners agree); min d^2 and the invalid flag likewise
        for (int off = S >> 1; off > 0; off >>= 1) {
          const double h2 = __shfl_xor_sync(kFull, hi, off);
          const double l2 = __shfl_xor_sync(kFull, lo, off);
          dd_merge(hi, lo, h2, l2);
          const double b2 = __shfl_xor_sync(kFull, best, off);
          best = b2 < best ? b2 : best;
          const int bo = __shfl_xor_sync(kFull, (int)bad, off);
          bad = bad || bo != 0;
        }
        // H8: E = hi + lo; d = sqrt(min d^2) below D_cap^2, else +inf; NaN if invalid (O8)
        if (has && sub == 0) {
          RS_DCHECK(pp >= 0 && pp < a.P);
          a.E[pp] = bad ? NAN : __dadd_rn(hi, lo);
          a.D[pp] = bad ? NAN : (best < a.dcap2 ? __dsqrt_rn(best) : INFINITY);
          if (bad && a.invalid) atomicAdd(a.invalid, 1ull);
        }
      }
#if RS_TILE_OVERLAP
      // No barrier of its own at the end of a tile: the next barrier every warp meets ends it --
      // the first barrier of the next tile's scan (window launches: the scan starts with
      // per-warp work, pose loads and warp scans, that touches nothing the units use, so warps
      // that finish early overlap it with the slower warps' last units), or at the end of a chunk
      // the barrier behind the next chunk's claim.  Nothing the units read is written before
      // that barrier.  Kept where the next tile's set-up follows without one (interior tiles of
      // L2 launches) and in streamed launches (the completion counters below).
      if (a.done || (!window_mode && p + T < p_end)) __syncthreads();
#else
      __syncthreads();
#endif
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

// Per-device launch state, set up once (std::call_once: concurrent first launches are safe)
struct DevCache {
  std::once_flag once;
  int sms = 0;
  int smem_optin = 0;
  int init_err = 0;
  std::once_flag attr_once[32];
  int attr_err[32] = {0};
  int max_dyn[32] = {0};
};
DevCache g_dev[64];

constexpr int kNoWindow = -12345;   // launch_t<.., WIN = true>: use the L2 variant instead

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                    CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);
PFN_encodeTiled encode_tiled() {
  static std::once_flag once;
  static PFN_encodeTiled fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled)p;
    cudaGetLastError();
  });
  return fn;
}

// Tensor map of the packed neighbour ranges (uint32, z fastest) with a cd x cd x (cd + 4) box; false if it
// cannot be built (the kernel then uses global range lookups)
bool local_table_map(const ScoreArgs& a, int cd, CUtensorMap* m) {
  PFN_encodeTiled enc = encode_tiled();
  if (!enc || !a.t.nb_pack || cd <= 0) return false;
  const cuuint64_t e1 = (cuuint64_t)a.nb_dim[1] + kPackPad, e0 = (cuuint64_t)a.nb_dim[0] + kPackPad;
  const cuuint64_t dims[3] = {(cuuint64_t)a.nb_dim2p, e1, e0};
  const cuuint64_t strides[2] = {(cuuint64_t)a.nb_dim2p * 4u, (cuuint64_t)a.nb_dim2p * e1 * 4u};
  const cuuint32_t box[3] = {(cuuint32_t)cd + 4u, (cuuint32_t)cd, (cuuint32_t)cd};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, (void*)a.t.nb_pack, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

constexpr int kPlanned = -12346;    // launch_t in plan-only mode: the variant would launch
template <int RT, bool F32, bool WIN>
int launch_t(const ScoreArgs& a, cudaStream_t st, int dev, int slot, bool plan_only = false) {
  DevCache& dc = g_dev[dev & 63];
  std::call_once(dc.attr_once[slot], [&] {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, score_kernel<RT, F32, WIN>);
    if (e == cudaSuccess) {
      const int m = dc.smem_optin - (int)fa.sharedSizeBytes;
      e = cudaFuncSetAttribute(score_kernel<RT, F32, WIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
      if (e == cudaSuccess) dc.max_dyn[slot] = m;
    }
    dc.attr_err[slot] = (int)e;
  });
  if (dc.attr_err[slot]) return dc.attr_err[slot];
  constexpr int kChp = F32 ? Geo32<(RT > 0 ? RT : 4)>::CHP : Geo<(RT > 0 ? RT : 2)>::CHP;
  constexpr size_t kRowB = 16 * (size_t)kChp;
  // alignment slack of the window base, neighbour queues, and (N5) the Tucker core
  const size_t fixed = 256 + kQueueBytes + (RT < 0 ? (size_t)a.tr[0] * a.tr[1] * a.tr[2] * sizeof(double) : 0);
  const size_t avail = (size_t)dc.max_dyn[slot] > fixed ? (size_t)dc.max_dyn[slot] - fixed : 0;
  const size_t lig_res = std::min<size_t>(avail, (size_t)std::min<int64_t>(a.L, 256) * sizeof(double4));
  int cap_rows = 0, loc_cap = 0, loc_cd = 0;
  CUtensorMap tmap;
  std::memset(&tmap, 0, sizeof(tmap));
  if constexpr (RT > 0 && WIN) {
    if (!(F32 ? (const void*)a.t.Fw32[0] : (const void*)a.t.Fw[0])) return kNoWindow;
#ifndef RS_NO_TMA_LOC
    if (a.loc4 && a.t.nb_pack) {
#else
    if (false) {
#endif
      // local range table: a cd^3 box of coarse cells, cd a multiple of 4 (16-byte TMA rows),
      // large enough for one translation's atoms when the ligand radius is known
      int cd = 20;
      if (a.rmax_hint >= 0) {
        const double rows = 2.0 * (a.rmax_hint * (1.0 + 1e-12) + 2.0 * a.h) / a.h + 3.0;
        cd = (int)std::ceil(rows / double(1 << a.nb_shift)) + 1;
        cd = (cd + 3) / 4 * 4;
      }
      if (cd * cd * (cd + 4) <= RS_LOC_CELLS && local_table_map(a, cd, &tmap)) {
        loc_cd = cd;
        loc_cap = cd * cd * (cd + 4);
      }
    }
    const size_t loc_b = (size_t)loc_cap * sizeof(unsigned);
    cap_rows = (int)std::min<size_t>((avail - lig_res - std::min(avail - lig_res, loc_b)) / kRowB,
                                     (1u << 20) / kRowB - 1);
    if (3 * a.n <= cap_rows) {
      // the whole factor set fits (small grids, e.g. C1): stage it once, every tile fits
      cap_rows = 3 * a.n;
    } else if (a.rmax_hint >= 0) {
      // what one translation's window needs plus RS_WIN_SLACK (the rest of the 228 KB is L1
      // for the candidate lists, records and the short-range memo); no window at all when even
      // one translation's rows do not fit (every pose would be its own tile with its own
      // restage: the L2 variant is faster then)
      const double need = 3.0 * (2.0 * (a.rmax_hint + 2.0 * a.h) / a.h + 8.0);
      if (need > cap_rows) return kNoWindow;
      cap_rows = std::min(cap_rows, (int)std::max(64.0, RS_WIN_SLACK * need));
    }
    if (cap_rows <= 0) return kNoWindow;
  }
  const size_t win_b = (size_t)cap_rows * kRowB;
  const size_t loc_b = (size_t)loc_cap * sizeof(unsigned);
  const size_t used = std::min(avail, win_b + loc_b);
  const int64_t lig_fit = (int64_t)((avail - used) / sizeof(double4));
  const int lig_n = (int)std::min<int64_t>(a.L, cap_rows > 0 ? std::min<int64_t>(lig_fit, 256) : lig_fit);
  const size_t dyn = fixed + win_b + loc_b + (size_t)lig_n * sizeof(double4);
  // chunk plan: big chunks for the first (1 - 1/RS_TAIL_DIV) of the poses, then tail chunks of
  // at most kTailChunk poses, small enough that every SM gets work when P is small
  // (big chunks also shrink with P: at least ~4 per SM, so one chunk never dominates a launch)
  ChunkPlan cp;
  cp.big = (int)std::max<int64_t>(kMinBig, std::min<int64_t>(kChunk, a.P / (4 * (int64_t)dc.sms)));
  cp.nbig = (a.P - a.P / RS_TAIL_DIV) / cp.big;
  const int64_t rest = a.P - cp.nbig * cp.big;
  cp.tail = (int)std::max<int64_t>(1, std::min<int64_t>(kTailChunk, (rest + 2 * dc.sms - 1) / (2 * dc.sms)));
  const int64_t chunks = cp.nbig + (rest + cp.tail - 1) / cp.tail;
  int grid = (int)std::min<int64_t>(chunks, (int64_t)dc.sms);
  if (grid < 1) grid = 1;
  if (plan_only) return kPlanned;
  score_kernel<RT, F32, WIN><<<grid, kThreads, dyn, st>>>(a, cap_rows, lig_n, loc_cap, cp, tmap, loc_cd);
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

// Dispatch of one scoring launch: the compiled width's shared-memory window variant, else its
// L2 variant, else the runtime-width kernel.  plan_only: decide without launching and return
// the path (kPathWindow / kPathL2 / kPathL2Runtime) or a CUDA error code.
int launch_or_plan(const ScoreArgs& a, void* stream, int device, int* launches, bool plan_only) {
  if (a.P <= 0 && !plan_only) return 0;
  if (a.L > (int64_t)1 << 30) return (int)cudaErrorInvalidValue;   // the kernel indexes atoms in int
  DevCache& dc = g_dev[device & 63];
  std::call_once(dc.once, [&] {
    cudaError_t e = cudaDeviceGetAttribute(&dc.sms, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&dc.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    dc.init_err = (int)e;
  });
  if (dc.init_err) return dc.init_err;
  cudaStream_t st = (cudaStream_t)stream;
  int e;
  if (a.tk) {
    // N5: Tucker-format evaluation (rows from L2, the core in shared memory)
    e = launch_t<-1, false, false>(a, st, device, 14, plan_only);
    if (e == kPlanned) return kPathTucker;
    if (launches) *launches += 1;
    return e;
  }
  if (a.f32) {
    // binary32 factors (A21): compiled widths only (the build refuses others)
#define RS_F32_CASE(RR, SLOT)                                                               \
  case RR:                                                                                 \
    e = launch_t<RR, true, true>(a, st, device, SLOT, plan_only);                          \
    if (e == kPlanned) return kPathWindow;                                                 \
    if (e == kNoWindow) e = launch_t<RR, true, false>(a, st, device, SLOT + 1, plan_only); \
    if (e == kPlanned) return kPathL2;                                                     \
    break;
    switch (a.R) {
      RS_F32_CASE(4, 20) RS_F32_CASE(8, 22) RS_F32_CASE(12, 24) RS_F32_CASE(16, 26)
      RS_F32_CASE(24, 28) RS_F32_CASE(32, 30)
      default: return (int)cudaErrorInvalidValue;
    }
#undef RS_F32_CASE
  } else {
#define RS_F64_CASE(RR, SLOT)                                                               \
  case RR:                                                                                 \
    e = launch_t<RR, false, true>(a, st, device, SLOT, plan_only);                         \
    if (e == kPlanned) return kPathWindow;                                                 \
    if (e == kNoWindow) e = launch_t<RR, false, false>(a, st, device, SLOT + 1, plan_only); \
    if (e == kPlanned) return kPathL2;                                                     \
    break;
    switch (a.R) {
      RS_F64_CASE(4, 2) RS_F64_CASE(8, 4) RS_F64_CASE(12, 6) RS_F64_CASE(16, 8)
      RS_F64_CASE(24, 10) RS_F64_CASE(32, 12)
      default:
        e = launch_t<0, false, false>(a, st, device, 0, plan_only);
        if (e == kPlanned) return kPathL2Runtime;
        break;
    }
#undef RS_F64_CASE
  }
  if (launches) *launches += 1;
  return e;
}

int launch_score(const ScoreArgs& a, void* stream, int device, int* launches) {
  return launch_or_plan(a, stream, device, launches, false);
}

int plan_score(const ScoreArgs& a, int device) { return launch_or_plan(a, nullptr, device, nullptr, true); }

}  // namespace rs
