// PPIEM scan (NEXT row N2): Algorithm PPIEM steps A3-A5, DESIGN.md
// reading A23.  The scoring itself is the fused kernel (score_kernel.cu); this file holds the
// small per-pose kernels of the approach loop: the initial poses and the sphere-tracing update
// of the distance s along each position's line toward the protein centre.  Only the poses still
// moving are scored again: the update compacts them into the next launch's pose list (slot[p] is
// a pose's place in that list; the order of the list is free, every pose is scored alone).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "rs_internal.h"
#include "rs_device.cuh"

namespace rs {
namespace {

// pose (j, k) = orientation quats[k], translation centre + s dirs[j]  (t_a = c_a + s u_a)
__device__ __forceinline__ void write_pose(double* pose, const double* centre, const double* u,
                                           const double* q, double s) {
  for (int i = 0; i < 4; ++i) pose[i] = q[i];
  for (int a = 0; a < 3; ++a) pose[4 + a] = __dadd_rn(centre[a], __dmul_rn(s, u[a]));
}

__global__ void scan_init_kernel(const double* centre, const double* dirs, const double* quats,
                                 int m_P, int m_L, double s_start, double* poses, double* s,
                                 int* status, int* slot) {
  const int64_t P = (int64_t)m_P * m_L;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(p / m_L), k = (int)(p % m_L);
    s[p] = s_start;
    status[p] = -1;                                   // active
    slot[p] = (int)p;
    write_pose(poses + 7 * p, centre, dirs + 3 * j, quats + 4 * k, s_start);
  }
}

// One sphere-tracing step from the scored minimum distances Dc (+inf at or beyond D_cap, NaN
// for an invalid pose) and energies Ec of the current list (pose p at slot[p]).  Status: -1
// active, 0 contact, 1 left the box (an invalid pose), 2 clash at the start, 3 passed the
// centre.  The directions are unit vectors (the host checks), so a step of at most the
// clearance d - sigma never jumps the first contact on the line.  Poses that
// move are appended to the next list (poses_next, slot[p], *count).
__global__ void scan_update_kernel(const double* centre, const double* dirs, const double* quats,
                                   int m_P, int m_L, const double* Dc, const double* Ec,
                                   double sigma, double dcap, double tol, int first, double* E,
                                   double* s, int* status, int* slot, double* poses_next,
                                   int* count) {
  const int64_t P = (int64_t)m_P * m_L;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (status[p] != -1) continue;
    const int sl = slot[p];
    RS_DCHECK(sl >= 0 && sl < P);
    const double d = Dc[sl];
    E[p] = Ec[sl];
    double sn;
    if (isnan(d)) {
      status[p] = 1;
      continue;
    }
    if (isinf(d)) {
      sn = __dsub_rn(s[p], __dsub_rn(dcap, sigma));
    } else {
      const double delta = __dsub_rn(d, sigma);
      if (delta < 0.0) {
        // at the start: a clash; later the steps never close more than the clearance, so only
        // rounding can put d below sigma: that is contact (reading A23)
        status[p] = first ? 2 : 0;
        continue;
      }
      if (delta <= tol) {
        status[p] = 0;
        continue;
      }
      sn = __dsub_rn(s[p], __dmul_rn(delta, 0.999));
    }
    if (sn < 0.0) {
      status[p] = 3;
      continue;
    }
    s[p] = sn;
    const int j = (int)(p / m_L), k = (int)(p % m_L);
    const int ns = atomicAdd(count, 1);
    RS_DCHECK(ns >= 0 && ns < P);
    slot[p] = ns;
    write_pose(poses_next + 7 * (int64_t)ns, centre, dirs + 3 * j, quats + 4 * k, sn);
  }
}

// energies of the poses still moving after the last iteration, scored where they stand
__global__ void scan_gather_kernel(int64_t P, const int* status, const int* slot, const double* Ec,
                                   double* E) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x)
    if (status[p] == -1) E[p] = Ec[slot[p]];
}

int blocks_for(int64_t P) { return (int)std::max<int64_t>(1, std::min<int64_t>((P + 255) / 256, 4096)); }

}  // namespace

int launch_scan_init(const double* centre, const double* dirs, const double* quats, int m_P,
                     int m_L, double s_start, double* poses, double* s, int* status, int* slot,
                     void* st) {
  scan_init_kernel<<<blocks_for((int64_t)m_P * m_L), 256, 0, (cudaStream_t)st>>>(
      centre, dirs, quats, m_P, m_L, s_start, poses, s, status, slot);
  return (int)cudaGetLastError();
}

int launch_scan_update(const double* centre, const double* dirs, const double* quats, int m_P,
                       int m_L, const double* Dc, const double* Ec, double sigma, double dcap,
                       double tol, int first, double* E, double* s, int* status, int* slot,
                       double* poses_next, int* count, void* st) {
  scan_update_kernel<<<blocks_for((int64_t)m_P * m_L), 256, 0, (cudaStream_t)st>>>(
      centre, dirs, quats, m_P, m_L, Dc, Ec, sigma, dcap, tol, first, E, s, status, slot,
      poses_next, count);
  return (int)cudaGetLastError();
}

int launch_scan_gather(int64_t P, const int* status, const int* slot, const double* Ec, double* E,
                       void* st) {
  scan_gather_kernel<<<blocks_for(P), 256, 0, (cudaStream_t)st>>>(P, status, slot, Ec, E);
  return (int)cudaGetLastError();
}

}  // namespace rs
