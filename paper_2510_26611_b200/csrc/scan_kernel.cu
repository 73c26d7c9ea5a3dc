// PPIEM scan (NEXT row N2): Algorithm PPIEM steps A3-A5, DESIGN.md
// reading A23.  The scoring itself is the fused kernel (score_kernel.cu); this file holds the
// two small per-pose kernels of the approach loop: the initial poses and the sphere-tracing
// update of the distance s along each position's line toward the protein centre.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "rs_internal.h"

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
                                 int* status) {
  const int64_t P = (int64_t)m_P * m_L;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(p / m_L), k = (int)(p % m_L);
    s[p] = s_start;
    status[p] = -1;                                   // active
    write_pose(poses + 7 * p, centre, dirs + 3 * j, quats + 4 * k, s_start);
  }
}

// One sphere-tracing step from the scored minimum distances D (+inf at or beyond D_cap, NaN for
// an invalid pose).  Status: -1 active, 0 contact, 1 left the box, 2 clash at the start,
// 3 passed the centre.
__global__ void scan_update_kernel(const double* centre, const double* dirs, const double* quats,
                                   int m_P, int m_L, const double* D, double sigma, double dcap,
                                   double tol, int first, double* poses, double* s, int* status,
                                   int* active) {
  const int64_t P = (int64_t)m_P * m_L;
  int mine = 0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (status[p] != -1) continue;
    const double d = D[p];
    double sn;
    if (isnan(d)) {
      status[p] = 1;
      continue;
    }
    if (isinf(d)) {
      sn = __dsub_rn(s[p], __dsub_rn(dcap, sigma));
    } else {
      const double delta = __dsub_rn(d, sigma);
      if (delta < 0.0) {                               // only possible at the start
        status[p] = first ? 2 : 1;
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
    write_pose(poses + 7 * p, centre, dirs + 3 * j, quats + 4 * k, sn);
    ++mine;
  }
  // warp-aggregated count of poses still moving
  for (int off = 16; off > 0; off >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, off);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(active, mine);
}

}  // namespace

int launch_scan_init(const double* centre, const double* dirs, const double* quats, int m_P,
                     int m_L, double s_start, double* poses, double* s, int* status, void* st) {
  const int64_t P = (int64_t)m_P * m_L;
  const int blocks = (int)std::min<int64_t>((P + 255) / 256, 4096);
  scan_init_kernel<<<blocks, 256, 0, (cudaStream_t)st>>>(centre, dirs, quats, m_P, m_L, s_start,
                                                         poses, s, status);
  return (int)cudaGetLastError();
}

int launch_scan_update(const double* centre, const double* dirs, const double* quats, int m_P,
                       int m_L, const double* D, double sigma, double dcap, double tol, int first,
                       double* poses, double* s, int* status, int* active, void* st) {
  const int64_t P = (int64_t)m_P * m_L;
  const int blocks = (int)std::min<int64_t>((P + 255) / 256, 4096);
  scan_update_kernel<<<blocks, 256, 0, (cudaStream_t)st>>>(centre, dirs, quats, m_P, m_L, D, sigma,
                                                           dcap, tol, first, poses, s, status,
                                                           active);
  return (int)cudaGetLastError();
}

}  // namespace rs
