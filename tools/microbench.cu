// Microbenchmarks that supply the roofline denominators MEASURED_PEAKS.json lacks
// for this path: FP64 DFMA issue rate, shared-memory
// LDS.128 bandwidth (conflict-free, random-row, random-row with lane-rotated chunks),
// and L2 gather bandwidth over an L2-resident table.  Prints one JSON object.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
         x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[blockIdx.x] = s;
}

// mode 0: conflict-free by construction -- each quarter-warp reads the 8 chunks of one row
//         (lane-rotated), the 4 rows of a warp random per iteration
// mode 1: random row per lane, chunk c same for all lanes (unrotated: 8-way conflicts)
// mode 2: random row per lane, chunk (c + lane) & 7 (rotated: what the scoring kernel does)
// The row index of the next iteration depends on the loaded data (acc bits), so no load can be
// hoisted or elided; the table holds small integers, so the dependence is cheap.
template <int MODE>
__global__ void k_lds(unsigned long long* out, int iters, int nrows) {
  extern __shared__ double4 sm4[];
  double2* sm = reinterpret_cast<double2*>(sm4);
  for (int i = threadIdx.x; i < nrows * 8; i += blockDim.x) sm[i] = make_double2((double)(i & 7), 0.0);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t st = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x * 7919u;
  double acc0 = 0, acc1 = 0;
  for (int it = 0; it < iters; ++it) {
    st = st * 1664525u + 1013904223u + (uint32_t)acc1;   // acc1 stays 0: a data dependence only
    uint32_t r = st >> 8;
    if (MODE == 0) r = __shfl_sync(0xffffffffu, r, lane & ~7);
    const int row = (int)(r % (uint32_t)nrows);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      int ch = (MODE == 1) ? c : ((c + lane) & 7);
      double2 v;
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y)
                   : "r"((unsigned)__cvta_generic_to_shared(&sm[row * 8 + ch])));
      acc0 += v.x; acc1 += v.y;
    }
  }
  if (acc0 + acc1 == -1.0) out[blockIdx.x] = 1;
}

// L2 gather like the scoring kernel's L2 path (C4: R = 24, C5: R = 8..32): every lane reads its
// own random row of W 32-byte sectors (a row of 4W doubles) with 256-bit loads.  CG = 1 uses
// ld.global.cg (L2 only, no L1 allocation): the L2 service rate; CG = 0 uses ld.global.nc
// (L1-allocating, what the kernel issues).
template <int W, int CG>
__global__ void k_l2gather(const double4* __restrict__ tab, unsigned long long* out, int iters,
                           uint32_t nrows) {
  uint32_t st = 0x9E3779B9u * (threadIdx.x + 1 + blockIdx.x * blockDim.x);
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    st = st * 1664525u + 1013904223u + (uint32_t)acc;   // acc stays 0: a data dependence only
    const uint32_t row = (st >> 4) % nrows;
    const double4* p = tab + (size_t)row * W;
#pragma unroll
    for (int c = 0; c < W; ++c) {
      double4 v;
      if (CG)
        asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p + c));
      else
        asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p + c));
      acc += v.x + v.w;
    }
  }
  if (acc == -1.0) out[blockIdx.x] = 1;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int nsm = p.multiProcessorCount;
  int clk_khz = 0; CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  double* dout; CK(cudaMalloc(&dout, 1 << 20));
  unsigned long long* uout; CK(cudaMalloc(&uout, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;

  // FP64 DFMA: 8 warps-worth of blocks per SM
  int blocks = nsm * 8, threads = 256, iters = 4096;
  k_dfma<<<blocks, threads>>>(dout, 16, 1.0000001, 1e-9);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  k_dfma<<<blocks, threads>>>(dout, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  double dfma = (double)blocks * threads * iters * 16 * 8;
  double dfma_per_s = dfma / (ms * 1e-3);

  // LDS
  int nrows = 279 * 3;  // C3 window scale: 279 rows x 3 axes x 128 B = 107 KB
  size_t smem = (size_t)nrows * 128;
  CK(cudaFuncSetAttribute(k_lds<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_lds<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_lds<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  double lds_gbs[3];
  int lblocks = nsm * 2, lthreads = 512, liters = 8192;
  for (int m = 0; m < 3; ++m) {
    auto run = [&](int it) {
      if (m == 0) k_lds<0><<<lblocks, lthreads, smem>>>(uout, it, nrows);
      if (m == 1) k_lds<1><<<lblocks, lthreads, smem>>>(uout, it, nrows);
      if (m == 2) k_lds<2><<<lblocks, lthreads, smem>>>(uout, it, nrows);
    };
    run(16); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); run(liters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double bytes = (double)lblocks * lthreads * liters * 8 * 16;
    lds_gbs[m] = bytes / (ms * 1e-3) / 1e9;
  }

  // L2 gather: rows of 6 sectors (R = 24 doubles) over the C4 factor size (3 x 16384 rows,
  // 9.4 MB) and rows of 4 sectors (R = 16) over the C3 size (3 x 4096 rows, 1.6 MB)
  double l2_cg_gbs[2], l2_nc_gbs[2];
  const uint32_t rows_l2[2] = {3u * 16384u, 3u * 4096u};
  double4* tab; CK(cudaMalloc(&tab, (size_t)rows_l2[0] * 6 * 32));
  CK(cudaMemset(tab, 0, (size_t)rows_l2[0] * 6 * 32));
  for (int m = 0; m < 2; ++m) {
    for (int cg = 0; cg < 2; ++cg) {
      int gb = nsm * 4, gt = 512, gi = 1024;
      auto run = [&](int it) {
        if (m == 0 && cg) k_l2gather<6, 1><<<gb, gt>>>(tab, uout, it, rows_l2[m]);
        if (m == 0 && !cg) k_l2gather<6, 0><<<gb, gt>>>(tab, uout, it, rows_l2[m]);
        if (m == 1 && cg) k_l2gather<4, 1><<<gb, gt>>>(tab, uout, it, rows_l2[m]);
        if (m == 1 && !cg) k_l2gather<4, 0><<<gb, gt>>>(tab, uout, it, rows_l2[m]);
      };
      run(16); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0); run(gi); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      const double g = (double)gb * gt * gi * (m == 0 ? 6 : 4) * 32 / (ms * 1e-3) / 1e9;
      (cg ? l2_cg_gbs : l2_nc_gbs)[m] = g;
    }
  }
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_rate_khz_attr\": %d, "
         "\"dfma_instr_per_s\": %.6e, \"fp64_tflops\": %.4f, "
         "\"lds128_conflict_free_gbs\": %.1f, \"lds128_random_row_unrotated_gbs\": %.1f, "
         "\"lds128_random_row_rotated_gbs\": %.1f, "
         "\"l2_gather_cg_9p4MB_gbs\": %.1f, \"l2_gather_cg_1p6MB_gbs\": %.1f, "
         "\"l2_gather_nc_9p4MB_gbs\": %.1f, \"l2_gather_nc_1p6MB_gbs\": %.1f, "
         "\"l2_bytes\": %d, \"smem_per_block_optin\": %zu}\n",
         p.name, nsm, clk_khz, dfma_per_s, 2 * dfma_per_s / 1e12, lds_gbs[0], lds_gbs[1], lds_gbs[2],
         l2_cg_gbs[0], l2_cg_gbs[1], l2_nc_gbs[0], l2_nc_gbs[1], p.l2CacheSize, p.sharedMemPerBlockOptin);
  return 0;
}
