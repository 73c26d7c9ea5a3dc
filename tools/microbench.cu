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

// mode 0: 4 rows per warp (one per quarter-warp), lane-rotated chunks (conflict-free)
// mode 1: random row per lane, chunk c same for all lanes (unrotated)
// mode 2: random row per lane, chunk (c + lane) & 7 (rotated)
template <int MODE>
__global__ void k_lds(unsigned long long* out, int iters, int nrows) {
  extern __shared__ double4 sm4[];
  double2* sm = reinterpret_cast<double2*>(sm4);
  for (int i = threadIdx.x; i < nrows * 8; i += blockDim.x) sm[i] = make_double2(i, i + 1);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t st = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x * 7919u;
  double acc0 = 0, acc1 = 0;
  for (int it = 0; it < iters; ++it) {
    st = st * 1664525u + 1013904223u;
    int row = (MODE == 0) ? (((lane >> 3) + it * 4) % nrows) : (int)((st >> 8) % (uint32_t)nrows);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      int ch = (MODE == 1) ? c : ((c + lane) & 7);
      double2 v = sm[row * 8 + ch];
      acc0 += v.x; acc1 += v.y;
    }
  }
  if (acc0 + acc1 == -1.0) out[blockIdx.x] = 1;
}

__global__ void k_l2gather(const double2* __restrict__ tab, unsigned long long* out, int iters,
                           uint32_t nrows) {
  const int lane = threadIdx.x & 31;
  uint32_t st = 0x9E3779B9u * (threadIdx.x + 1 + blockIdx.x * blockDim.x);
  double acc0 = 0, acc1 = 0;
  for (int it = 0; it < iters; ++it) {
    st = st * 1664525u + 1013904223u;
    uint32_t row = (st >> 4) % nrows;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      double2 v = __ldg(&tab[(size_t)row * 8 + ((c + lane) & 7)]);
      acc0 += v.x; acc1 += v.y;
    }
  }
  if (acc0 + acc1 == -1.0) out[blockIdx.x] = 1;
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

  // L2 gather over 1.5 MB (C3 factors) and 9.4 MB (C4 factors) tables
  double l2_gbs[2]; uint32_t rows_l2[2] = {12288, 73728};
  double2* tab; CK(cudaMalloc(&tab, (size_t)rows_l2[1] * 128));
  CK(cudaMemset(tab, 0, (size_t)rows_l2[1] * 128));
  for (int m = 0; m < 2; ++m) {
    int gb = nsm * 8, gt = 256, gi = 2048;
    k_l2gather<<<gb, gt>>>(tab, uout, 16, rows_l2[m]); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_l2gather<<<gb, gt>>>(tab, uout, gi, rows_l2[m]);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    l2_gbs[m] = (double)gb * gt * gi * 8 * 16 / (ms * 1e-3) / 1e9;
  }
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_rate_khz_attr\": %d, "
         "\"dfma_instr_per_s\": %.6e, \"fp64_tflops\": %.4f, "
         "\"lds128_conflict_free_gbs\": %.1f, \"lds128_random_row_unrotated_gbs\": %.1f, "
         "\"lds128_random_row_rotated_gbs\": %.1f, "
         "\"l2_gather_1p5MB_gbs\": %.1f, \"l2_gather_9p4MB_gbs\": %.1f, "
         "\"l2_bytes\": %d, \"smem_per_block_optin\": %zu}\n",
         p.name, nsm, clk_khz, dfma_per_s, 2 * dfma_per_s / 1e12, lds_gbs[0], lds_gbs[1], lds_gbs[2],
         l2_gbs[0], l2_gbs[1], p.l2CacheSize, p.sharedMemPerBlockOptin);
  return 0;
}
