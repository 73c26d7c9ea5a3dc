// Probe: 3-D TMA tensor copy (uint32, cd^3 box, negative/out-of-range coordinates zero-filled)
// of a packed table, through cuTensorMapEncodeTiled from the runtime's driver entry point.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <cstdint>
#include <cstdlib>
typedef CUresult (*PFN_enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                            const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                            CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap m, int c0, int c1, int c2, int cd, unsigned* out) {
  extern __shared__ __align__(128) unsigned sm[];
  __shared__ __align__(8) uint64_t bar;
  const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar), sd = (unsigned)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"((unsigned)(cd * cd * cd * 4)));
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(sd), "l"(reinterpret_cast<uint64_t>(&m)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(sb) : "memory");
  }
  __syncthreads();
  asm volatile("{\n .reg .pred p;\n W:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(sb));
  for (int i = threadIdx.x; i < cd * cd * cd; i += blockDim.x) out[i] = sm[i];
}
int main(int argc, char** argv) {
  const int X = 30, Y = 25, Z = 22, Zp = 24; const int cd = argc > 1 ? atoi(argv[1]) : 20;
  unsigned* h = new unsigned[X * Y * Zp];
  for (int x = 0; x < X; ++x) for (int y = 0; y < Y; ++y) for (int z = 0; z < Zp; ++z)
    h[(x * Y + y) * Zp + z] = z < Z ? (unsigned)((x << 20) | (y << 10) | z) + 1u : 0u;
  unsigned *d, *o;
  cudaMalloc(&d, X * Y * Zp * 4); cudaMalloc(&o, cd * cd * cd * 4);
  cudaMemcpy(d, h, X * Y * Zp * 4, cudaMemcpyHostToDevice);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  PFN_enc enc = (PFN_enc)p;
  CUtensorMap m; memset(&m, 0, sizeof m);
  cuuint64_t dims[3] = {(cuuint64_t)Zp, (cuuint64_t)Y, (cuuint64_t)X};
  cuuint64_t str[2] = {(cuuint64_t)Zp * 4, (cuuint64_t)Zp * Y * 4};
  cuuint32_t box[3] = {cd, cd, cd}, es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  const int c0 = argc > 2 ? atoi(argv[2]) : -3, c1 = 2, c2 = 3;   // z, y, x origin
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, cd * cd * cd * 4);
  k<<<1, 256, cd * cd * cd * 4>>>(m, c0, c1, c2, cd, o);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  unsigned* ho = new unsigned[cd * cd * cd];
  cudaMemcpy(ho, o, cd * cd * cd * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < cd; ++i) for (int j = 0; j < cd; ++j) for (int l = 0; l < cd; ++l) {
    const int x = c2 + i, y = c1 + j, z = c0 + l;
    const unsigned want = (x >= 0 && x < X && y >= 0 && y < Y && z >= 0 && z < Zp) ? h[(x * Y + y) * Zp + z] : 0u;
    if (ho[(i * cd + j) * cd + l] != want) ++bad;
  }
  printf("mismatches %d\n", bad);
  return 0;
}
