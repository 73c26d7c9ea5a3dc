// Probe: does __reduce_min_sync with per-group masks (disjoint, covering the warp) compute
// per-group minima in one converged call?  Prints mismatches (0 expected).
#include <cstdio>
__global__ void k(const unsigned* v, const unsigned* grp, unsigned* out) {
  const int lane = threadIdx.x & 31;
  const unsigned g = grp[lane];
  const unsigned m = __match_any_sync(0xffffffffu, g);
  out[lane] = __reduce_min_sync(m, v[lane]);
}
int main() {
  unsigned hv[32], hg[32], ho[32];
  unsigned *dv, *dg, *dout;
  cudaMalloc(&dv, 128); cudaMalloc(&dg, 128); cudaMalloc(&dout, 128);
  int bad = 0;
  for (int trial = 0; trial < 200; ++trial) {
    unsigned s = 12345 + trial * 777;
    int seg = 0;
    for (int i = 0; i < 32; ++i) {
      s = s * 1664525u + 1013904223u;
      hv[i] = s >> 3;
      if (i > 0 && ((s >> 28) & 3) == 0) ++seg;   // contiguous segments
      hg[i] = seg;
    }
    cudaMemcpy(dv, hv, 128, cudaMemcpyHostToDevice);
    cudaMemcpy(dg, hg, 128, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(dv, dg, dout);
    cudaMemcpy(ho, dout, 128, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 32; ++i) {
      unsigned mn = 0xffffffffu;
      for (int j = 0; j < 32; ++j) if (hg[j] == hg[i] && hv[j] < mn) mn = hv[j];
      if (ho[i] != mn) ++bad;
    }
  }
  printf("redux per-group mismatches: %d\n", bad);
  return 0;
}
