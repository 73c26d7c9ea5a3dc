// NEXT row N4 (part): step S6 of the setup (Algorithm TEP), the Tucker core
// G[a,b,c] = sum_k sum_m (z_m a_k H0_k[i_m0, a]) H1_k[i_m1, b] H2_k[i_m2, c] of the long-range
// part, on the device.  Each thread owns one core entry and runs the host loop's exact op
// sequence (per k: row = 0; for m in order: w = (z_m a_k) H0, skipped when 0, wb = w H1,
// row += wb H2; then G += row), compiled with -fmad=false like the host's -ffp-contract=off,
// so the core -- and every table built from it -- is bitwise the host-only build's.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "rs_internal.h"

namespace rs {
namespace {

__global__ void core_k_kernel(int r0, int r1, int r2, int64_t M, const int* cells, const double* z,
                              double ak, const double* H0, const double* H1, const double* H2,
                              double* G) {
  const int a = blockIdx.x / r1, b = blockIdx.x % r1;
  for (int c = threadIdx.x; c < r2; c += blockDim.x) {
    double row = 0.0;
    for (int64_t m = 0; m < M; ++m) {
      const double w = __dmul_rn(__dmul_rn(z[m], ak), H0[(size_t)cells[3 * m] * r0 + a]);
      if (w == 0.0) continue;
      const double wb = __dmul_rn(w, H1[(size_t)cells[3 * m + 1] * r1 + b]);
      row = __dadd_rn(row, __dmul_rn(wb, H2[(size_t)cells[3 * m + 2] * r2 + c]));
    }
    double* g = G + ((size_t)a * r1 + b) * r2 + c;
    *g = __dadd_rn(*g, row);
  }
}

}  // namespace

struct CoreDevice::Impl {
  int device = 0, r[3] = {0, 0, 0}, n = 0;
  int64_t M = 0;
  int* cells = nullptr;
  double *z = nullptr, *H[3] = {nullptr, nullptr, nullptr}, *G = nullptr;
  bool ok = false;
};

CoreDevice::CoreDevice(int device, int n, const int* r, const std::vector<int32_t>& cells,
                       const std::vector<double>& z)
    : p(new Impl) {
  p->device = device;
  p->n = n;
  p->M = (int64_t)z.size();
  for (int l = 0; l < 3; ++l) p->r[l] = r[l];
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) { cudaGetLastError(); return; }
  bool good = cudaMalloc(&p->cells, std::max<size_t>(1, cells.size()) * sizeof(int)) == cudaSuccess &&
              cudaMalloc(&p->z, std::max<size_t>(1, z.size()) * sizeof(double)) == cudaSuccess &&
              cudaMalloc(&p->G, (size_t)r[0] * r[1] * r[2] * sizeof(double)) == cudaSuccess;
  for (int l = 0; l < 3 && good; ++l)
    good = cudaMalloc(&p->H[l], (size_t)n * r[l] * sizeof(double)) == cudaSuccess;
  good = good && cudaMemcpy(p->cells, cells.data(), cells.size() * sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(p->z, z.data(), z.size() * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemset(p->G, 0, (size_t)r[0] * r[1] * r[2] * sizeof(double)) == cudaSuccess;
  p->ok = good;
  if (!good) cudaGetLastError();
  cudaSetDevice(prev);
}

CoreDevice::~CoreDevice() {
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  cudaFree(p->cells);
  cudaFree(p->z);
  cudaFree(p->G);
  for (double* h : p->H) cudaFree(h);
  cudaSetDevice(prev);
  delete p;
}

bool CoreDevice::ok() const { return p->ok; }

bool CoreDevice::add_term(double a_k, const std::vector<double> H[3]) {
  if (!p->ok) return false;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  bool good = true;
  for (int l = 0; l < 3 && good; ++l)
    good = cudaMemcpy(p->H[l], H[l].data(), H[l].size() * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess;
  if (good) {
    const int threads = std::min(256, ((p->r[2] + 31) / 32) * 32);
    core_k_kernel<<<p->r[0] * p->r[1], threads>>>(p->r[0], p->r[1], p->r[2], p->M, p->cells, p->z, a_k,
                                                 p->H[0], p->H[1], p->H[2], p->G);
    good = cudaGetLastError() == cudaSuccess;
  }
  if (!good) { cudaGetLastError(); p->ok = false; }
  cudaSetDevice(prev);
  return good;
}

bool CoreDevice::fetch(std::vector<double>& G) {
  if (!p->ok) return false;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  G.assign((size_t)p->r[0] * p->r[1] * p->r[2], 0.0);
  const bool good = cudaMemcpy(G.data(), p->G, G.size() * sizeof(double), cudaMemcpyDeviceToHost) == cudaSuccess;
  if (!good) cudaGetLastError();
  cudaSetDevice(prev);
  return good;
}

}  // namespace rs

// ---- opt-in (RS_FLAG_DEVICE_FFT): the setup's convolutions y = T_k x on the device (cuFFT) ---
#include <cufft.h>
#include <mutex>

namespace rs {
namespace {

__global__ void pack_pairs(const double* X, int n, int N, int p, cufftDoubleComplex* buf) {
  const int pairs = (p + 1) / 2;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)pairs * N;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(t / N), i = (int)(t % N), s = 2 * q;
    cufftDoubleComplex v;
    v.x = i < n ? X[(size_t)s * n + i] : 0.0;
    v.y = (i < n && s + 1 < p) ? X[(size_t)(s + 1) * n + i] : 0.0;
    buf[t] = v;
  }
}

__global__ void mul_kernel(cufftDoubleComplex* buf, const cufftDoubleComplex* fg, int N, int pairs) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)pairs * N;
       t += (int64_t)gridDim.x * blockDim.x) {
    const cufftDoubleComplex a = buf[t], b = fg[t % N];
    cufftDoubleComplex c;
    c.x = a.x * b.x - a.y * b.y;
    c.y = a.x * b.y + a.y * b.x;
    buf[t] = c;
  }
}

__global__ void unpack_pairs(const cufftDoubleComplex* buf, int n, int N, int p, double* Y) {
  const double inv = 1.0 / N;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)p * n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(t / n), i = (int)(t % n);
    const cufftDoubleComplex v = buf[(size_t)(s / 2) * N + i + n - 1];
    Y[t] = ((s & 1) ? v.y : v.x) * inv;
  }
}

// S6 accumulation for the device-FFT path, split over atoms: block (a, chunk) adds
// sum_{m in chunk} (z_m a_k H0[m,a]) H1[m,b] H2[m,c] for all (b, c) into its partial; atoms in
// ascending order, the chunks' partials summed in ascending order by core_reduce_kernel, so the
// core is deterministic (not bitwise the per-entry loop's order: device-FFT builds are
// validated by their accuracy)
constexpr int kCoreChunk = 512, kCoreSub = 64;
__global__ void core_chunk_kernel(int r0, int r1, int r2, int64_t M, const int* __restrict__ cells,
                                  const double* __restrict__ z, double ak, const double* __restrict__ H0,
                                  const double* __restrict__ H1, const double* __restrict__ H2,
                                  double* __restrict__ part) {
  extern __shared__ double sm[];
  double* sw = sm;                         // kCoreSub weights
  double* s1 = sm + kCoreSub;              // kCoreSub x r1
  double* s2 = s1 + (size_t)kCoreSub * r1; // kCoreSub x r2
  const int a = blockIdx.x % r0, chunk = blockIdx.x / r0;
  const int64_t m0 = (int64_t)chunk * kCoreChunk, m1 = min(M, m0 + kCoreChunk);
  const int nout = r1 * r2;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t mb = m0; mb < m1; mb += kCoreSub) {
    const int cnt = (int)min((int64_t)kCoreSub, m1 - mb);
    __syncthreads();
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
      const int64_t m = mb + t;
      sw[t] = __dmul_rn(__dmul_rn(z[m], ak), H0[(size_t)cells[3 * m] * r0 + a]);
    }
    for (int t = threadIdx.x; t < cnt * r1; t += blockDim.x) {
      const int u = t / r1, b = t % r1;
      s1[t] = H1[(size_t)cells[3 * (mb + u) + 1] * r1 + b];
    }
    for (int t = threadIdx.x; t < cnt * r2; t += blockDim.x) {
      const int u = t / r2, c = t % r2;
      s2[t] = H2[(size_t)cells[3 * (mb + u) + 2] * r2 + c];
    }
    __syncthreads();
    for (int u = 0; u < cnt; ++u) {
      const double w = sw[u];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int idx = threadIdx.x + j * blockDim.x;
        if (idx < nout) {
          const int b = idx / r2, c = idx % r2;
          acc[j] = __dadd_rn(acc[j], __dmul_rn(__dmul_rn(w, s1[u * r1 + b]), s2[u * r2 + c]));
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int idx = threadIdx.x + j * blockDim.x;
    if (idx < nout) part[((size_t)chunk * r0 + a) * nout + idx] = acc[j];
  }
}

__global__ void core_reduce_kernel(int nchunk, int64_t ng, const double* __restrict__ part, double* G) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ng; t += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < nchunk; ++c) s = __dadd_rn(s, part[(size_t)c * ng + t]);
    G[t] = __dadd_rn(G[t], s);
  }
}

// the same values transposed: Yr row-major n x p (row i holds the p columns at i)
__global__ void unpack_pairs_rows(const cufftDoubleComplex* buf, int n, int N, int p, double* Yr) {
  const double inv = 1.0 / N;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)p * n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t / p), s = (int)(t % p);
    const cufftDoubleComplex v = buf[(size_t)(s / 2) * N + i + n - 1];
    Yr[t] = ((s & 1) ? v.y : v.x) * inv;
  }
}

}  // namespace

struct DeviceConv::Impl {
  int device = 0, n = 0, N = 0, RL = 0;
  cufftDoubleComplex* fg = nullptr;
  cufftDoubleComplex* buf = nullptr;
  double *X = nullptr, *Y = nullptr;
  size_t cap_pairs = 0, cap_xy = 0;
  cufftHandle plan = 0;
  int plan_batch = 0;
  bool ok = false;
  std::mutex mtx;
};

DeviceConv::DeviceConv(int device, int n, int N, const std::vector<std::vector<std::complex<double>>>& FG)
    : p(new Impl) {
  p->device = device;
  p->n = n;
  p->N = N;
  p->RL = (int)FG.size();
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) { cudaGetLastError(); return; }
  bool good = cudaMalloc(&p->fg, (size_t)p->RL * N * sizeof(cufftDoubleComplex)) == cudaSuccess;
  for (int k = 0; k < p->RL && good; ++k)
    good = cudaMemcpy(p->fg + (size_t)k * N, FG[k].data(), (size_t)N * sizeof(cufftDoubleComplex),
                      cudaMemcpyHostToDevice) == cudaSuccess;
  p->ok = good;
  if (!good) cudaGetLastError();
  cudaSetDevice(prev);
}

DeviceConv::~DeviceConv() {
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  if (p->plan) cufftDestroy(p->plan);
  cudaFree(p->fg);
  cudaFree(p->buf);
  cudaFree(p->X);
  cudaFree(p->Y);
  cudaSetDevice(prev);
  delete p;
}

bool DeviceConv::ok() const { return p->ok; }

bool DeviceConv::apply(int k, const double* X, double* Y, int cols) {
  std::lock_guard<std::mutex> lock(p->mtx);
  if (!p->ok) return false;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  const int n = p->n, N = p->N, pairs = (cols + 1) / 2;
  bool good = true;
  if ((size_t)pairs > p->cap_pairs) {
    cudaFree(p->buf);
    good = cudaMalloc(&p->buf, (size_t)pairs * N * sizeof(cufftDoubleComplex)) == cudaSuccess;
    p->cap_pairs = good ? pairs : 0;
  }
  if (good && (size_t)cols * n > p->cap_xy) {
    cudaFree(p->X);
    cudaFree(p->Y);
    good = cudaMalloc(&p->X, (size_t)cols * n * sizeof(double)) == cudaSuccess &&
           cudaMalloc(&p->Y, (size_t)cols * n * sizeof(double)) == cudaSuccess;
    p->cap_xy = good ? (size_t)cols * n : 0;
  }
  if (good && p->plan_batch != pairs) {
    if (p->plan) cufftDestroy(p->plan);
    p->plan = 0;
    good = cufftPlan1d(&p->plan, N, CUFFT_Z2Z, pairs) == CUFFT_SUCCESS;
    p->plan_batch = good ? pairs : 0;
  }
  good = good && cudaMemcpy(p->X, X, (size_t)cols * n * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess;
  if (good) {
    pack_pairs<<<1184, 256>>>(p->X, n, N, cols, p->buf);
    good = cufftExecZ2Z(p->plan, p->buf, p->buf, CUFFT_FORWARD) == CUFFT_SUCCESS;
  }
  if (good) {
    mul_kernel<<<1184, 256>>>(p->buf, p->fg + (size_t)k * N, N, pairs);
    good = cufftExecZ2Z(p->plan, p->buf, p->buf, CUFFT_INVERSE) == CUFFT_SUCCESS;
  }
  if (good) {
    unpack_pairs<<<1184, 256>>>(p->buf, n, N, cols, p->Y);
    good = cudaMemcpy(Y, p->Y, (size_t)cols * n * sizeof(double), cudaMemcpyDeviceToHost) == cudaSuccess;
  }
  if (!good) { cudaGetLastError(); p->ok = false; }
  cudaSetDevice(prev);
  return good;
}

}  // namespace rs

// ---- sampled compression error (setup report) on the device ----------------------------
// The uncompressed long-range value at each sample cell c: sum_m z_m sum_k a_k g_k[|c0 - i_m0|]
// g_k[|c1 - i_m1|] g_k[|c2 - i_m2|] (Eq. (6)); one block per sample, threads over the protein
// atoms, a fixed shared-memory tree per block (deterministic).  Only the reported error uses it.
namespace rs {
namespace {

__global__ void exact_long_kernel(int n, int RL, int64_t M, const double* __restrict__ G,
                                  const double* __restrict__ a, const int* __restrict__ cells,
                                  const double* __restrict__ z, const int* __restrict__ pts,
                                  double* __restrict__ out) {
  __shared__ double red[256];
  const int s = blockIdx.x;
  const int c0 = pts[3 * s], c1 = pts[3 * s + 1], c2 = pts[3 * s + 2];
  double v = 0.0;
  for (int64_t m = threadIdx.x; m < M; m += blockDim.x) {
    const int d0 = abs(c0 - cells[3 * m]), d1 = abs(c1 - cells[3 * m + 1]), d2 = abs(c2 - cells[3 * m + 2]);
    double acc = 0.0;
    for (int k = 0; k < RL; ++k) {
      const double* g = G + (size_t)k * n;
      acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(__dmul_rn(a[k], __ldg(g + d0)), __ldg(g + d1)), __ldg(g + d2)));
    }
    v = __dadd_rn(v, __dmul_rn(z[m], acc));
  }
  red[threadIdx.x] = v;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + off]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[s] = red[0];
}

}  // namespace

bool exact_long_values_device(int device, int n, const std::vector<double>& G,
                              const std::vector<double>& a_long, const std::vector<int32_t>& cells,
                              const std::vector<double>& z, const std::vector<int>& pts,
                              std::vector<double>& out) {
  const int RL = (int)a_long.size();
  const int64_t M = (int64_t)z.size();
  const int ns = (int)pts.size() / 3;
  out.assign(ns, 0.0);
  if (ns == 0) return true;
  int prev = 0;
  if (cudaGetDevice(&prev) != cudaSuccess || cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  double *dG = nullptr, *da = nullptr, *dz = nullptr, *dout = nullptr;
  int *dc = nullptr, *dp = nullptr;
  bool ok = cudaMalloc(&dG, G.size() * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&da, RL * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&dz, M * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&dout, ns * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&dc, cells.size() * sizeof(int)) == cudaSuccess &&
            cudaMalloc(&dp, pts.size() * sizeof(int)) == cudaSuccess;
  ok = ok && cudaMemcpy(dG, G.data(), G.size() * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMemcpy(da, a_long.data(), RL * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMemcpy(dz, z.data(), M * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMemcpy(dc, cells.data(), cells.size() * sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMemcpy(dp, pts.data(), pts.size() * sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess;
  if (ok) {
    exact_long_kernel<<<ns, 256>>>(n, RL, M, dG, da, dc, dz, dp, dout);
    ok = cudaGetLastError() == cudaSuccess &&
         cudaMemcpy(out.data(), dout, ns * sizeof(double), cudaMemcpyDeviceToHost) == cudaSuccess;
  }
  for (void* q : {(void*)dG, (void*)da, (void*)dz, (void*)dout, (void*)dc, (void*)dp})
    if (q) cudaFree(q);
  cudaGetLastError();
  cudaSetDevice(prev);
  return ok;
}

}  // namespace rs

// ---- S6 end to end on the device ------------------------------------------------------------
namespace rs {

bool CoreDevice::add_terms_device(DeviceConv& conv, const std::vector<double> U[3],
                                  const std::vector<double>& a_long) {
  if (!p->ok || !conv.p->ok || conv.p->device != p->device || conv.p->n != p->n) return false;
  std::lock_guard<std::mutex> lock(conv.p->mtx);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  const int n = p->n, N = conv.p->N;
  int maxr = std::max(p->r[0], std::max(p->r[1], p->r[2]));
  const int maxpairs = (maxr + 1) / 2;
  double* dU[3] = {nullptr, nullptr, nullptr};
  cufftDoubleComplex* buf = nullptr;
  cufftHandle plans[3] = {0, 0, 0};
  const int64_t ng = (int64_t)p->r[0] * p->r[1] * p->r[2];
  double* part = nullptr;
  bool good = p->r[1] * p->r[2] <= 1024 &&
              cudaMalloc(&buf, (size_t)maxpairs * N * sizeof(cufftDoubleComplex)) == cudaSuccess &&
              cudaMalloc(&part, (size_t)((p->M + kCoreChunk - 1) / kCoreChunk) * ng * sizeof(double)) == cudaSuccess;
  for (int l = 0; l < 3 && good; ++l) {
    good = cudaMalloc(&dU[l], (size_t)n * p->r[l] * sizeof(double)) == cudaSuccess &&
           cudaMemcpy(dU[l], U[l].data(), (size_t)n * p->r[l] * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess &&
           cufftPlan1d(&plans[l], N, CUFFT_Z2Z, (p->r[l] + 1) / 2) == CUFFT_SUCCESS;
  }
  const bool timing = std::getenv("RS_SETUP_TIMING") != nullptr;
  cudaEvent_t ev[2];
  float t_conv = 0.f, t_acc = 0.f;
  if (timing) { cudaEventCreate(&ev[0]); cudaEventCreate(&ev[1]); }
  for (int k = 0; k < (int)a_long.size() && good; ++k) {
    if (timing) cudaEventRecord(ev[0]);
    for (int l = 0; l < 3 && good; ++l) {
      const int r = p->r[l], pairs = (r + 1) / 2;
      pack_pairs<<<1184, 256>>>(dU[l], n, N, r, buf);
      good = cufftExecZ2Z(plans[l], buf, buf, CUFFT_FORWARD) == CUFFT_SUCCESS;
      if (good) {
        mul_kernel<<<1184, 256>>>(buf, conv.p->fg + (size_t)k * N, N, pairs);
        good = cufftExecZ2Z(plans[l], buf, buf, CUFFT_INVERSE) == CUFFT_SUCCESS;
      }
      if (good) unpack_pairs_rows<<<1184, 256>>>(buf, n, N, r, p->H[l]);
    }
    if (timing) {
      float ms = 0.f;
      cudaEventRecord(ev[1]);
      cudaEventSynchronize(ev[1]);
      cudaEventElapsedTime(&ms, ev[0], ev[1]);
      t_conv += ms;
      cudaEventRecord(ev[0]);
    }
    if (good) {
      const int nchunk = (int)((p->M + kCoreChunk - 1) / kCoreChunk);
      const size_t shm = (size_t)kCoreSub * (1 + p->r[1] + p->r[2]) * sizeof(double);
      core_chunk_kernel<<<nchunk * p->r[0], 256, shm>>>(p->r[0], p->r[1], p->r[2], p->M, p->cells, p->z,
                                                        a_long[k], p->H[0], p->H[1], p->H[2], part);
      core_reduce_kernel<<<256, 256>>>(nchunk, ng, part, p->G);
      good = cudaGetLastError() == cudaSuccess;
    }
    if (timing) {
      float ms = 0.f;
      cudaEventRecord(ev[1]);
      cudaEventSynchronize(ev[1]);
      cudaEventElapsedTime(&ms, ev[0], ev[1]);
      t_acc += ms;
    }
  }
  if (timing) {
    std::fprintf(stderr, "[rs setup]     core on the device: convolutions %.3f s, accumulation %.3f s\n",
                 t_conv * 1e-3, t_acc * 1e-3);
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
  }
  good = good && cudaDeviceSynchronize() == cudaSuccess;
  for (int l = 0; l < 3; ++l) {
    if (plans[l]) cufftDestroy(plans[l]);
    cudaFree(dU[l]);
  }
  cudaFree(buf);
  cudaFree(part);
  if (!good) { cudaGetLastError(); p->ok = false; }
  cudaSetDevice(prev);
  return good;
}

}  // namespace rs

