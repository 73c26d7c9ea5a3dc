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

// ---- the RHOSVD range finder's convolutions on the device ------------------------------------
namespace rs {
namespace {

__device__ __forceinline__ uint64_t splitmix_dev(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
// la::normal (setup_linalg.cpp) on the device: the same counter-based draws (Box-Muller of two
// splitmix64 uniforms; device log/cos, so the last bits may differ from the host's libm)
__device__ __forceinline__ double normal_dev(uint64_t seed, uint64_t i) {
  const uint64_t a = splitmix_dev(seed * 0x100000001B3ull + 2 * i);
  const uint64_t b = splitmix_dev(seed * 0x100000001B3ull + 2 * i + 1);
  const double u1 = (double((a >> 11) + 1)) * (1.0 / 9007199254740993.0);
  const double u2 = double(b >> 11) * (1.0 / 9007199254740992.0);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

// X (n x p column-major) = sqrt(c_k[j]) xi_{k,j,s} at occupied rows j, 0 elsewhere
__global__ void sketch_kernel(int n, int p, int k, const double* __restrict__ c, const unsigned char* __restrict__ occ,
                              uint64_t seed, double* __restrict__ X) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)n * p;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(t / n), j = (int)(t % n);
    X[t] = occ[j] ? sqrt(c[j]) * normal_dev(seed, ((uint64_t)k * n + j) * 4096u + s) : 0.0;
  }
}
__global__ void add_kernel(int64_t len, const double* __restrict__ A, double* __restrict__ Y) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < len; t += (int64_t)gridDim.x * blockDim.x)
    Y[t] += A[t];
}
__global__ void scale_rows_kernel(int n, int p, const double* __restrict__ c, double* __restrict__ Z) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)n * p;
       t += (int64_t)gridDim.x * blockDim.x)
    Z[t] *= c[t % n];
}
// partial weighted Gram of Z (n x p column-major) over a fixed row block: G[s][t] (s <= t) =
// sum_{j in block} c[j] Z[s][j] Z[t][j]; blocks summed in order on the host
__global__ void wgram_kernel(int n, int p, int nblk, const double* __restrict__ c, const double* __restrict__ Z,
                             double* __restrict__ part) {
  const int blk = blockIdx.y;
  const int j0 = (int)((int64_t)n * blk / nblk), j1 = (int)((int64_t)n * (blk + 1) / nblk);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < p * p; e += gridDim.x * blockDim.x) {
    const int s = e / p, t = e % p;
    double g = 0.0;
    if (s <= t)
      for (int j = j0; j < j1; ++j) {
        const double w = c[j];
        if (w != 0.0) g += w * Z[(size_t)s * n + j] * Z[(size_t)t * n + j];
      }
    part[(size_t)blk * p * p + e] = g;
  }
}

}  // namespace

struct RangeFinderDevice::Impl {
  DeviceConv* conv = nullptr;
  int n = 0, RL = 0, cap = 0;
  double *c = nullptr, *X = nullptr, *Y = nullptr, *Z = nullptr, *W = nullptr, *part = nullptr;
  unsigned char* occ = nullptr;
  cufftDoubleComplex* buf = nullptr;
  cufftHandle plan = 0;
  int plan_pairs = 0;
  bool ok = false;
};

RangeFinderDevice::RangeFinderDevice(DeviceConv& conv, const std::vector<std::vector<double>>& c, int n)
    : q(new Impl) {
  q->conv = &conv;
  q->n = n;
  q->RL = (int)c.size();
  if (!conv.p->ok || conv.p->n != n) return;
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(conv.p->device) != cudaSuccess) { cudaGetLastError(); return; }
  bool good = cudaMalloc(&q->c, (size_t)q->RL * n * sizeof(double)) == cudaSuccess &&
              cudaMalloc(&q->occ, n) == cudaSuccess;
  for (int k = 0; k < q->RL && good; ++k)
    good = cudaMemcpy(q->c + (size_t)k * n, c[k].data(), n * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess;
  q->ok = good;
  if (!good) cudaGetLastError();
  cudaSetDevice(prev);
}

RangeFinderDevice::~RangeFinderDevice() {
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(q->conv->p->device);
  if (q->plan) cufftDestroy(q->plan);
  for (void* x : {(void*)q->c, (void*)q->X, (void*)q->Y, (void*)q->Z, (void*)q->W, (void*)q->part,
                  (void*)q->occ, (void*)q->buf})
    if (x) cudaFree(x);
  cudaSetDevice(prev);
  delete q;
}

bool RangeFinderDevice::ok() const { return q->ok; }

bool RangeFinderDevice::reserve(int p) {
  const int n = q->n, N = q->conv->p->N, pairs = (p + 1) / 2;
  if (p > q->cap) {
    for (double** b : {&q->X, &q->Y, &q->Z, &q->W}) {
      cudaFree(*b);
      *b = nullptr;
      if (cudaMalloc(b, (size_t)n * p * sizeof(double)) != cudaSuccess) { cudaGetLastError(); return false; }
    }
    cudaFree(q->buf);
    q->buf = nullptr;
    if (cudaMalloc(&q->buf, (size_t)pairs * N * sizeof(cufftDoubleComplex)) != cudaSuccess) { cudaGetLastError(); return false; }
    cudaFree(q->part);
    q->part = nullptr;
    if (cudaMalloc(&q->part, (size_t)64 * p * p * sizeof(double)) != cudaSuccess) { cudaGetLastError(); return false; }
    q->cap = p;
  }
  if (q->plan_pairs != pairs) {
    if (q->plan) cufftDestroy(q->plan);
    q->plan = 0;
    if (cufftPlan1d(&q->plan, N, CUFFT_Z2Z, pairs) != CUFFT_SUCCESS) { q->plan_pairs = 0; return false; }
    q->plan_pairs = pairs;
  }
  return true;
}

// dY = T_k dX with the same kernels and FFT-domain product as DeviceConv::apply
bool RangeFinderDevice::apply(int k, const double* dX, double* dY, int p) {
  const int n = q->n, N = q->conv->p->N, pairs = (p + 1) / 2;
  pack_pairs<<<1184, 256>>>(dX, n, N, p, q->buf);
  if (cufftExecZ2Z(q->plan, q->buf, q->buf, CUFFT_FORWARD) != CUFFT_SUCCESS) return false;
  mul_kernel<<<1184, 256>>>(q->buf, q->conv->p->fg + (size_t)k * N, N, pairs);
  if (cufftExecZ2Z(q->plan, q->buf, q->buf, CUFFT_INVERSE) != CUFFT_SUCCESS) return false;
  unpack_pairs<<<1184, 256>>>(q->buf, n, N, p, dY);
  return cudaGetLastError() == cudaSuccess;
}

bool RangeFinderDevice::sketch(int p, uint64_t seed, int mode, const std::vector<int>& occj, std::vector<double>& Y) {
  if (!q->ok) return false;
  std::lock_guard<std::mutex> lock(q->conv->p->mtx);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(q->conv->p->device);
  const int n = q->n;
  bool good = reserve(p);
  if (good) {
    std::vector<unsigned char> occ(n, 0);
    for (int j : occj) occ[j] = 1;
    good = cudaMemcpy(q->occ, occ.data(), n, cudaMemcpyHostToDevice) == cudaSuccess &&
           cudaMemset(q->Y, 0, (size_t)n * p * sizeof(double)) == cudaSuccess;
  }
  const uint64_t s = seed + 0x51ED27ull * (mode + 1);   // mode_basis's stream
  for (int k = 0; k < q->RL && good; ++k) {
    sketch_kernel<<<1184, 256>>>(n, p, k, q->c + (size_t)k * n, q->occ, s, q->X);
    good = apply(k, q->X, q->Z, p);
    if (good) add_kernel<<<1184, 256>>>((int64_t)n * p, q->Z, q->Y);
  }
  Y.resize((size_t)n * p);
  good = good && cudaMemcpy(Y.data(), q->Y, (size_t)n * p * sizeof(double), cudaMemcpyDeviceToHost) == cudaSuccess;
  if (!good) { cudaGetLastError(); q->ok = false; }
  cudaSetDevice(prev);
  return good;
}

bool RangeFinderDevice::power(const std::vector<double>& Q, int p, std::vector<double>& Y) {
  if (!q->ok) return false;
  std::lock_guard<std::mutex> lock(q->conv->p->mtx);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(q->conv->p->device);
  const int n = q->n;
  bool good = reserve(p) &&
              cudaMemcpy(q->X, Q.data(), (size_t)n * p * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaMemset(q->Y, 0, (size_t)n * p * sizeof(double)) == cudaSuccess;
  for (int k = 0; k < q->RL && good; ++k) {
    good = apply(k, q->X, q->Z, p);
    if (good) {
      scale_rows_kernel<<<1184, 256>>>(n, p, q->c + (size_t)k * n, q->Z);
      good = apply(k, q->Z, q->W, p);
    }
    if (good) add_kernel<<<1184, 256>>>((int64_t)n * p, q->W, q->Y);
  }
  Y.resize((size_t)n * p);
  good = good && cudaMemcpy(Y.data(), q->Y, (size_t)n * p * sizeof(double), cudaMemcpyDeviceToHost) == cudaSuccess;
  if (!good) { cudaGetLastError(); q->ok = false; }
  cudaSetDevice(prev);
  return good;
}

bool RangeFinderDevice::gram(const std::vector<double>& Q, int p, std::vector<double>& Gm) {
  if (!q->ok) return false;
  std::lock_guard<std::mutex> lock(q->conv->p->mtx);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(q->conv->p->device);
  const int n = q->n;
  constexpr int kBlk = 64;
  bool good = reserve(p) &&
              cudaMemcpy(q->X, Q.data(), (size_t)n * p * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess;
  Gm.assign((size_t)p * p, 0.0);
  std::vector<double> part((size_t)kBlk * p * p);
  for (int k = 0; k < q->RL && good; ++k) {
    good = apply(k, q->X, q->Z, p);
    if (good) {
      wgram_kernel<<<dim3((p * p + 255) / 256, kBlk), 256>>>(n, p, kBlk, q->c + (size_t)k * n, q->Z, q->part);
      good = cudaGetLastError() == cudaSuccess &&
             cudaMemcpy(part.data(), q->part, part.size() * sizeof(double), cudaMemcpyDeviceToHost) == cudaSuccess;
    }
    // per-k Gram: blocks in order, then added to the total in k order (deterministic)
    for (int blk = 0; blk < kBlk && good; ++blk)
      for (size_t e = 0; e < (size_t)p * p; ++e) Gm[e] += part[(size_t)blk * p * p + e];
  }
  for (int s_ = 0; s_ < p; ++s_)
    for (int t = s_ + 1; t < p; ++t) Gm[(size_t)t * p + s_] = Gm[(size_t)s_ * p + t];
  if (!good) { cudaGetLastError(); q->ok = false; }
  cudaSetDevice(prev);
  return good;
}

}  // namespace rs

