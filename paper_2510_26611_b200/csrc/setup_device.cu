// NEXT row N4 (part): step S6 of the setup (Algorithm TEP), the Tucker core
// G[a,b,c] = sum_k sum_m (z_m a_k H0_k[i_m0, a]) H1_k[i_m1, b] H2_k[i_m2, c] of the long-range
// part, on the device.  Each thread owns one core entry and runs the host loop's exact op
// sequence (per k: row = 0; for m in order: w = (z_m a_k) H0, skipped when 0, wb = w H1,
// row += wb H2; then G += row), compiled with -fmad=false like the host's -ffp-contract=off,
// so the core -- and every table built from it -- is bitwise the host-only build's.
#include <cuda_runtime.h>

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

