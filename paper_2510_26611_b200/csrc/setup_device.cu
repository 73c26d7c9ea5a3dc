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
