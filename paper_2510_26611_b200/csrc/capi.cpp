// C ABI of librsdock (include/rs_dock.h): handle build (Algorithm TEP, host C++), upload,
// and the scoring entry points that enqueue the fused sm_100a kernel (score_kernel.cu).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "rs_internal.h"

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

thread_local std::string g_err;

void set_err(const std::string& s) { g_err = s; }

#define CUDA_TRY(expr, code)                                                               \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      set_err(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #expr);        \
      return code;                                                                         \
    }                                                                                      \
  } while (0)

// cuStreamWaitValue32 through the runtime's driver entry point (no libcuda link); null if the
// driver does not offer it (the host-buffer pipeline then falls back to per-chunk launches)
typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_waitValue32 wait_value32() {
  static PFN_waitValue32 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_waitValue32)p;
    cudaGetLastError();
  }
  return fn;
}

bool finite_all(const double* p, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(p[i])) return false;
  return true;
}

// O3 snapping, the library's copy (the oracle has its own): u = (x + b) * inv_h,
// i = ceil(u) - 1 clamped to [0, n-1]; -1 outside [-b, b].
int snap_cell(double x, double b, double inv_h, int n) {
  if (!(x >= -b && x <= b)) return -1;
  double u = (x + b) * inv_h;
  double c = std::ceil(u) - 1.0;
  c = std::min(std::max(c, 0.0), double(n - 1));
  return (int)c;
}

void free_device(rs_handle* h) {
  if (!h->on_device) return;
  cudaSetDevice(h->device);
  for (void*& p : h->dmem) {
    if (p) cudaFree(p);
    p = nullptr;
  }
  if (h->d_work) cudaFree(h->d_work);
  h->d_work = nullptr;
  for (void*& ev : h->work_ev) {
    if (ev) cudaEventDestroy((cudaEvent_t)ev);
    ev = nullptr;
  }
  if (h->scan_buf) cudaFree(h->scan_buf);
  h->scan_buf = nullptr;
  h->scan_bytes = 0;
  for (void** p : {&h->d_Ut[0], &h->d_Ut[1], &h->d_Ut[2], &h->d_TG, &h->d_prec, &h->d_nb_ent, &h->d_memo, &h->d_Fw[0], &h->d_Fw[1], &h->d_Fw[2],
                   &h->d_Fw32[0], &h->d_Fw32[1], &h->d_Fw32[2],
                   &h->d_nb_range, &h->d_nb_pack}) {
    if (*p) cudaFree(*p);
    *p = nullptr;
  }
  if (h->stage) cudaFree(h->stage);
  h->stage = nullptr;
  if (h->h_ones) cudaFreeHost(h->h_ones);
  h->h_ones = nullptr;
  for (void*& s : h->streams) {
    if (s) cudaStreamDestroy((cudaStream_t)s);
    s = nullptr;
  }
  h->on_device = false;
}

template <class T>
int upload(void** dst, const std::vector<T>& v, int64_t* bytes) {
  size_t nb = std::max<size_t>(sizeof(T), v.size() * sizeof(T));
  CUDA_TRY(cudaMalloc(dst, nb), RS_E_NOMEM);
  if (!v.empty()) CUDA_TRY(cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), RS_E_CUDA);
  *bytes += (int64_t)nb;
  return 0;
}

int upload_handle(rs_handle* h) {
  CUDA_TRY(cudaSetDevice(h->device), RS_E_CUDA);
  h->on_device = true;
  int64_t bytes = 0;
  for (int a = 0; a < 3; ++a) {
    if (int e = upload(&h->dmem[a], h->F[a], &bytes)) return e;
    if (int e = upload(&h->dmem[3 + a], h->S[a], &bytes)) return e;
  }
  {
    // S9 on the device.  Protein atoms are renumbered in coarse-cell order (spatially sorted,
    // so the few atoms near one pose tile share cache lines); each list entry carries the
    // atom's fine cell (for the integer prefilter) and its sorted index:
    //   nb_range[c] = (first entry, count)       int2 per coarse cell
    //   nb_ent[j]   = (i0 | i1 << 15 | (k & 3) << 30, i2 | (k >> 2) << 15, q)  16 bytes per
    //                 list entry: the fine cell (15 bits per axis, n <= 32768), the sorted
    //                 index k (19 bits) and the charge (8 bytes), so the H5 term needs no record
    //   prec[k]     = (x, y, z, q)               double4 per protein atom (the H6 distance)
    const int64_t M = h->M;
    if (M > rs::kMaxPackedAtoms) {
      set_err("protein too large for the packed neighbour lists (max 524288 atoms)");
      return RS_E_INVALID_ARG;
    }
    std::vector<int64_t> key(M);
    std::vector<int32_t> order(M), rank(M);
    for (int64_t m = 0; m < M; ++m) {
      int64_t k = 0;
      for (int a = 0; a < 3; ++a) k = k * 65536 + (h->cells[3 * m + a] >> h->cg.shift);
      key[m] = k;
      order[m] = (int32_t)m;
    }
    std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return key[x] < key[y]; });
    for (int64_t k = 0; k < M; ++k) rank[order[k]] = (int32_t)k;
    std::vector<double> prec(4 * (size_t)M);
    for (int64_t k = 0; k < M; ++k) {
      const size_t m = (size_t)order[k];
      for (int a = 0; a < 3; ++a) prec[4 * k + a] = h->xyz[3 * m + a];
      prec[4 * k + 3] = h->z[m];
    }
    if (int e = upload(&h->d_prec, prec, &bytes)) return e;
    // every list starts at an even entry (a padding entry after odd-length lists), so the
    // kernel reads its candidates in aligned 32-byte pairs
    const size_t nc = h->cg.off.size() - 1;
    std::vector<int32_t> rng(2 * nc);
    size_t tot = 0;
    for (size_t c = 0; c < nc; ++c) {
      const int32_t cnt = h->cg.off[c + 1] - h->cg.off[c];
      rng[2 * c] = (int32_t)tot;
      rng[2 * c + 1] = cnt;
      tot += (size_t)(cnt + (cnt & 1));
    }
    if (tot > (size_t)INT32_MAX) { set_err("neighbour lists exceed 2^31 entries"); return RS_E_NOMEM; }
    {
      int32_t maxcnt = 0;
      for (size_t c = 0; c < nc; ++c) maxcnt = std::max(maxcnt, rng[2 * c + 1]);
      h->loc4 = tot < ((size_t)1 << 24) && maxcnt < 256;
    }
    std::vector<int32_t> ent(4 * std::max<size_t>(tot, 2), 0);
    // each list in ascending distance of the atom's fine cell from the coarse cell's centre
    // (key = |2 i_m - C|^2 in half cells, C = 2^(s+1) c + 2^s - 1; ties by atom index), so the
    // kernel can end a walk at the first entry too far from the centre to matter
    const int sh = h->cg.shift;
    const int cd1 = h->cg.dim[1], cd2 = h->cg.dim[2];
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t c = 0; c < (int64_t)nc; ++c) {
      const int32_t cnt = rng[2 * c + 1];
      if (cnt == 0) continue;
      const int64_t cc[3] = {c / ((int64_t)cd1 * cd2) + h->cg.lo[0], (c / cd2) % cd1 + h->cg.lo[1],
                             c % cd2 + h->cg.lo[2]};
      std::vector<std::pair<int64_t, int32_t>> lk((size_t)cnt);
      for (int32_t u = 0; u < cnt; ++u) {
        const int32_t m = h->cg.idx[(size_t)h->cg.off[c] + u];
        int64_t key = 0;
        for (int ax = 0; ax < 3; ++ax) {
          const int64_t d = 2 * (int64_t)h->cells[3 * (size_t)m + ax] - (cc[ax] * (2 << sh) + (1 << sh) - 1);
          key += d * d;
        }
        lk[(size_t)u] = {key, m};
      }
      std::sort(lk.begin(), lk.end());
      for (int32_t u = 0; u < cnt; ++u) {
        const size_t j = (size_t)rng[2 * c] + u;
        const size_t m = (size_t)lk[(size_t)u].second;
        const uint32_t k = (uint32_t)rank[m];
        ent[4 * j] = (int32_t)((uint32_t)h->cells[3 * m] | ((uint32_t)h->cells[3 * m + 1] << 15) | ((k & 3u) << 30));
        ent[4 * j + 1] = (int32_t)((uint32_t)h->cells[3 * m + 2] | ((k >> 2) << 15));
        std::memcpy(&ent[4 * j + 2], &h->z[m], sizeof(double));
      }
    }
    if (int e = upload(&h->d_nb_ent, ent, &bytes)) return e;
    h->n_ent = (int64_t)(ent.size() / 4);
    if (int e = upload(&h->d_nb_range, rng, &bytes)) return e;
    if (h->loc4) {
      // the same ranges packed into 4 bytes, z rows padded to 16 bytes, with rs::kPackPad zero
      // cells before every axis (a TMA tensor copy takes no negative coordinates): the scoring
      // kernel copies a tile's box of it into shared memory with one TMA tensor copy
      const int P = rs::kPackPad;
      const int d0 = h->cg.dim[0], d1 = h->cg.dim[1], d2 = h->cg.dim[2];
      const int e0 = d0 + P, e1 = d1 + P;
      h->nb_dim2p = (d2 + P + 3) / 4 * 4;
      std::vector<uint32_t> pk((size_t)e0 * e1 * h->nb_dim2p, 0u);
#pragma omp parallel for schedule(static)
      for (int x = 0; x < d0; ++x)
        for (int y = 0; y < d1; ++y)
          for (int z = 0; z < d2; ++z) {
            const size_t c = ((size_t)x * d1 + y) * d2 + z;
            pk[((size_t)(x + P) * e1 + (y + P)) * h->nb_dim2p + (z + P)] =
                (uint32_t)rng[2 * c] | ((uint32_t)rng[2 * c + 1] << 24);
          }
      if (int e = upload(&h->d_nb_pack, pk, &bytes)) return e;
    }
  }
  if (h->prm.flags & RS_FLAG_TUCKER_EVAL) {
    // the Tucker form for the scoring kernel (N5): bases row-major (row i = U_l[i, :]), core
    const rs::TuckerRep& tk = h->tucker;
    for (int l = 0; l < 3; ++l) {
      std::vector<double> rows((size_t)h->n * tk.r[l]);
      for (int i = 0; i < h->n; ++i)
        for (int a = 0; a < tk.r[l]; ++a) rows[(size_t)i * tk.r[l] + a] = tk.U[l][(size_t)a * h->n + i];
      if (int e = upload(&h->d_Ut[l], rows, &bytes)) return e;
    }
    if (int e = upload(&h->d_TG, tk.G, &bytes)) return e;
  }
  if (h->f32) {
    // binary32 copy of the factors (A21), rows as 16-byte quads padded/replicated like Fw
    std::vector<float> packed;
    for (int a = 0; a < 3; ++a) {
      rs::pack_window_rows32(h->F[a], h->n, h->R, packed);
      if (int e = upload(&h->d_Fw32[a], packed, &bytes)) return e;
    }
  } else if (rs::window_row_chunks(h->R) > 0) {
    // row-padded copy of the factors: the shared-memory window is staged by 1-D bulk copies
    std::vector<double> packed;
    for (int a = 0; a < 3; ++a) {
      rs::pack_window_rows(h->F[a], h->n, h->R, packed);
      if (int e = upload(&h->d_Fw[a], packed, &bytes)) return e;
    }
  }
  // dense memo of the short-range chain over |D_a| <= n_sigma, filled on the device by the same
  // O5 op sequence (ascending k; all zeros when R_s = 0); the scoring kernel reads O5 values
  // only from it (C3: 2.2 MB, C5 at sigma_s = 6 A: 136 MB)
  const double memo_b = 8.0 * std::pow(double(h->n_sigma + 1), 3.0);
  if (memo_b > 2.0 * 1024 * 1024 * 1024) {
    set_err("n_sigma = " + std::to_string(h->n_sigma) + ": the short-range memo ((n_sigma+1)^3 "
            "doubles) would exceed 2 GiB; use a larger grid step or a smaller sigma_split");
    return RS_E_NOMEM;
  }
  CUDA_TRY(cudaMalloc(&h->d_work, rs::kWorkSlots * sizeof(int)), RS_E_NOMEM);
  for (int k = 0; k < rs::kWorkSlots; ++k)
    CUDA_TRY(cudaEventCreateWithFlags((cudaEvent_t*)&h->work_ev[k], cudaEventDisableTiming), RS_E_CUDA);
  CUDA_TRY(cudaMalloc(&h->d_memo, (size_t)memo_b), RS_E_NOMEM);
  bytes += (int64_t)memo_b;
  {
    int e = rs::launch_fill_short_memo((const double*)h->dmem[3], (const double*)h->dmem[4],
                                       (const double*)h->dmem[5], h->Rs, h->n_sigma,
                                       (double*)h->d_memo, nullptr);
    if (e != 0) { set_err("short-range memo fill failed"); return RS_E_CUDA; }
    CUDA_TRY(cudaDeviceSynchronize(), RS_E_CUDA);
  }
  h->device_bytes = bytes;
  return 0;
}

rs::ScoreArgs base_args(const rs_handle* h) {
  rs::ScoreArgs a{};
  a.n = h->n;
  a.R = h->R;
  a.Rs = h->Rs;
  a.n_sigma = h->n_sigma;
  a.b = h->b;
  a.inv_h = h->inv_h;
  a.h = h->h;
  a.dcap2 = h->prm.dmin_cap * h->prm.dmin_cap;
  a.nb_shift = h->cg.shift;
  for (int i = 0; i < 3; ++i) {
    a.nb_lo[i] = h->cg.lo[i];
    a.nb_dim[i] = h->cg.dim[i];
    a.t.F[i] = (const double*)h->dmem[i];
    a.t.Fw[i] = (const double2*)h->d_Fw[i];
    a.t.Fw32[i] = (const float4*)h->d_Fw32[i];
    a.t.S[i] = (const double*)h->dmem[3 + i];
  }
  a.t.nb_ent = (const int4*)h->d_nb_ent;
  a.t.prec = (const double4*)h->d_prec;
  a.n_ent = h->n_ent;
  a.n_prot = h->M;
  a.t.short_memo = (const double*)h->d_memo;
  a.t.nb_range = (const int2*)h->d_nb_range;
  a.t.nb_pack = (const unsigned*)h->d_nb_pack;
  a.nb_dim2p = h->nb_dim2p;
  a.ns2 = (unsigned)((int64_t)h->n_sigma * h->n_sigma);
  a.f32 = h->f32 ? 1 : 0;
  if (h->d_TG) {
    a.tk = 1;
    for (int l = 0; l < 3; ++l) {
      a.tr[l] = h->tucker.r[l];
      a.t.Ut[l] = (const double*)h->d_Ut[l];
    }
    a.t.TG = (const double*)h->d_TG;
  }
  a.loc4 = h->loc4 ? 1 : 0;
  {
    // |x_l - x_m| >= (|D| - sqrt 3) h for cells D apart; +2 cells of margin for snap rounding
    const double t = h->prm.dmin_cap / h->h + std::sqrt(3.0) + 2.0;
    a.vdw_cells2 = (unsigned)std::min(std::ceil(t * t), 4294967295.0);
    // the kernel's running bounds without a square root: (sqrt(x) c1 + c2)^2 <=
    // (1 + e) c1^2 x + (1 + 1/e) c2^2 for any e > 0 (AM-GM on the cross term), e = 1/4, each
    // coefficient rounded up to binary32 plus a relative 1e-6 (the kernel adds 2 after its
    // rounded-up evaluation)
    const double c2 = std::sqrt(3.0) + 2.0;
    const double up = 1.0 + 1e-6;
    a.thr_a = std::nextafter((float)(1.25 * h->inv_h * h->inv_h * up), INFINITY);
    a.thr_b = std::nextafter((float)(5.0 * c2 * c2 * up), INFINITY);
  }
  a.rmax_hint = -1.0;
  return a;
}

// 1 = device (or managed) pointer of the handle's device, 0 = host memory
int pointer_kind(const void* p) {
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) ? 1 : 0;
}

// Ligand radius max |y_l| (body frame).  Only steers the launch shape (shared-memory window
// or not, local-table box); correctness never depends on it (the kernel recomputes it).  Device
// ligands are read back once per (pointer, L) with a copy ordered on the caller's stream and
// cached on the handle (a reused buffer keeps the old shape hint: at worst a slower launch);
// under stream capture no readback happens and the launch sizes itself without the hint.
double ligand_rmax(rs_handle* h, const double* yl, int64_t L, bool dev, cudaStream_t st) {
  if (L <= 0) return 0.0;
  std::vector<double> tmp;
  const double* y = yl;
  if (dev) {
    if (h->rmax_key == (const void*)yl && h->rmax_L == L) return h->rmax_val;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      return -1.0;
    }
    tmp.resize(3 * (size_t)L);
    if (cudaMemcpyAsync(tmp.data(), yl, 3 * (size_t)L * sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      cudaGetLastError();
      return -1.0;
    }
    y = tmp.data();
  }
  double r2 = 0.0;
  for (int64_t l = 0; l < L; ++l)
    r2 = std::max(r2, y[3 * l] * y[3 * l] + y[3 * l + 1] * y[3 * l + 1] + y[3 * l + 2] * y[3 * l + 2]);
  const double r = std::sqrt(r2);
  if (dev) {
    h->rmax_key = (const void*)yl;
    h->rmax_L = L;
    h->rmax_val = r;
  }
  return r;
}

// One scoring launch with a dynamic-schedule work counter that no other launch in flight holds:
// a ring of kWorkSlots counters on the handle, each reused only after the event recorded behind
// its previous launch (the stream waits on it; a per-slot lock keeps the wait-reset-launch-record
// sequence of one caller together), so launches on different streams never share a counter
int launch_with_counter(rs_handle* h, rs::ScoreArgs& a, cudaStream_t st) {
  const unsigned k = h->work_slot.fetch_add(1) % rs::kWorkSlots;
  std::lock_guard<std::mutex> lock(h->work_mtx[k]);
  // (under stream capture the graph's own order stands in for the event: no cross-capture wait)
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) return (int)cudaGetLastError();
  const bool capturing = cs != cudaStreamCaptureStatusNone;
  cudaError_t e = capturing ? cudaSuccess : cudaStreamWaitEvent(st, (cudaEvent_t)h->work_ev[k], 0);
  if (e != cudaSuccess) return (int)e;
  a.work = h->d_work + k;
  e = cudaMemsetAsync(a.work, 0, sizeof(int), st);
  if (e != cudaSuccess) return (int)e;
  const int r = rs::launch_score(a, st, h->device, nullptr);
  if (r != 0 || capturing) return r;
  return (int)cudaEventRecord((cudaEvent_t)h->work_ev[k], st);
}

}  // namespace

extern "C" {

void rs_params_default(rs_params* p) {
  if (!p) return;
  std::memset(p, 0, sizeof(*p));
  p->grid_n = 256;
  p->rank_R = 16;
  p->eps_compress = 1e-8;
  p->eps_quad = 1e-6;
  p->sigma_split = 2.0;
  p->eps_split = 1e-6;
  p->sigma_vdw = 2.5;
  p->dmin_cap = 2.5;
  p->tucker_rank_max = 0;
  p->als_sweeps = 0;
  p->device = 0;
  p->n_threads = 0;
  p->seed = 0x5EED5EEDull;
  p->flags = 0;
}

const char* rs_last_error(void) { return g_err.c_str(); }

rs_handle* rs_build_protein(const double* q, const double* xyz, int64_t n_atoms,
                            double box_half_width, const rs_params* params) {
  rs::NvtxRange nvtx_("rs_build_protein");
  g_err.clear();
  auto t0 = std::chrono::steady_clock::now();
  rs_params prm;
  if (params) prm = *params; else rs_params_default(&prm);
  if (!q || !xyz) { set_err("null input pointer"); return nullptr; }
  if (n_atoms <= 0) { set_err("n_atoms must be > 0"); return nullptr; }
  if (n_atoms > rs::kMaxPackedAtoms) { set_err("n_atoms exceeds 524288 (19-bit atom index of a list entry)"); return nullptr; }
  if (!(box_half_width > 0) || !std::isfinite(box_half_width)) { set_err("box_half_width must be finite and > 0"); return nullptr; }
  if (prm.grid_n < 2 || (prm.grid_n & 1)) { set_err("grid_n must be even and >= 2"); return nullptr; }
  if (prm.grid_n > 32768) { set_err("grid_n too large (max 32768)"); return nullptr; }
  if (prm.rank_R < 0) { set_err("rank_R must be >= 0"); return nullptr; }
  if (!(prm.nbr_cell >= 0) || !std::isfinite(prm.nbr_cell)) { set_err("nbr_cell must be finite and >= 0"); return nullptr; }
  if (!(prm.eps_compress > 0 && prm.eps_compress < 1)) { set_err("eps_compress must be in (0,1)"); return nullptr; }
  if (!(prm.eps_quad > 0 && prm.eps_quad < 1)) { set_err("eps_quad must be in (0,1)"); return nullptr; }
  if (!(prm.eps_split > 0 && prm.eps_split < 1)) { set_err("eps_split must be in (0,1)"); return nullptr; }
  if (!(prm.sigma_vdw >= 0) || !(prm.dmin_cap >= prm.sigma_vdw) || !std::isfinite(prm.dmin_cap)) {
    set_err("need 0 <= sigma_vdw <= dmin_cap < inf");
    return nullptr;
  }
  if (!finite_all(q, n_atoms) || !finite_all(xyz, 3 * n_atoms)) { set_err("non-finite protein input"); return nullptr; }
  const int n = prm.grid_n;
  const double b = box_half_width;
  const double h = 2.0 * b / double(n);
  if (!(prm.sigma_split >= h) || !std::isfinite(prm.sigma_split)) { set_err("sigma_split must be >= h = 2b/n"); return nullptr; }
  const bool host_only = (prm.flags & RS_FLAG_HOST_ONLY) != 0;
  if (!host_only) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= prm.device || prm.device < 0) {
      cudaGetLastError();
      set_err("no CUDA device (there is no CPU fallback; use RS_FLAG_HOST_ONLY for host-only tables)");
      return nullptr;
    }
  }
#ifdef _OPENMP
  if (prm.n_threads > 0) omp_set_num_threads(prm.n_threads);
#endif
  std::unique_ptr<rs_handle> H;
  try {
    H.reset(new rs_handle());
  } catch (...) {
    set_err("out of host memory");
    return nullptr;
  }
  rs_handle* hd = H.get();
  hd->prm = prm;
  hd->n = n;
  hd->b = b;
  hd->h = h;
  hd->inv_h = double(n) / (2.0 * b);
  hd->device = prm.device;
  hd->M = n_atoms;
  try {
    hd->xyz.assign(xyz, xyz + 3 * n_atoms);
    hd->z.assign(q, q + n_atoms);
    // S4: snap protein atoms
    hd->cells.resize(3 * n_atoms);
    for (int64_t m = 0; m < n_atoms; ++m)
      for (int a = 0; a < 3; ++a) {
        int c = snap_cell(xyz[3 * m + a], b, hd->inv_h, n);
        if (c < 0) {
          set_err("protein atom " + std::to_string(m) + " outside [-b, b]^3");
          return nullptr;
        }
        hd->cells[3 * m + a] = c;
      }
    // S1: quadrature on [h/4, 2 sqrt(3) b]
    const double Ls = 2.0 * std::sqrt(3.0) * b;
    hd->quad = rs::choose_quadrature(prm.eps_quad, h / 4.0, Ls, Ls);
    if (hd->quad.K < 0) { set_err("quadrature search failed for eps_quad"); return nullptr; }
    // S2: split
    std::vector<double> tl, al, ts, as;
    hd->is_long.resize(hd->quad.t.size());
    for (size_t k = 0; k < hd->quad.t.size(); ++k) {
      bool lg = rs::is_long_term(hd->quad.t[k], prm.sigma_split, prm.eps_split);
      hd->is_long[k] = lg ? 1 : 0;
      if (lg) { tl.push_back(hd->quad.t[k]); al.push_back(hd->quad.a[k]); }
      else { ts.push_back(hd->quad.t[k]); as.push_back(hd->quad.a[k]); }
    }
    hd->R_long_ref = (int)tl.size();
    hd->Rs = (int)ts.size();
    hd->n_sigma = (int)std::ceil(prm.sigma_split / h);
    auto lap = [&](const char* what) {
      nvtxMarkA(what);                    // end of a setup phase on the NVTX timeline
      static const bool on = std::getenv("RS_SETUP_TIMING") != nullptr;
      if (on)
        std::fprintf(stderr, "[rs setup] %-22s %8.3f s (at %.3f)\n", what,
                     std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(),
                     std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count());
    };
    lap("S1-S4");
    // S5-S7
    rs::compress_long_range(n, h, hd->cells, hd->z, tl, al, prm.rank_R, prm.eps_compress,
                            prm.tucker_rank_max, prm.als_sweeps, prm.seed, hd->F, &hd->R, &hd->rep,
                            &hd->tucker, nullptr, nullptr, host_only ? -1 : prm.device,
                            (prm.flags & RS_FLAG_HOST_FFT) == 0);
    hd->f32 = (prm.flags & RS_FLAG_F32_FACTORS) != 0;
    if (hd->f32 && rs::window_row_chunks32(hd->R) == 0) {
      set_err("RS_FLAG_F32_FACTORS needs a compiled CP width R in {4, 8, 12, 16, 24, 32}, got " +
              std::to_string(hd->R));
      return nullptr;
    }
    if (prm.flags & RS_FLAG_TUCKER_EVAL) {
      const int* r = hd->tucker.r;
      if (hd->f32 || r[0] < 1 || r[0] > 32 || r[1] < 1 || r[1] > 32 || r[2] < 1 || r[2] > 32 ||
          (int64_t)r[0] * r[1] * r[2] > 16384) {
        set_err("RS_FLAG_TUCKER_EVAL needs Tucker ranks r_l <= 32 with r0 r1 r2 <= 16384 (and no "
                "RS_FLAG_F32_FACTORS); got " + std::to_string(r[0]) + " x " + std::to_string(r[1]) +
                " x " + std::to_string(r[2]));
        return nullptr;
      }
    }
    if (hd->R > (1 << 20)) {
      set_err("compressed CP width " + std::to_string(hd->R) + " exceeds 2^20 (raise eps_compress or fix rank_R)");
      return nullptr;
    }
    lap("S5-S7 (RHOSVD, core, CP)");
    // S8: short-range reference rows, a_k folded into S1 (Def. 2.1, A_0)
    const int ns = hd->n_sigma, Rs = hd->Rs;
    for (int a = 0; a < 3; ++a) hd->S[a].assign((size_t)(2 * ns + 1) * Rs, 0.0);
    for (int d = -ns; d <= ns; ++d)
      for (int k = 0; k < Rs; ++k) {
        const double g = rs::cell_average(ts[k], h, d);
        hd->S[0][(size_t)(d + ns) * Rs + k] = g * as[k];
        hd->S[1][(size_t)(d + ns) * Rs + k] = g;
        hd->S[2][(size_t)(d + ns) * Rs + k] = g;
      }
    // S9: cell lists covering every pair that can matter: vdW pairs (< dmin_cap) and the
    // short-range ball (|i_l - i_m|_2 <= n_sigma => |x_l - x_m| <= (n_sigma + sqrt 3) h)
    const double rho = std::max(prm.dmin_cap, (ns + std::sqrt(3.0)) * h);
    rs::build_cell_lists(n, b, h, hd->xyz, hd->cells, rho, prm.nbr_cell, &hd->cg);
    lap("S8-S9 (short, cells)");
    // sampled compression error at exterior cells
    const double work = double(n_atoms) * double(tl.size());
    const int nsamp = (int)std::max(100.0, std::min(2000.0, 4e9 / std::max(work, 1.0)));
    rs::sample_compression_error(n, b, h, hd->xyz, hd->cells, hd->z, tl, al, hd->F, hd->R,
                                 std::max(prm.sigma_vdw, h), hd->cg, nsamp, prm.seed, &hd->rep,
                                 host_only ? -1 : prm.device);
    lap("error samples");
  } catch (const std::bad_alloc&) {
    set_err("out of host memory during setup");
    return nullptr;
  }
  if (!host_only) {
    if (upload_handle(hd) != 0) {
      std::string msg = g_err;
      free_device(hd);
      set_err(msg.empty() ? "upload failed" : msg);
      return nullptr;
    }
  }
  hd->setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return H.release();
}

// NEXT row N4 (multi-protein, Eq. (23); reading A24): the
// potential of a complex is the sum of its proteins' potentials, so on a shared grid the
// long-range CP factors concatenate along the rank (R = sum R_p, no recompression), and the
// short-range part and the vdW distance run over the union of the atoms.
rs_handle* rs_combine_proteins(const rs_handle* const* parts, int32_t n_parts, int32_t flags) {
  rs::NvtxRange nvtx_("rs_combine_proteins");
  g_err.clear();
  auto t0 = std::chrono::steady_clock::now();
  if (!parts || n_parts < 1) { set_err("need n_parts >= 1 handles"); return nullptr; }
  for (int32_t p = 0; p < n_parts; ++p)
    if (!parts[p]) { set_err("null part handle " + std::to_string(p)); return nullptr; }
  const rs_handle* p0 = parts[0];
  for (int32_t p = 1; p < n_parts; ++p) {
    const rs_handle* q = parts[p];
    // Same grid, quadrature and split => identical short-range rows and n_sigma; same vdW rule.
    if (q->n != p0->n || q->b != p0->b || q->prm.eps_quad != p0->prm.eps_quad ||
        q->prm.sigma_split != p0->prm.sigma_split || q->prm.eps_split != p0->prm.eps_split ||
        q->prm.sigma_vdw != p0->prm.sigma_vdw || q->prm.dmin_cap != p0->prm.dmin_cap) {
      set_err("part " + std::to_string(p) + " differs from part 0 in grid_n, b, eps_quad, "
              "sigma_split, eps_split, sigma_vdw or dmin_cap");
      return nullptr;
    }
    for (int a = 0; a < 3; ++a)
      if (q->S[a] != p0->S[a]) { set_err("short-range rows differ between parts"); return nullptr; }
  }
  int64_t R = 0, M = 0;
  for (int32_t p = 0; p < n_parts; ++p) { R += parts[p]->R; M += parts[p]->M; }
  if (R > (1 << 20)) { set_err("combined CP width exceeds 2^20"); return nullptr; }
  if (M > rs::kMaxPackedAtoms) { set_err("combined protein exceeds 524288 atoms"); return nullptr; }
  rs_params prm = p0->prm;
  prm.flags = flags;
  if (flags & RS_FLAG_TUCKER_EVAL) { set_err("RS_FLAG_TUCKER_EVAL: a combined handle has no Tucker form"); return nullptr; }
  const bool host_only = (flags & RS_FLAG_HOST_ONLY) != 0;
  if (!host_only) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= prm.device || prm.device < 0) {
      cudaGetLastError();
      set_err("no CUDA device (there is no CPU fallback; use RS_FLAG_HOST_ONLY for host-only tables)");
      return nullptr;
    }
  }
  if ((flags & RS_FLAG_F32_FACTORS) && rs::window_row_chunks32((int)R) == 0) {
    set_err("RS_FLAG_F32_FACTORS needs a compiled CP width R in {4, 8, 12, 16, 24, 32}, got " +
            std::to_string(R));
    return nullptr;
  }
  std::unique_ptr<rs_handle> H;
  try {
    H.reset(new rs_handle());
    rs_handle* hd = H.get();
    hd->prm = prm;
    hd->n = p0->n;
    hd->b = p0->b;
    hd->h = p0->h;
    hd->inv_h = p0->inv_h;
    hd->quad = p0->quad;
    hd->is_long = p0->is_long;
    hd->R = (int)R;
    hd->Rs = p0->Rs;
    hd->n_sigma = p0->n_sigma;
    hd->R_long_ref = p0->R_long_ref;
    hd->device = prm.device;
    hd->f32 = (flags & RS_FLAG_F32_FACTORS) != 0;
    for (int a = 0; a < 3; ++a) hd->S[a] = p0->S[a];
    // factor rows i: [F_a^(0)[i, :] | F_a^(1)[i, :] | ...]  (rank concatenation)
    const size_t n = (size_t)hd->n;
    for (int a = 0; a < 3; ++a) {
      hd->F[a].assign(n * (size_t)R, 0.0);
      size_t col = 0;
      for (int32_t p = 0; p < n_parts; ++p) {
        const int Rp = parts[p]->R;
        for (size_t i = 0; i < n; ++i)
          std::copy(parts[p]->F[a].begin() + i * Rp, parts[p]->F[a].begin() + (i + 1) * Rp,
                    hd->F[a].begin() + i * R + col);
        col += (size_t)Rp;
      }
    }
    hd->M = M;
    for (int32_t p = 0; p < n_parts; ++p) {
      hd->xyz.insert(hd->xyz.end(), parts[p]->xyz.begin(), parts[p]->xyz.end());
      hd->z.insert(hd->z.end(), parts[p]->z.begin(), parts[p]->z.end());
      hd->cells.insert(hd->cells.end(), parts[p]->cells.begin(), parts[p]->cells.end());
    }
    // report: ranks add; the sampled errors are the parts' worst (each part's own samples)
    hd->rep.R_exact = 0;
    for (int32_t p = 0; p < n_parts; ++p) {
      const rs::SetupReport& r = parts[p]->rep;
      hd->rep.R_exact += r.R_exact;
      for (int a = 0; a < 3; ++a) hd->rep.tucker_r[a] += r.tucker_r[a];
      hd->rep.tucker_err = std::max(hd->rep.tucker_err, r.tucker_err);
      hd->rep.cp_core_err = std::max(hd->rep.cp_core_err, r.cp_core_err);
      hd->rep.sampled_max = std::max(hd->rep.sampled_max, r.sampled_max);
      hd->rep.sampled_rms = std::max(hd->rep.sampled_rms, r.sampled_rms);
      hd->rep.n_samples += r.n_samples;
    }
    const double rho = std::max(prm.dmin_cap, (hd->n_sigma + std::sqrt(3.0)) * hd->h);
    rs::build_cell_lists(hd->n, hd->b, hd->h, hd->xyz, hd->cells, rho, prm.nbr_cell, &hd->cg);
  } catch (const std::bad_alloc&) {
    set_err("out of host memory while combining");
    return nullptr;
  }
  rs_handle* hd = H.get();
  if (!host_only) {
    if (upload_handle(hd) != 0) {
      std::string msg = g_err;
      free_device(hd);
      set_err(msg.empty() ? "upload failed" : msg);
      return nullptr;
    }
  }
  hd->setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return H.release();
}

rs_handle* rs_restrict_box(const rs_handle* h, const int32_t* lo, const int32_t* hi, int32_t rank,
                           int32_t flags) {
  rs::NvtxRange nvtx_("rs_restrict_box");
  g_err.clear();
  auto t0 = std::chrono::steady_clock::now();
  if (!h || !lo || !hi) { set_err("null argument"); return nullptr; }
  if (rank < 0) { set_err("rank must be >= 0"); return nullptr; }
  if (flags & RS_FLAG_TUCKER_EVAL) { set_err("RS_FLAG_TUCKER_EVAL: a box handle scores its box CP"); return nullptr; }
  for (int a = 0; a < 3; ++a)
    if (lo[a] < 0 || hi[a] >= h->n || lo[a] > hi[a]) {
      set_err("need 0 <= lo <= hi < n on every axis");
      return nullptr;
    }
  if (h->tucker.G.empty() && !(flags & RS_FLAG_BOX_SCHEME_B)) {
    set_err("handle has no Tucker form (combined or restricted handles cannot be restricted)");
    return nullptr;
  }
  if ((flags & RS_FLAG_BOX_SCHEME_B) && h->z.size() != (size_t)h->M) {
    set_err("handle has no protein atoms");
    return nullptr;
  }
  const bool host_only = (flags & RS_FLAG_HOST_ONLY) != 0;
  if (!host_only) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= h->prm.device || h->prm.device < 0) {
      cudaGetLastError();
      set_err("no CUDA device (there is no CPU fallback; use RS_FLAG_HOST_ONLY for host-only tables)");
      return nullptr;
    }
  }
  std::unique_ptr<rs_handle> H;
  try {
    H.reset(new rs_handle());
    rs_handle* hd = H.get();
    hd->prm = h->prm;
    hd->prm.flags = flags;
    hd->n = h->n;
    hd->b = h->b;
    hd->h = h->h;
    hd->inv_h = h->inv_h;
    hd->quad = h->quad;
    hd->is_long = h->is_long;
    hd->Rs = h->Rs;
    hd->n_sigma = h->n_sigma;
    hd->R_long_ref = h->R_long_ref;
    for (int a = 0; a < 3; ++a) hd->S[a] = h->S[a];
    hd->M = h->M;
    hd->xyz = h->xyz;
    hd->z = h->z;
    hd->cells = h->cells;
    hd->cg = h->cg;
    hd->device = h->device;
    hd->f32 = (flags & RS_FLAG_F32_FACTORS) != 0;
    int lo_[3], hi_[3];
    for (int a = 0; a < 3; ++a) { lo_[a] = lo[a]; hi_[a] = hi[a]; hd->box_lo[a] = lo[a]; hd->box_hi[a] = hi[a]; }
    if (flags & RS_FLAG_BOX_SCHEME_B) {
      // scheme (B): a new RHOSVD of the long-range sum restricted to the box rows
      std::vector<double> tl, al;
      for (size_t k = 0; k < h->quad.t.size(); ++k)
        if (h->is_long[k]) { tl.push_back(h->quad.t[k]); al.push_back(h->quad.a[k]); }
      rs::compress_long_range(h->n, h->h, h->cells, h->z, tl, al, rank, h->prm.eps_compress,
                              h->prm.tucker_rank_max, h->prm.als_sweeps, h->prm.seed, hd->F,
                              &hd->R, &hd->rep, nullptr, lo_, hi_, host_only ? -1 : hd->device,
                              (flags & RS_FLAG_HOST_FFT) == 0);
    } else {
      hd->rep.tucker_err = h->rep.tucker_err;
      hd->R = rs::restrict_to_box(h->n, h->tucker, lo_, hi_, rank, h->prm.eps_compress,
                                  h->prm.als_sweeps, hd->F, &hd->rep);
    }
    if (hd->R > (1 << 20)) { set_err("box CP width exceeds 2^20"); return nullptr; }
    if (hd->f32 && rs::window_row_chunks32(hd->R) == 0) {
      set_err("RS_FLAG_F32_FACTORS needs a compiled CP width R in {4, 8, 12, 16, 24, 32}, got " +
              std::to_string(hd->R));
      return nullptr;
    }
  } catch (const std::bad_alloc&) {
    set_err("out of host memory while restricting");
    return nullptr;
  }
  rs_handle* hd = H.get();
  if (!host_only) {
    if (upload_handle(hd) != 0) {
      std::string msg = g_err;
      free_device(hd);
      set_err(msg.empty() ? "upload failed" : msg);
      return nullptr;
    }
  }
  hd->setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return H.release();
}

int rs_export_tucker(const rs_handle* h, int32_t* r, double* U0, double* U1, double* U2, double* G) {
  if (!h || !r) { set_err("null argument"); return RS_E_INVALID_ARG; }
  const rs::TuckerRep& tk = h->tucker;
  if (tk.G.empty()) { set_err("this handle keeps no Tucker form (combined or box handle)"); return RS_E_INVALID_ARG; }
  for (int l = 0; l < 3; ++l) r[l] = tk.r[l];
  double* U[3] = {U0, U1, U2};
  for (int l = 0; l < 3; ++l)
    if (U[l])
      for (int i = 0; i < h->n; ++i)
        for (int a = 0; a < tk.r[l]; ++a) U[l][(size_t)i * tk.r[l] + a] = tk.U[l][(size_t)a * h->n + i];
  if (G) std::memcpy(G, tk.G.data(), tk.G.size() * sizeof(double));
  return 0;
}

int rs_score_path(rs_handle* h, const double* xyz_lig, int64_t n_lig) {
  if (!h || (n_lig > 0 && !xyz_lig) || n_lig < 0) { set_err("null or invalid argument"); return RS_E_INVALID_ARG; }
  if (n_lig > (int64_t)1 << 30) { set_err("n_lig too large"); return RS_E_INVALID_ARG; }
  if (!h->on_device) { set_err("handle has no device tables"); return RS_E_NO_DEVICE; }
  if (pointer_kind(xyz_lig) != 0) { set_err("rs_score_path needs a host ligand"); return RS_E_INVALID_ARG; }
  CUDA_TRY(cudaSetDevice(h->device), RS_E_CUDA);
  rs::ScoreArgs a = base_args(h);
  a.L = n_lig;
  a.P = 0;
  a.rmax_hint = ligand_rmax(h, xyz_lig, n_lig, false, nullptr);
  const int e = rs::plan_score(a, h->device);
  if (e < rs::kPathWindow || e > rs::kPathTucker) {
    set_err(std::string("launch plan failed: ") + cudaGetErrorString((cudaError_t)e));
    return RS_E_CUDA;
  }
  return e;
}

int rs_get_info(const rs_handle* h, rs_info* out) {
  if (!h || !out) { set_err("null argument"); return RS_E_INVALID_ARG; }
  std::memset(out, 0, sizeof(*out));
  out->n = h->n;
  out->b = h->b;
  out->h = h->h;
  out->inv_h = h->inv_h;
  out->R = h->R;
  out->R_exact = h->rep.R_exact;
  for (int i = 0; i < 3; ++i) out->tucker_r[i] = h->rep.tucker_r[i];
  out->quad_K = h->quad.K;
  out->quad_s = h->quad.s;
  out->quad_Ls = h->quad.Ls;
  out->quad_err = h->quad.err;
  out->R_long_ref = h->R_long_ref;
  out->R_short = h->Rs;
  out->n_sigma = h->n_sigma;
  out->n_atoms = h->M;
  out->tucker_err = h->rep.tucker_err;
  out->cp_core_err = h->rep.cp_core_err;
  out->sampled_max_err = h->rep.sampled_max;
  out->sampled_rms_err = h->rep.sampled_rms;
  out->n_err_samples = h->rep.n_samples;
  out->sigma_vdw = h->prm.sigma_vdw;
  out->dmin_cap = h->prm.dmin_cap;
  out->nbr_cells = (int64_t)h->cg.dim[0] * h->cg.dim[1] * h->cg.dim[2];
  out->nbr_entries = (int64_t)h->cg.idx.size();
  out->nbr_shift = h->cg.shift;
  out->device_bytes = h->device_bytes;
  out->setup_seconds = h->setup_seconds;
  out->on_device = h->on_device ? 1 : 0;
  out->factor_bits = h->f32 ? 32 : 64;
  for (int a = 0; a < 3; ++a) { out->box_lo[a] = h->box_lo[a]; out->box_hi[a] = h->box_hi[a]; }
  return 0;
}

int rs_export_tables(const rs_handle* h, double* F1, double* F2, double* F3, double* S1,
                     double* S2, double* S3) {
  if (!h) { set_err("null handle"); return RS_E_INVALID_ARG; }
  double* F[3] = {F1, F2, F3};
  double* S[3] = {S1, S2, S3};
  for (int a = 0; a < 3; ++a) {
    if (F[a]) std::copy(h->F[a].begin(), h->F[a].end(), F[a]);
    if (S[a]) std::copy(h->S[a].begin(), h->S[a].end(), S[a]);
  }
  return 0;
}

int rs_export_setup(const rs_handle* h, double* t, double* a, int32_t* is_long,
                    int32_t* protein_cells) {
  if (!h) { set_err("null handle"); return RS_E_INVALID_ARG; }
  if (t) std::copy(h->quad.t.begin(), h->quad.t.end(), t);
  if (a) std::copy(h->quad.a.begin(), h->quad.a.end(), a);
  if (is_long) std::copy(h->is_long.begin(), h->is_long.end(), is_long);
  if (protein_cells) std::copy(h->cells.begin(), h->cells.end(), protein_cells);
  return 0;
}

void rs_free(rs_handle* h) {
  if (!h) return;
  free_device(h);
  delete h;
}

int64_t rs_score_poses_async(rs_handle* h, const double* q_lig, const double* xyz_lig,
                             int64_t n_lig, const double* poses, int64_t P,
                             double* energies_out, double* mindist_out,
                             int64_t* invalid_count_dev, void* cuda_stream) {
  rs::NvtxRange nvtx_("rs_score_poses_async");
  if (!h) { set_err("null handle"); return RS_E_INVALID_ARG; }
  if (!h->on_device) { set_err("handle has no device tables"); return RS_E_NO_DEVICE; }
  if (n_lig < 0 || P < 0) { set_err("negative size"); return RS_E_INVALID_ARG; }
  if (P > 0 && (!poses || !energies_out || !mindist_out)) { set_err("null pose/output pointer"); return RS_E_INVALID_ARG; }
  if (n_lig > 0 && (!q_lig || !xyz_lig)) { set_err("null ligand pointer"); return RS_E_INVALID_ARG; }
  if (n_lig > (int64_t)1 << 30) { set_err("n_lig too large"); return RS_E_INVALID_ARG; }
  const void* ptrs[5] = {q_lig, xyz_lig, poses, energies_out, mindist_out};
  for (const void* p : ptrs)
    if (p && pointer_kind(p) != 1) { set_err("rs_score_poses_async needs device pointers"); return RS_E_INVALID_ARG; }
  CUDA_TRY(cudaSetDevice(h->device), RS_E_CUDA);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (invalid_count_dev)
    CUDA_TRY(cudaMemsetAsync(invalid_count_dev, 0, sizeof(int64_t), st), RS_E_CUDA);
  if (P == 0) return 0;
  rs::ScoreArgs a = base_args(h);
  a.zl = q_lig;
  a.yl = xyz_lig;
  a.L = n_lig;
  a.poses = poses;
  a.P = P;
  a.E = energies_out;
  a.D = mindist_out;
  a.invalid = (unsigned long long*)invalid_count_dev;
  {
    std::lock_guard<std::mutex> lock(h->mtx);
    a.rmax_hint = ligand_rmax(h, xyz_lig, n_lig, true, st);
  }
  int e = launch_with_counter(h, a, st);
  if (e != 0) {
    set_err(std::string("kernel launch failed: ") + cudaGetErrorString((cudaError_t)e));
    return RS_E_CUDA;
  }
  return 0;
}

int64_t rs_score_forces(rs_handle* h, const double* q_lig, const double* xyz_lig, int64_t n_lig,
                        const double* poses, int64_t P, double* forces_out,
                        int64_t* invalid_count_dev, void* cuda_stream) {
  rs::NvtxRange nvtx_("rs_score_forces");
  if (!h) { set_err("null handle"); return RS_E_INVALID_ARG; }
  if (!h->on_device) { set_err("handle has no device tables"); return RS_E_NO_DEVICE; }
  if (n_lig < 0 || P < 0) { set_err("negative size"); return RS_E_INVALID_ARG; }
  if (P > 0 && (!poses || !forces_out)) { set_err("null pose/output pointer"); return RS_E_INVALID_ARG; }
  if (n_lig > 0 && (!q_lig || !xyz_lig)) { set_err("null ligand pointer"); return RS_E_INVALID_ARG; }
  if (n_lig > (int64_t)1 << 30) { set_err("n_lig too large"); return RS_E_INVALID_ARG; }
  const void* ptrs[4] = {q_lig, xyz_lig, poses, forces_out};
  for (const void* p : ptrs)
    if (p && pointer_kind(p) != 1) { set_err("rs_score_forces needs device pointers"); return RS_E_INVALID_ARG; }
  CUDA_TRY(cudaSetDevice(h->device), RS_E_CUDA);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (invalid_count_dev)
    CUDA_TRY(cudaMemsetAsync(invalid_count_dev, 0, sizeof(int64_t), st), RS_E_CUDA);
  if (P == 0) return 0;
  rs::ScoreArgs a = base_args(h);
  a.zl = q_lig;
  a.yl = xyz_lig;
  a.L = n_lig;
  a.poses = poses;
  a.P = P;
  a.invalid = (unsigned long long*)invalid_count_dev;
  int e = rs::launch_forces(a, forces_out, st, h->device);
  if (e != 0) {
    set_err(std::string("force kernel launch failed: ") + cudaGetErrorString((cudaError_t)e));
    return RS_E_CUDA;
  }
  return 0;
}

int64_t rs_score_poses(rs_handle* h, const double* q_lig, const double* xyz_lig, int64_t n_lig,
                       const double* poses, int64_t P, double* energies_out, double* mindist_out) {
  rs::NvtxRange nvtx_("rs_score_poses");
  if (!h) { set_err("null handle"); return RS_E_INVALID_ARG; }
  if (!h->on_device) { set_err("handle has no device tables"); return RS_E_NO_DEVICE; }
  if (n_lig < 0 || P < 0) { set_err("negative size"); return RS_E_INVALID_ARG; }
  if (P > 0 && (!poses || !energies_out || !mindist_out)) { set_err("null pose/output pointer"); return RS_E_INVALID_ARG; }
  if (n_lig > 0 && (!q_lig || !xyz_lig)) { set_err("null ligand pointer"); return RS_E_INVALID_ARG; }
  if (n_lig > (int64_t)1 << 30) { set_err("n_lig too large"); return RS_E_INVALID_ARG; }
  if (P == 0) return 0;
  std::lock_guard<std::mutex> lock(h->mtx);
  CUDA_TRY(cudaSetDevice(h->device), RS_E_CUDA);
  // synchronous API: order after any prior work on the device that produced the inputs
  CUDA_TRY(cudaDeviceSynchronize(), RS_E_CUDA);
  const bool lig_dev = n_lig == 0 || (pointer_kind(q_lig) == 1 && pointer_kind(xyz_lig) == 1);
  const bool pose_dev = pointer_kind(poses) == 1;
  const bool e_dev = pointer_kind(energies_out) == 1;
  const bool d_dev = pointer_kind(mindist_out) == 1;
  // pipeline over kStreams streams: H2D(chunk) -> kernel -> D2H(chunk), chunk sizes growing
  // geometrically (x1.5 from ~P/16), so the first copy exposes little and the later copies hide
  // behind the kernels of the earlier chunks; every chunk has its own staging region, and the
  // kernels of different chunks may overlap on the device
  constexpr int kStreams = 3;
  // 256-byte aligned sections (the streamed pipeline relies on 128-byte aligned pose chunks)
  const size_t lig_b = ((size_t)4 * std::max<int64_t>(n_lig, 1) * sizeof(double) + 255) / 256 * 256;
  const size_t pose_b = pose_dev ? 0 : (size_t)P * 7 * sizeof(double);
  const size_t out_b = (size_t)P * sizeof(double);
  const size_t need = lig_b + pose_b + (e_dev ? 0 : out_b) + (d_dev ? 0 : out_b) + 64 * kStreams +
                      4096;   // + streamed-pipeline flags, counters and chunk bounds
  if (h->stage_bytes < need) {
    if (h->stage) cudaFree(h->stage);
    h->stage = nullptr;
    h->stage_bytes = 0;
    CUDA_TRY(cudaMalloc(&h->stage, need), RS_E_NOMEM);
    h->stage_bytes = need;
  }
  for (void*& s : h->streams)
    if (!s) CUDA_TRY(cudaStreamCreateWithFlags((cudaStream_t*)&s, cudaStreamNonBlocking), RS_E_CUDA);
  char* base = (char*)h->stage;
  double* d_lig = (double*)base;
  double* d_pose = (double*)(base + lig_b);
  double* d_E = (double*)(base + lig_b + pose_b);
  double* d_D = (double*)(base + lig_b + pose_b + (e_dev ? 0 : out_b));
  unsigned long long* d_cnt =
      (unsigned long long*)(base + lig_b + pose_b + (e_dev ? 0 : out_b) + (d_dev ? 0 : out_b));
  cudaStream_t st[kStreams];
  for (int i = 0; i < kStreams; ++i) st[i] = (cudaStream_t)h->streams[i];
  const double *zl = q_lig, *yl = xyz_lig;
  if (!lig_dev) {
    CUDA_TRY(cudaMemcpyAsync(d_lig, q_lig, n_lig * sizeof(double), cudaMemcpyHostToDevice, st[0]), RS_E_CUDA);
    CUDA_TRY(cudaMemcpyAsync(d_lig + n_lig, xyz_lig, 3 * n_lig * sizeof(double), cudaMemcpyHostToDevice, st[0]), RS_E_CUDA);
    zl = d_lig;
    yl = d_lig + n_lig;
  }
  CUDA_TRY(cudaMemsetAsync(d_cnt, 0, kStreams * sizeof(unsigned long long), st[0]), RS_E_CUDA);
  cudaEvent_t ready;
  CUDA_TRY(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), RS_E_CUDA);
  CUDA_TRY(cudaEventRecord(ready, st[0]), RS_E_CUDA);
  for (int i = 1; i < kStreams; ++i) CUDA_TRY(cudaStreamWaitEvent(st[i], ready, 0), RS_E_CUDA);
  cudaEventDestroy(ready);
  rs::ScoreArgs a = base_args(h);
  a.zl = zl;
  a.yl = yl;
  a.L = n_lig;
  a.rmax_hint = ligand_rmax(h, xyz_lig, n_lig, lig_dev, st[0]);
  static const bool streamed_off = std::getenv("RS_NO_STREAMED") != nullptr;
  // streamed only for large batches: below ~4e5 poses (C2: 1e5) the per-chunk stream waits cost
  // more than the launch ramps they save (measured: C2 all-host 0.40 ms streamed, 0.36 chunked).
  // RS_STREAM_MIN_POSES moves the threshold (the sanitizer runs use it on small batches).
  static const int64_t stream_min = [] {
    const char* v = std::getenv("RS_STREAM_MIN_POSES");
    return v ? std::max<int64_t>(1, std::atoll(v)) : (int64_t)400000;
  }();
  static std::atomic<bool> stream_broken{false};   // a streamed launch stalled once: no more
  if (!pose_dev && !e_dev && !d_dev && P >= stream_min && wait_value32() && !streamed_off &&
      !stream_broken.load()) {
    // Streamed pipeline: ONE launch over all P poses on stream 0 while stream 1 copies the
    // poses in geometrically growing chunks, each followed by its arrival flag; the kernel
    // waits for a chunk's flag before it scores poses from it and counts finished poses per
    // chunk; stream 2 waits for each chunk's count (cuStreamWaitValue32) and copies its
    // energies and distances back.  No per-chunk launch ramp or tail.
    constexpr int kMaxCb = 64;
    long long cb[kMaxCb + 1];
    int n_cb = 0;
    cb[0] = 0;
    // sizes grow x1.5 over the first half and mirror over the second (the middle never more
    // than 1.5x its neighbours), so the last result copy, exposed after the kernel, is small
    std::vector<int64_t> up;
    int64_t tot = 0;
    // first chunk P/16 (C3, all-host call: P/128 2.01 ms, P/32 1.99, P/16 1.95, P/8 2.00): the
    // kernel's 148 CTAs hold ~150K claimed poses at a time, so early chunks must not be tiny
    for (int64_t sz = std::max<int64_t>(4096, P / 16); 2 * (tot + sz) <= P && (int)up.size() < kMaxCb / 2 - 2;
         sz += sz / 2) {
      up.push_back(sz);
      tot += sz;
    }
    std::vector<int64_t> sizes(up);
    const int64_t mid = P - 2 * tot;               // never more than 1.5x its neighbours
    if (mid > 0 && !up.empty() && mid > up.back() + up.back() / 2) {
      sizes.push_back(mid / 2);
      sizes.push_back(mid - mid / 2);
    } else if (mid > 0) {
      sizes.push_back(mid);
    }
    sizes.insert(sizes.end(), up.rbegin(), up.rend());
    for (int64_t sz : sizes) {
      int64_t e = cb[n_cb] + sz;
      e = (e + 15) / 16 * 16;                                      // 16 poses = 7 x 128 bytes
      if (e >= P || n_cb + 1 == kMaxCb) e = P;
      if (e <= cb[n_cb]) continue;
      cb[++n_cb] = e;
      if (e == P) break;
    }
    if (cb[n_cb] < P) cb[++n_cb] = P;
    unsigned* d_arrive = (unsigned*)(d_cnt + kStreams);
    unsigned* d_done = d_arrive + kMaxCb;
    unsigned* d_stall = d_done + kMaxCb;
    long long* d_cb = (long long*)(d_stall + 2);
    if (!h->h_ones) {
      CUDA_TRY(cudaMallocHost((void**)&h->h_ones, kMaxCb * sizeof(unsigned)), RS_E_NOMEM);
      for (int i = 0; i < kMaxCb; ++i) h->h_ones[i] = 1u;
    }
    CUDA_TRY(cudaMemsetAsync(d_arrive, 0, (2 * kMaxCb + 2) * sizeof(unsigned), st[0]), RS_E_CUDA);
    CUDA_TRY(cudaMemcpyAsync(d_cb, cb, (n_cb + 1) * sizeof(long long), cudaMemcpyHostToDevice, st[0]), RS_E_CUDA);
    cudaEvent_t armed;
    CUDA_TRY(cudaEventCreateWithFlags(&armed, cudaEventDisableTiming), RS_E_CUDA);
    CUDA_TRY(cudaEventRecord(armed, st[0]), RS_E_CUDA);
    CUDA_TRY(cudaStreamWaitEvent(st[1], armed, 0), RS_E_CUDA);
    CUDA_TRY(cudaStreamWaitEvent(st[2], armed, 0), RS_E_CUDA);
    cudaEventDestroy(armed);
    // fault injection for the stall path's test: arrival flags never sent
    static const bool drop_flags = std::getenv("RS_STREAM_FAULT_DROP_FLAGS") != nullptr;
    for (int i = 0; i < n_cb; ++i) {
      CUDA_TRY(cudaMemcpyAsync(d_pose + 7 * cb[i], poses + 7 * cb[i], (cb[i + 1] - cb[i]) * 7 * sizeof(double),
                               cudaMemcpyHostToDevice, st[1]), RS_E_CUDA);
      if (!drop_flags)
        CUDA_TRY(cudaMemcpyAsync(d_arrive + i, h->h_ones + i, sizeof(unsigned), cudaMemcpyHostToDevice, st[1]), RS_E_CUDA);
    }
    a.poses = d_pose;
    a.P = P;
    a.E = d_E;
    a.D = d_D;
    a.invalid = d_cnt;
    a.arrive = d_arrive;
    a.done = d_done;
    a.cb = d_cb;
    a.n_cb = n_cb;
    a.stall = d_stall;
    int e = launch_with_counter(h, a, st[0]);
    if (e != 0) {
      set_err(std::string("kernel launch failed: ") + cudaGetErrorString((cudaError_t)e));
      return RS_E_CUDA;
    }
    PFN_waitValue32 wv = wait_value32();
    for (int i = 0; i < n_cb; ++i) {
      const int64_t off = cb[i], cnt = cb[i + 1] - cb[i];
      if (wv((CUstream)st[2], (CUdeviceptr)(d_done + i), (cuuint32_t)cnt, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) {
        set_err("cuStreamWaitValue32 failed");
        return RS_E_CUDA;
      }
      CUDA_TRY(cudaMemcpyAsync(energies_out + off, d_E + off, cnt * sizeof(double), cudaMemcpyDeviceToHost, st[2]), RS_E_CUDA);
      CUDA_TRY(cudaMemcpyAsync(mindist_out + off, d_D + off, cnt * sizeof(double), cudaMemcpyDeviceToHost, st[2]), RS_E_CUDA);
    }
    for (int i = 0; i < kStreams; ++i) CUDA_TRY(cudaStreamSynchronize(st[i]), RS_E_CUDA);
    unsigned long long cnt0 = 0;
    unsigned stall = 0;
    CUDA_TRY(cudaMemcpy(&cnt0, d_cnt, sizeof(cnt0), cudaMemcpyDeviceToHost), RS_E_CUDA);
    CUDA_TRY(cudaMemcpy(&stall, d_stall, sizeof(stall), cudaMemcpyDeviceToHost), RS_E_CUDA);
    if (!stall) return (int64_t)cnt0;
    // the copies did not run beside the kernel: its results are void; recompute the batch with
    // the chunked launches below (every later call skips streaming)
    stream_broken.store(true);
    CUDA_TRY(cudaMemset(d_cnt, 0, kStreams * sizeof(unsigned long long)), RS_E_CUDA);
    std::fprintf(stderr, "[rsdock] streamed pipeline stalled (copy engine not concurrent with the kernel); "
                         "recomputing with chunked launches\n");
  }
  int chunk = 0;
  // first chunk P/16 (measured at C3 on pinned host buffers: P/64 2.185 ms, P/16 2.147 ms; the
  // rest of the gap to the 1.69 ms device-resident launch is the ramp and tail of each chunk's
  // launch: the same chunking on device buffers takes 1.93-2.04 ms, one launch 1.72 ms)
  int64_t csz = std::min<int64_t>(P, std::max<int64_t>(4096, P / 16));
  for (int64_t off = 0; off < P; off += csz, csz = csz + csz / 2, ++chunk) {
    const int64_t cnt = std::min(csz, P - off);
    const int s = chunk % kStreams;
    const double* pp = poses + 7 * off;
    if (!pose_dev) {
      CUDA_TRY(cudaMemcpyAsync(d_pose + 7 * off, pp, cnt * 7 * sizeof(double), cudaMemcpyHostToDevice, st[s]), RS_E_CUDA);
      pp = d_pose + 7 * off;
    }
    a.poses = pp;
    a.P = cnt;
    a.E = e_dev ? energies_out + off : d_E + off;
    a.D = d_dev ? mindist_out + off : d_D + off;
    a.invalid = d_cnt + s;
    int e = launch_with_counter(h, a, st[s]);
    if (e != 0) {
      set_err(std::string("kernel launch failed: ") + cudaGetErrorString((cudaError_t)e));
      return RS_E_CUDA;
    }
    if (!e_dev) CUDA_TRY(cudaMemcpyAsync(energies_out + off, d_E + off, cnt * sizeof(double), cudaMemcpyDeviceToHost, st[s]), RS_E_CUDA);
    if (!d_dev) CUDA_TRY(cudaMemcpyAsync(mindist_out + off, d_D + off, cnt * sizeof(double), cudaMemcpyDeviceToHost, st[s]), RS_E_CUDA);
  }
  for (int i = 0; i < kStreams; ++i) CUDA_TRY(cudaStreamSynchronize(st[i]), RS_E_CUDA);
  unsigned long long cnts[kStreams] = {0, 0, 0};
  CUDA_TRY(cudaMemcpy(cnts, d_cnt, sizeof(cnts), cudaMemcpyDeviceToHost), RS_E_CUDA);
  return (int64_t)(cnts[0] + cnts[1] + cnts[2]);
}

int32_t rs_landscape_minima(const double* E, int32_t m_P, int32_t m_L, int32_t top_k,
                            int32_t* idx_out) {
  if (!E || m_P <= 0 || m_L <= 0 || top_k < 0 || (top_k > 0 && !idx_out)) {
    set_err("rs_landscape_minima: bad arguments");
    return RS_E_INVALID_ARG;
  }
  // PPIEM step A6 (reading A23): strict local minima on the periodic grid; a tie with
  // a neighbour goes to the lexicographically smaller index; NaN entries are skipped
  std::vector<int32_t> mins;
  for (int32_t j = 0; j < m_P; ++j)
    for (int32_t k = 0; k < m_L; ++k) {
      const double e = E[(int64_t)j * m_L + k];
      if (std::isnan(e)) continue;
      bool is_min = true;
      for (int dj = -1; dj <= 1 && is_min; ++dj)
        for (int dk = -1; dk <= 1 && is_min; ++dk) {
          const int32_t jj = ((j + dj) % m_P + m_P) % m_P, kk = ((k + dk) % m_L + m_L) % m_L;
          if (jj == j && kk == k) continue;
          const double f = E[(int64_t)jj * m_L + kk];
          if (std::isnan(f)) continue;
          if (f < e || (f == e && (jj < j || (jj == j && kk < k)))) is_min = false;
        }
      if (is_min) mins.push_back(j * m_L + k);
    }
  std::stable_sort(mins.begin(), mins.end(), [&](int32_t x, int32_t y) { return E[x] < E[y]; });
  const int32_t cnt = std::min<int32_t>(top_k, (int32_t)mins.size());
  for (int32_t i = 0; i < cnt; ++i) idx_out[i] = mins[i];
  return cnt;
}

int64_t rs_ppiem_scan(rs_handle* h, const double* q_lig, const double* xyz_lig, int64_t n_lig,
                      const double* centre, const double* dirs, int32_t m_P, const double* quats,
                      int32_t m_L, double s_start, double tol, int32_t max_iter,
                      double* energies_out, double* s_out, int32_t* status_out) {
  rs::NvtxRange nvtx_("rs_ppiem_scan");
  if (!h) { set_err("null handle"); return RS_E_INVALID_ARG; }
  if (!h->on_device) { set_err("handle has no device tables"); return RS_E_NO_DEVICE; }
  if (!centre || !dirs || !quats || !energies_out || !s_out || !status_out || m_P <= 0 || m_L <= 0 ||
      max_iter < 1 || !(tol > 0) || !std::isfinite(s_start) || s_start < 0 || n_lig < 0 ||
      (n_lig > 0 && (!q_lig || !xyz_lig))) {
    set_err("rs_ppiem_scan: bad arguments");
    return RS_E_INVALID_ARG;
  }
  if (!(h->prm.dmin_cap > h->prm.sigma_vdw)) {
    set_err("rs_ppiem_scan needs dmin_cap > sigma_vdw (the sphere-tracing step)");
    return RS_E_INVALID_ARG;
  }
  if (n_lig > ((int64_t)1 << 30)) { set_err("n_lig too large"); return RS_E_INVALID_ARG; }
  for (int32_t j = 0; j < m_P; ++j) {
    // the sphere-tracing step never exceeds the clearance only along unit directions
    const double* u = dirs + 3 * (size_t)j;
    const double nn = std::sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
    if (!(std::fabs(nn - 1.0) <= 1e-9)) {
      set_err("rs_ppiem_scan: dirs[" + std::to_string(j) + "] is not a unit vector");
      return RS_E_INVALID_ARG;
    }
  }
  std::lock_guard<std::mutex> lock(h->mtx);
  CUDA_TRY(cudaSetDevice(h->device), RS_E_CUDA);
  const int64_t P = (int64_t)m_P * m_L;
  const bool lig_dev = n_lig == 0 || (pointer_kind(q_lig) == 1 && pointer_kind(xyz_lig) == 1);
  // device scratch, kept on the handle (grow-only):
  //   [ligand 4L][centre 3][dirs 3 m_P][quats 4 m_L][poses 2 x 7P][Ec P][Dc P][E P][s P]
  //   [status P int][slot P int][count 2 int][invalid u64]
  const size_t nd = 4 * (size_t)std::max<int64_t>(n_lig, 1) + 3 + 3 * (size_t)m_P + 4 * (size_t)m_L +
                    18 * (size_t)P;
  const size_t bytes = nd * sizeof(double) + (2 * (size_t)P + 4) * sizeof(int) + 16;
  if (h->scan_bytes < bytes) {
    if (h->scan_buf) cudaFree(h->scan_buf);
    h->scan_buf = nullptr;
    h->scan_bytes = 0;
    CUDA_TRY(cudaMalloc(&h->scan_buf, bytes), RS_E_NOMEM);
    h->scan_bytes = bytes;
  }
  double* d_lig = (double*)h->scan_buf;
  double* d_c = d_lig + 4 * std::max<int64_t>(n_lig, 1);
  double* d_dirs = d_c + 3;
  double* d_q = d_dirs + 3 * (size_t)m_P;
  double* d_pose[2] = {d_q + 4 * (size_t)m_L, d_q + 4 * (size_t)m_L + 7 * P};
  double* d_Ec = d_pose[1] + 7 * P;
  double* d_Dc = d_Ec + P;
  double* d_E = d_Dc + P;
  double* d_s = d_E + P;
  int* d_st = (int*)(d_s + P);
  int* d_slot = d_st + P;
  int* d_count = d_slot + P;
  unsigned long long* d_inv = (unsigned long long*)(((uintptr_t)(d_count + 2) + 7) & ~(uintptr_t)7);
  const double *zl = q_lig, *yl = xyz_lig;
  if (!lig_dev) {
    CUDA_TRY(cudaMemcpy(d_lig, q_lig, n_lig * sizeof(double), cudaMemcpyHostToDevice), RS_E_CUDA);
    CUDA_TRY(cudaMemcpy(d_lig + n_lig, xyz_lig, 3 * n_lig * sizeof(double), cudaMemcpyHostToDevice), RS_E_CUDA);
    zl = d_lig;
    yl = d_lig + n_lig;
  }
  CUDA_TRY(cudaMemcpy(d_c, centre, 3 * sizeof(double), cudaMemcpyHostToDevice), RS_E_CUDA);
  CUDA_TRY(cudaMemcpy(d_dirs, dirs, 3 * (size_t)m_P * sizeof(double), cudaMemcpyHostToDevice), RS_E_CUDA);
  CUDA_TRY(cudaMemcpy(d_q, quats, 4 * (size_t)m_L * sizeof(double), cudaMemcpyHostToDevice), RS_E_CUDA);
  cudaStream_t st = nullptr;
  if (int e = rs::launch_scan_init(d_c, d_dirs, d_q, m_P, m_L, s_start, d_pose[0], d_s, d_st, d_slot, st)) {
    set_err(std::string("scan init failed: ") + cudaGetErrorString((cudaError_t)e));
    return RS_E_CUDA;
  }
  rs::ScoreArgs a = base_args(h);
  a.zl = zl;
  a.yl = yl;
  a.L = n_lig;
  a.rmax_hint = ligand_rmax(h, xyz_lig, n_lig, lig_dev, nullptr);
  a.E = d_Ec;
  a.D = d_Dc;
  a.invalid = d_inv;
  const double sigma = h->prm.sigma_vdw, dcap = h->prm.dmin_cap;
  auto score = [&](const double* poses_cur, int64_t n) -> int {
    a.poses = poses_cur;
    a.P = n;
    return launch_with_counter(h, a, st);
  };
  int cur = 0;
  int64_t n_cur = P;
  for (int it = 0; it < max_iter && n_cur > 0; ++it) {
    // score the poses still moving (compacted), then step them and compact the next list
    if (int e = score(d_pose[cur], n_cur)) { set_err("scan scoring launch failed: " + std::to_string(e)); return RS_E_CUDA; }
    CUDA_TRY(cudaMemsetAsync(d_count, 0, sizeof(int), st), RS_E_CUDA);
    if (int e = rs::launch_scan_update(d_c, d_dirs, d_q, m_P, m_L, d_Dc, d_Ec, sigma, dcap, tol,
                                       it == 0, d_E, d_s, d_st, d_slot, d_pose[1 - cur], d_count, st)) {
      set_err(std::string("scan update failed: ") + cudaGetErrorString((cudaError_t)e));
      return RS_E_CUDA;
    }
    int n_next = 0;
    CUDA_TRY(cudaMemcpy(&n_next, d_count, sizeof(int), cudaMemcpyDeviceToHost), RS_E_CUDA);
    n_cur = n_next;
    cur = 1 - cur;
  }
  // poses still moving after max_iter were stepped after their last scoring: score them where
  // they stand (feasible by construction) and report status 4
  if (n_cur > 0) {
    if (int e = score(d_pose[cur], n_cur)) { set_err("scan scoring launch failed: " + std::to_string(e)); return RS_E_CUDA; }
    if (int e = rs::launch_scan_gather(P, d_st, d_slot, d_Ec, d_E, st)) {
      set_err(std::string("scan gather failed: ") + cudaGetErrorString((cudaError_t)e));
      return RS_E_CUDA;
    }
  }
  CUDA_TRY(cudaDeviceSynchronize(), RS_E_CUDA);
  std::vector<int> stv(P);
  CUDA_TRY(cudaMemcpy(energies_out, d_E, P * sizeof(double), cudaMemcpyDeviceToHost), RS_E_CUDA);
  CUDA_TRY(cudaMemcpy(s_out, d_s, P * sizeof(double), cudaMemcpyDeviceToHost), RS_E_CUDA);
  CUDA_TRY(cudaMemcpy(stv.data(), d_st, P * sizeof(int), cudaMemcpyDeviceToHost), RS_E_CUDA);
  for (int64_t p = 0; p < P; ++p) {
    const int sv = stv[p] == -1 ? 4 : stv[p];
    status_out[p] = sv;
    if (sv != 0 && sv != 4) energies_out[p] = NAN;
  }
  return 0;
}

}  // extern "C"

// ---- handle save / load (SPEC.md:207's kernel cache) ---------------------------
// One binary file: "RSDOCK02", then every host-side field of the handle in a fixed order (PODs
// raw, vectors as a u64 count + elements), then a 64-bit FNV-1a hash of everything before it.
// Loading restores the host tables bit for bit and uploads them like a build (S10).
namespace {
struct Writer {
  std::vector<unsigned char> buf;
  template <class T> void pod(const T& v) {
    const unsigned char* p = reinterpret_cast<const unsigned char*>(&v);
    buf.insert(buf.end(), p, p + sizeof(T));
  }
  template <class T> void vec(const std::vector<T>& v) {
    pod<uint64_t>(v.size());
    const unsigned char* p = reinterpret_cast<const unsigned char*>(v.data());
    buf.insert(buf.end(), p, p + v.size() * sizeof(T));
  }
};
struct Reader {
  const unsigned char* p;
  size_t left;
  bool ok = true;
  template <class T> void pod(T& v) {
    if (!ok || left < sizeof(T)) { ok = false; return; }
    std::memcpy(&v, p, sizeof(T));
    p += sizeof(T);
    left -= sizeof(T);
  }
  template <class T> void vec(std::vector<T>& v) {
    uint64_t n = 0;
    pod(n);
    if (!ok || n > left / sizeof(T)) { ok = false; return; }
    v.assign(reinterpret_cast<const T*>(p), reinterpret_cast<const T*>(p) + n);
    p += n * sizeof(T);
    left -= n * sizeof(T);
  }
};
uint64_t fnv1a(const unsigned char* p, size_t n) {
  uint64_t x = 1469598103934665603ull;
  for (size_t i = 0; i < n; ++i) x = (x ^ p[i]) * 1099511628211ull;
  return x;
}
constexpr char kMagic[8] = {'R', 'S', 'D', 'O', 'C', 'K', '0', '2'};

// the handle's host fields in file order (Archive = Writer or Reader)
template <class A, class H>
void archive_handle(A& ar, H& h) {
  ar.pod(h.prm);
  ar.pod(h.n); ar.pod(h.b); ar.pod(h.h); ar.pod(h.inv_h);
  ar.pod(h.quad.s); ar.pod(h.quad.Ls); ar.pod(h.quad.err); ar.pod(h.quad.K);
  ar.vec(h.quad.t); ar.vec(h.quad.a);
  ar.vec(h.is_long);
  ar.pod(h.R); ar.pod(h.Rs); ar.pod(h.n_sigma); ar.pod(h.R_long_ref);
  for (int a = 0; a < 3; ++a) ar.vec(h.F[a]);
  for (int a = 0; a < 3; ++a) ar.vec(h.S[a]);
  ar.pod(h.M);
  ar.vec(h.xyz); ar.vec(h.z); ar.vec(h.cells);
  ar.pod(h.cg.shift); ar.pod(h.cg.lo); ar.pod(h.cg.dim); ar.vec(h.cg.off); ar.vec(h.cg.idx);
  ar.pod(h.rep);
  ar.pod(h.tucker.r);
  for (int a = 0; a < 3; ++a) ar.vec(h.tucker.U[a]);
  ar.vec(h.tucker.G);
  ar.pod(h.box_lo); ar.pod(h.box_hi);
  ar.pod(h.setup_seconds);
  ar.pod(h.f32);
}
}  // namespace

extern "C" {

int rs_save_handle(const rs_handle* h, const char* path) {
  if (!h || !path) { set_err("null argument"); return RS_E_INVALID_ARG; }
  rs::NvtxRange nvtx_("rs_save_handle");
  Writer w;
  try {
    w.buf.insert(w.buf.end(), kMagic, kMagic + 8);
    w.pod<uint32_t>(sizeof(rs_params));
    archive_handle(w, *h);
    w.pod(fnv1a(w.buf.data(), w.buf.size()));
  } catch (const std::bad_alloc&) {
    set_err("out of host memory");
    return RS_E_NOMEM;
  }
  FILE* f = std::fopen(path, "wb");
  if (!f) { set_err(std::string("cannot open ") + path + " for writing"); return RS_E_INVALID_ARG; }
  const size_t n = std::fwrite(w.buf.data(), 1, w.buf.size(), f);
  const int cl = std::fclose(f);
  if (n != w.buf.size() || cl != 0) { set_err(std::string("short write to ") + path); return RS_E_INVALID_ARG; }
  return 0;
}

rs_handle* rs_load_handle(const char* path, int32_t device, int32_t flags) {
  if (!path) { set_err("null argument"); return nullptr; }
  rs::NvtxRange nvtx_("rs_load_handle");
  std::vector<unsigned char> buf;
  {
    FILE* f = std::fopen(path, "rb");
    if (!f) { set_err(std::string("cannot open ") + path); return nullptr; }
    unsigned char tmp[1 << 16];
    size_t k;
    while ((k = std::fread(tmp, 1, sizeof(tmp), f)) > 0) buf.insert(buf.end(), tmp, tmp + k);
    std::fclose(f);
  }
  if (buf.size() < 8 + 4 + 8 || std::memcmp(buf.data(), kMagic, 8) != 0) {
    set_err(std::string(path) + ": not an rsdock handle file (magic)");
    return nullptr;
  }
  uint64_t stored = 0;
  std::memcpy(&stored, buf.data() + buf.size() - 8, 8);
  if (fnv1a(buf.data(), buf.size() - 8) != stored) {
    set_err(std::string(path) + ": checksum mismatch (truncated or corrupted)");
    return nullptr;
  }
  Reader r{buf.data() + 8, buf.size() - 16};
  uint32_t psz = 0;
  r.pod(psz);
  if (psz != sizeof(rs_params)) { set_err("handle file from an incompatible library version"); return nullptr; }
  std::unique_ptr<rs_handle> H;
  try {
    H.reset(new rs_handle());
    archive_handle(r, *H);
  } catch (const std::bad_alloc&) {
    set_err("out of host memory");
    return nullptr;
  }
  if (!r.ok || r.left != 0) { set_err(std::string(path) + ": malformed handle file"); return nullptr; }
  rs_handle* hd = H.get();
  const bool host_only = (flags & RS_FLAG_HOST_ONLY) != 0;
  hd->prm.device = device >= 0 ? device : hd->prm.device;
  hd->prm.flags = (hd->prm.flags & ~RS_FLAG_HOST_ONLY) | (flags & RS_FLAG_HOST_ONLY);
  hd->device = hd->prm.device;
  if (!host_only) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= hd->device || hd->device < 0) {
      cudaGetLastError();
      set_err("no CUDA device (there is no CPU fallback; use RS_FLAG_HOST_ONLY for host-only tables)");
      return nullptr;
    }
    if (upload_handle(hd) != 0) {
      std::string msg = g_err;
      free_device(hd);
      set_err(msg.empty() ? "upload failed" : msg);
      return nullptr;
    }
  }
  return H.release();
}

}  // extern "C"
