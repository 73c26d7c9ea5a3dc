// Internal declarations of librsdock (not part of the C ABI; see include/rs_dock.h).
#pragma once

#include <nvtx3/nvToolsExt.h>   // NVTX v3, header-only: ranges cost nothing without a profiler

#include <cuda_runtime.h>

#include <cstdint>
#include <atomic>
#include <complex>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rs_dock.h"

namespace rs {

// NVTX range over a C-ABI call or a setup phase (visible in nsys / ncu --nvtx timelines)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};


// ---- host setup (Algorithm TEP) --------------------------------------

struct Quadrature {          // S1: 1/r ~ sum_k a_k exp(-t_k^2 r^2)   (Eq. (2))
  double s = 0, Ls = 0, err = 0;
  int K = 0;
  std::vector<double> t, a;  // k = 0..K
};

Quadrature choose_quadrature(double eps, double rmin, double rmax, double Ls);
// S2: long iff t_k == 0 or sqrt(ln(1/eps_split))/t_k >= sigma_s  (Eq. (4))
bool is_long_term(double t, double sigma_s, double eps_split);
// S3: (1/h) * integral over cell d of exp(-t^2 x^2)  (Eq. (1))
double cell_average(double t, double h, long d);

struct CoarseGrid {          // S9 neighbour structure (cell lists over coarse cells)
  int shift = 0;             // coarse cell = 2^shift fine cells per axis
  int lo[3] = {0, 0, 0};     // first coarse index per axis
  int dim[3] = {0, 0, 0};    // coarse cells per axis
  std::vector<int32_t> off;  // CSR offsets (ncells + 1)
  std::vector<int32_t> idx;  // protein atom indices
};

struct SetupReport {
  int tucker_r[3] = {0, 0, 0};
  int R_exact = 0;
  double tucker_err = 0, cp_core_err = 0, sampled_max = 0, sampled_rms = 0;
  int n_samples = 0;
};

struct TuckerRep {           // the long-range part in Tucker format (S5-S6), kept for N3
  int r[3] = {0, 0, 0};
  std::vector<double> U[3];  // n x r_l, column-major (column a contiguous)
  std::vector<double> G;     // r0 x r1 x r2, row-major
};

// S6 on the device (setup_device.cu): accumulates the Tucker core term by term, bitwise equal to
// the host loop.  ok() is false when the device could not be used (the host loop runs then).
class CoreDevice {
 public:
  CoreDevice(int device, int n, const int* r, const std::vector<int32_t>& cells,
             const std::vector<double>& z);
  ~CoreDevice();
  bool ok() const;
  bool add_term(double a_k, const std::vector<double> H[3]);   // H_l: n x r_l row-major
  // every term k on the device: H_l = (T_k U_l) from the device convolutions straight into the
  // accumulation (U_l: n x r_l column-major, uploaded once; no host round trip per term)
  bool add_terms_device(class DeviceConv& conv, const std::vector<double> U[3],
                        const std::vector<double>& a_long);
  bool fetch(std::vector<double>& G);
 private:
  struct Impl;
  Impl* p;
};

// Opt-in (RS_FLAG_DEVICE_FFT): the setup's convolutions y_s = T_k x_s on the device with cuFFT
// (the same FFT-domain product as ConvOps::apply_one; tables then differ from the host-only
// build by rounding).  apply() is serialised internally.
class DeviceConv {
 public:
  DeviceConv(int device, int n, int N, const std::vector<std::vector<std::complex<double>>>& FG);
  ~DeviceConv();
  bool ok() const;
  bool apply(int k, const double* X, double* Y, int cols);   // X, Y: n x cols column-major
 private:
  friend class CoreDevice;
  friend class RangeFinderDevice;
  struct Impl;
  Impl* p;
};

// S7: Tucker core -> CP of width rank_R (0: eps mode); returns R
// The RHOSVD range finder of one mode with every convolution on the device (device-FFT builds,
// no box): the sketch sum_k T_k (sqrt(c_k) .* Xi_k) (the host's counter-based normal draws,
// generated on the device), the power step sum_k T_k (c_k .* (T_k Q)) and the p x p Gram matrix
// sum_k sum_j c_k[j] (T_k Q)[j,:]^T (T_k Q)[j,:], each sum in k order; the orthonormalisations
// stay on the host (small).  Any failure returns false and the caller runs the host path.
class RangeFinderDevice {
 public:
  RangeFinderDevice(DeviceConv& conv, const std::vector<std::vector<double>>& c, int n);
  ~RangeFinderDevice();
  bool ok() const;
  bool sketch(int p, uint64_t seed, int mode, const std::vector<int>& occj, std::vector<double>& Y);
  bool power(const std::vector<double>& Q, int p, std::vector<double>& Y);
  bool gram(const std::vector<double>& Q, int p, std::vector<double>& Gm);
 private:
  bool reserve(int p);
  bool apply(int k, const double* dX, double* dY, int p);   // device buffers, n x p col-major
  struct Impl;
  Impl* q;
};

int core_to_cp(const std::vector<double>& G, int r0, int r1, int r2, int rank_R, double eps,
               int als_sweeps, std::vector<double>& A, std::vector<double>& B,
               std::vector<double>& C, int* R_exact, double* rel_err);

// N3 scheme (C): CP of the long-range part restricted to the cell box [lo, hi] (rows outside NaN)
int restrict_to_box(int n, const TuckerRep& tk, const int lo[3], const int hi[3], int rank,
                    double eps, int als_sweeps, std::vector<double> F[3], SetupReport* rep);

// S5-S7: rank-R CP factors (n x R row-major each) of the protein's long-range potential
// P_l[i] = sum_m z_m sum_{k long} a_k prod_a g_k[i_a - i_{m,a}]   (Eq. (6))
void compress_long_range(int n, double h, const std::vector<int32_t>& cells,
                         const std::vector<double>& z, const std::vector<double>& t_long,
                         const std::vector<double>& a_long, int rank_R, double eps,
                         int tucker_cap, int als_sweeps, uint64_t seed,
                         std::vector<double> F[3], int* R_out, SetupReport* rep,
                         TuckerRep* tk = nullptr, const int* box_lo = nullptr,
                         const int* box_hi = nullptr, int device = -1, bool device_fft = false);

void build_cell_lists(int n, double b, double h, const std::vector<double>& xyz,
                      const std::vector<int32_t>& cells, double rho, double cell_edge,
                      CoarseGrid* cg);

void sample_compression_error(int n, double b, double h, const std::vector<double>& xyz,
                              const std::vector<int32_t>& cells, const std::vector<double>& z,
                              const std::vector<double>& t_long, const std::vector<double>& a_long,
                              const std::vector<double> F[3], int R, double r_excl,
                              const CoarseGrid& cg, int n_samples, uint64_t seed,
                              SetupReport* rep, int device = -1);
// the uncompressed long-range values at sample cells on the device (false: no device / error)
bool exact_long_values_device(int device, int n, const std::vector<double>& G,
                              const std::vector<double>& a_long, const std::vector<int32_t>& cells,
                              const std::vector<double>& z, const std::vector<int>& pts,
                              std::vector<double>& out);

// ---- device side -------------------------------------------------------------------------

struct DeviceTables {
  const double* F[3] = {nullptr, nullptr, nullptr};
  const double2* Fw[3] = {nullptr, nullptr, nullptr};  // rows padded/replicated to CHP chunks
  const float4* Fw32[3] = {nullptr, nullptr, nullptr}; // binary32 rows (A21), 16-byte quads
  const int2* nb_range = nullptr;     // per coarse cell: (list begin, count)
  const unsigned* nb_pack = nullptr;  // loc4 handles: begin | count << 24, z padded to nb_dim2p
  const double* S[3] = {nullptr, nullptr, nullptr};
  const int4* nb_ent = nullptr;       // per list entry: fine cell + sorted atom (packed), charge
  const double4* prec = nullptr;      // per sorted protein atom: (x, y, z, q)
  const double* short_memo = nullptr; // s(|D0|,|D1|,|D2|) for |D_a| <= n_sigma, or null
  const double* Ut[3] = {nullptr, nullptr, nullptr};  // Tucker bases n x r_l, row-major (N5)
  const double* TG = nullptr;         // Tucker core r0 x r1 x r2 (N5)
};

struct ScoreArgs {               // one launch of the scoring kernel
  int n, R, Rs, n_sigma;
  double b, inv_h, h, dcap2;
  int nb_shift, nb_lo[3], nb_dim[3];
  DeviceTables t;
  const double* zl;
  const double* yl;
  int64_t L;
  const double* poses;
  int64_t P;
  double* E;
  double* D;
  unsigned long long* invalid;   // may be null
  int* work;                     // this launch's zeroed work counter (dynamic pose chunks)
  double rmax_hint;              // ligand radius if known on the host (< 0: unknown)
  int64_t n_ent = 0, n_prot = 0;  // list entries and protein records (bounds for checked builds)
  unsigned vdw_cells2;           // keep a candidate for H6 iff |D|^2 < vdw_cells2 (conservative)
  float thr_a, thr_b;            // running H6 bound: |D|^2 < thr_a best + thr_b (AM-GM, rounded up)
  unsigned ns2;                  // n_sigma^2: H5 iff |D|^2 <= ns2
  int f32;                       // long-range part from the binary32 factors (A21)
  int tk = 0;                    // long-range part from the Tucker form (N5, reading A26)
  int tr[3] = {0, 0, 0};         // its ranks
  int loc4;                      // every list begin < 2^24 and count < 256: 4-byte local cells
  int nb_dim2p;                  // z extent of nb_pack (nb_dim[2] rounded up to a multiple of 4)
  // streamed launch (host-buffer pipeline): poses arrive in copy chunks [cb[i], cb[i+1]);
  // arrive[i] != 0 once chunk i landed; the kernel adds finished poses to done[i].  Null: off.
  const unsigned* arrive = nullptr;
  unsigned* done = nullptr;
  const long long* cb = nullptr;
  int n_cb = 0;
  unsigned* stall = nullptr;     // set to 1 if an arrival wait timed out
};

// Fill the dense short-range memo table s(d0,d1,d2), d_a = 0..n_sigma, with the O5 chain.
int launch_fill_short_memo(const double* S0, const double* S1, const double* S2, int Rs,
                           int n_sigma, double* out, void* stream);

constexpr int64_t kMaxPackedAtoms = (int64_t)1 << 19;   // sorted atom index: 19 bits of a list entry
constexpr int kWorkSlots = 64;   // work counters per handle, each reused behind its last launch
constexpr int kPackPad = 24;     // zero cells before each axis of the packed range table (TMA)

// Launch the fused scoring kernel (H1-H8).  Returns a cudaError_t as int.  *launches
// (if not null) is incremented by the number of kernels enqueued.
int launch_score(const ScoreArgs& a, void* stream, int device, int* launches);
// which variant launch_score would run for these arguments (no launch): a kPath* value, or a
// positive CUDA error code
constexpr int kPathWindow = 1, kPathL2 = 2, kPathL2Runtime = 3, kPathTucker = 4;
int plan_score(const ScoreArgs& a, int device);
const char* score_kernel_variant(int R);
// NEXT row N2: PPIEM scan kernels (scan_kernel.cu)
int launch_scan_init(const double* centre, const double* dirs, const double* quats, int m_P,
                     int m_L, double s_start, double* poses, double* s, int* status, int* slot,
                     void* st);
int launch_scan_update(const double* centre, const double* dirs, const double* quats, int m_P,
                       int m_L, const double* Dc, const double* Ec, double sigma, double dcap,
                       double tol, int first, double* E, double* s, int* status, int* slot,
                       double* poses_next, int* count, void* st);
int launch_scan_gather(int64_t P, const int* status, const int* slot, const double* Ec, double* E,
                       void* st);
// NEXT row N1: forces on the rigid ligand (force_kernel.cu), P x 9 outputs, device pointers.
int launch_forces(const ScoreArgs& a, double* out, void* stream, int device);
// Chunks (16 B) per row of the window copy of the factors for compiled width R (0: none), and
// the host packing of that copy (rows padded with zeros or replicated to CHP chunks).
int window_row_chunks(int R);
void pack_window_rows(const std::vector<double>& F, int n, int R, std::vector<double>& out);
// The same for the binary32 variant: rows of 16-byte quads of floats (0: width not compiled).
int window_row_chunks32(int R);
void pack_window_rows32(const std::vector<double>& F, int n, int R, std::vector<float>& out);

}  // namespace rs

struct rs_handle {
  rs_params prm;
  int n = 0;
  double b = 0, h = 0, inv_h = 0;
  rs::Quadrature quad;
  std::vector<int32_t> is_long;        // per quadrature term
  int R = 0, Rs = 0, n_sigma = 0, R_long_ref = 0;
  std::vector<double> F[3];            // n x R
  std::vector<double> S[3];            // (2 n_sigma + 1) x Rs
  int64_t M = 0;
  std::vector<double> xyz, z;          // protein
  std::vector<int32_t> cells;          // M x 3
  rs::CoarseGrid cg;
  rs::SetupReport rep;
  rs::TuckerRep tucker;                // S5-S6 Tucker form of the long-range part (N3)
  int box_lo[3] = {0, 0, 0}, box_hi[3] = {-1, -1, -1};   // N3 restriction box (hi < lo: none)
  double setup_seconds = 0;
  // device
  bool on_device = false;
  int device = 0;
  void* dmem[6] = {nullptr};           // F1..3, S1..3
  void* d_nb_ent = nullptr;
  int64_t n_ent = 0;                   // list entries uploaded (incl. padding)
  void* d_prec = nullptr;
  void* d_memo = nullptr;
  void* d_Ut[3] = {nullptr, nullptr, nullptr};   // RS_FLAG_TUCKER_EVAL: bases, row-major
  void* d_TG = nullptr;                          //                      core
  void* d_Fw[3] = {nullptr, nullptr, nullptr};
  void* d_Fw32[3] = {nullptr, nullptr, nullptr};
  bool f32 = false;
  bool loc4 = false;                   // cell ranges fit 24 + 8 bits (kernel's local range table)
  void* d_nb_range = nullptr;
  void* d_nb_pack = nullptr;           // loc4: packed ranges, the TMA source of the local table
  int nb_dim2p = 0;
  int* d_work = nullptr;               // kWorkSlots dynamic-schedule work counters
  void* work_ev[rs::kWorkSlots] = {};  // cudaEvent_t recorded behind each counter's last launch
  std::mutex work_mtx[rs::kWorkSlots];
  std::atomic<unsigned> work_slot{0};
  void* scan_buf = nullptr;            // rs_ppiem_scan scratch (grow-only)
  size_t scan_bytes = 0;
  int64_t device_bytes = 0;
  // staging for host-pointer calls
  std::mutex mtx;
  void* stage = nullptr;
  size_t stage_bytes = 0;
  void* streams[3] = {nullptr, nullptr, nullptr};
  unsigned* h_ones = nullptr;          // pinned 1s: arrival flags written by the copy stream
  // cached ligand radius for device-resident ligands (only steers the launch shape)
  const void* rmax_key = nullptr;
  int64_t rmax_L = -1;
  double rmax_val = -1;
};
