/*
 * rs_dock.h -- C ABI of the B200-native RS-tensor pose-rescoring library (librsdock.so).
 *
 * Path: batched rescoring of rigid ligand poses against a protein whose
 * free-space electrostatic potential is held in the range-separated (RS) canonical tensor
 * format of Benner, Khoromskij, Khoromskaia & Stein, arXiv 2510.26611 ("the paper",
 * PAPER.md):
 *   - rs_build_protein  = Algorithm TEP, once per protein, host C++;
 *   - rs_score_poses    = Algorithm PLIE with Lemma 3.2 / Eq. (18)
 *     (PAPER.md:864-891), the RS entry formula and the van der Waals
 *     constraint of Eq. (22), one fused sm_100a kernel;
 *   - rs_score_forces   = forces on the rigid ligand (§3.3 Eq. (21), §4 Eqs. (24)-(25));
 *   - rs_ppiem_scan     = Algorithm PPIEM steps A3-A6 on the device,
 *     with rs_landscape_minima (A6) on the host.
 *
 * Units: the library is unit-agnostic.  Lengths in the caller's unit (the tests and bench
 * use Angstrom), charges in e, energies in charge^2/length (x 0.529177210903 = hartree
 * when lengths are Angstrom).
 *
 * Conventions shared by every entry point:
 *   - All arrays are fp64, row-major, C-contiguous.  xyz arrays are N x 3.
 *   - Poses are P x 7: (w, x, y, z, tx, ty, tz) = quaternion (scalar first, need not be
 *     unit: it acts as its normalisation) and the translation of the ligand body frame.
 *     The ligand coordinates passed in are body-frame coordinates, i.e. the caller centres
 *     the ligand at its geometric centre (rotation about the centre,
 *     then translation of the centre), so an atom lands at x' = R(q) y + t.
 *   - The grid is Omega = [-b, b]^3 split into n^3 cells of width h = 2b/n (n even,
 *     PAPER.md:278-282).  A point is evaluated at its cell (piecewise-constant basis,
 *     PAPER.md:279-290); a point on a cell boundary belongs to the lower cell.
 *   - Ownership: every input is caller-owned and only read during the call.  The handle
 *     deep-copies what it needs and owns all device memory it allocates; rs_free releases
 *     it.  Outputs are written, never retained.
 *   - Errors: functions returning a pointer return NULL on error, functions returning an
 *     integer return a negative RS_E_* code; rs_last_error() gives a thread-local message.
 *     There is no CPU fallback: without a CUDA device rs_build_protein fails.
 *   - Thread safety: a handle is immutable after build.  rs_score_poses_async on one handle
 *     from several host threads / streams is safe.  rs_score_poses with host pointers
 *     serialises on a per-handle lock (it reuses the handle's staging buffers).
 */
#ifndef RS_DOCK_H
#define RS_DOCK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_E_INVALID_ARG (-1) /* a null pointer, a size < 0, a non-finite parameter ... */
#define RS_E_CUDA        (-2) /* a CUDA runtime error (message in rs_last_error)        */
#define RS_E_NOMEM       (-3) /* host or device allocation failed                        */
#define RS_E_NO_DEVICE   (-4) /* handle built with RS_FLAG_HOST_ONLY or no CUDA device     */

#define RS_FLAG_HOST_ONLY 1u  /* build the tables on the host only (no upload); for tests */
#define RS_FLAG_F32_FACTORS 2u /* score with the long-range factors rounded to binary32 (the
                                  north_star's fp32-factor variant, reading A21):
                                  half the gather bytes, products and rank sums in binary32,
                                  energies within 1e-6 of sum_l |z_l phi(x_l)| of the binary64
                                  path; needs a compiled width R in {4, 8, 12, 16, 24, 32} */

#define RS_FLAG_BOX_SCHEME_B 4u /* rs_restrict_box: scheme (B), a new RHOSVD + CP of the
                                  long-range sum restricted to the box,
                                  instead of scheme (C) from the kept Tucker form            */

#define RS_FLAG_DEVICE_FFT 8u  /* setup: the RHOSVD and core convolutions (S5-S6) with cuFFT on
                                  the device -- the default of every device build (kept as an
                                  explicit request); its tables differ from a host-only build's
                                  by rounding                                                */
#define RS_FLAG_TUCKER_EVAL 32u /* scoring evaluates the long range from the Tucker form of
                                  S5-S6 (RHOSVD bases U_l, core G) instead of the CP factors:
                                  NEXT row N5, r0 r1 r2 multiply-adds per atom instead of 3R
                                  products (reading A26); needs r_l <= 32 and a core
                                  of at most 16384 entries; not for combined/box handles       */
#define RS_FLAG_HOST_FFT 16u   /* setup: the S5-S6 convolutions on the host even with a device
                                  (tables bitwise equal to a RS_FLAG_HOST_ONLY build's)       */

typedef struct rs_handle rs_handle; /* opaque, immutable after build */

/* Build parameters.  Initialise with rs_params_default() and override fields. */
typedef struct {
    int32_t  grid_n;        /* n, cells per axis, even, >= 2                */
    int32_t  rank_R;        /* uploaded CP width R of the long-range part (Lemma 3.2's R;
                               BASELINE's "R_l").  0 = tolerance mode: R from eps_compress     */
    double   eps_compress;  /* relative tolerance of the Tucker (RHOSVD) and slice truncation  */
    double   eps_quad;      /* sinc-quadrature target max relative error of 1/r on
                               [h/4, 2 sqrt(3) b] (Eq. (2))                  */
    double   sigma_split;   /* sigma_s: range-split radius; n_sigma = ceil(sigma_s / h)
                               (TEP step 2 PAPER.md:1190-1193)               */
    double   eps_split;     /* Gaussian k is long-range iff sqrt(ln(1/eps_split))/t_k >= sigma_s */
    double   sigma_vdw;     /* vdW threshold: a pose clashes iff mindist < sigma_vdw (Eq. (22)) */
    double   dmin_cap;      /* D_cap >= sigma_vdw: mindist is reported exactly below D_cap,
                               +inf otherwise                                                   */
    int32_t  tucker_rank_max; /* cap on the Tucker ranks r_l, which follow eps_compress below it
                               (0 = automatic: at most rank_R + 8 when rank_R > 0).  A larger
                               cap keeps a richer Tucker form for rs_restrict_box              */
    int32_t  als_sweeps;    /* CP-ALS sweeps when R < the exact C2T2C rank (0 = default 300)    */
    int32_t  device;        /* CUDA device ordinal                                              */
    int32_t  n_threads;     /* host threads for the setup (0 = all)                             */
    uint64_t seed;          /* seed of the randomized range finder / ALS init                   */
    uint32_t flags;         /* RS_FLAG_*                                                        */
    double   nbr_cell;      /* edge [A] of the coarse cells of the neighbour lists used for the
                               short-range (H5) and vdW (H6) pairs; rounded to h * 2^k
                               (0 = automatic: about max(D_cap, n_sigma h) / 2)                 */
} rs_params;

/* Information about a built handle (all host values). */
typedef struct {
    int32_t  n;             /* grid cells per axis */
    double   b, h, inv_h;   /* half width, cell width 2b/n, n/(2b) */
    int32_t  R;             /* CP width of the uploaded long-range factors */
    int32_t  R_exact;       /* rank before CP-ALS (C2T2C rank of the Tucker core) */
    int32_t  tucker_r[3];   /* Tucker ranks of the RHOSVD step */
    int32_t  quad_K;        /* quadrature terms k = 0..K */
    double   quad_s, quad_Ls; /* sinc step s and scale L_s (t_k = sinh(k s)/L_s) */
    double   quad_err;      /* measured max relative error of the quadrature on its interval */
    int32_t  R_long_ref;    /* number of long-range reference terms (Eq. (4) R_l) */
    int32_t  R_short;       /* number of short-range reference terms R_s */
    int32_t  n_sigma;       /* short-range support radius in cells */
    int64_t  n_atoms;       /* protein atoms M */
    double   tucker_err;    /* estimated relative Frobenius error of the Tucker step */
    double   cp_core_err;   /* relative Frobenius error of the CP fit of the Tucker core */
    double   sampled_max_err;  /* max |P_l - CP| / max |P_l| over sampled exterior cells */
    double   sampled_rms_err;  /* rms of the same, relative to rms |P_l| */
    int32_t  n_err_samples;
    double   sigma_vdw, dmin_cap;
    int64_t  nbr_cells;     /* coarse cells of the neighbour (cell-list) structure */
    int64_t  nbr_entries;   /* total candidate entries */
    int32_t  nbr_shift;     /* coarse cell = 2^nbr_shift fine cells */
    int64_t  device_bytes;  /* bytes uploaded to the device */
    double   setup_seconds; /* wall time of the whole build */
    int32_t  on_device;     /* 1 when the tables are resident on a device */
    int32_t  factor_bits;   /* 64, or 32 with RS_FLAG_F32_FACTORS */
    int32_t  box_lo[3], box_hi[3]; /* rs_restrict_box cell box (hi < lo: the whole grid) */
} rs_info;

void rs_params_default(rs_params* p);

/*
 * Build the RS tensor of a protein (Algorithm TEP) and upload it once.
 *   q        : n_atoms charges z_m                         (host)
 *   xyz      : n_atoms x 3 positions x_m, inside [-b, b]^3 (host)
 *   box_half_width : b > 0
 *   params   : may be NULL (defaults)
 * Steps: S1 sinc quadrature of 1/r (Eq. (2)), S2 long/short split (Eq. (4)), S3 1D Galerkin
 * cell averages (Eq. (1)), S4 snapping of the atoms, S5 randomized RHOSVD of the implicit
 * side matrices of the rank-(M x R_l) long-range sum (Eq. (6)), S6 Tucker core, S7 core ->
 * CP of width R (exact canonical-Tucker-canonical when it fits, else CP-ALS), S8 short-range
 * reference rows (Def. 2.1), S9 cell lists for the short-range / vdW pass, S10 upload.
 * Returns NULL on error (invalid argument, more than 524,288 atoms (a neighbour-list entry holds
 * a 19-bit atom index), atom outside the box, odd n, sigma_split < h, sigma_vdw > dmin_cap, no
 * CUDA device unless RS_FLAG_HOST_ONLY, CUDA or allocation failure).
 */
rs_handle* rs_build_protein(const double* q, const double* xyz, int64_t n_atoms,
                            double box_half_width, const rs_params* params);

/*
 * Multi-protein complex (NEXT row N4; Eq. (23): the ligand's energy in
 * the field of several proteins is sum_l z_l (sum_p P_{M_p})(x_l); reading A24).
 *   parts   : n_parts >= 1 handles from rs_build_protein (host-only handles are fine), built
 *             with the same grid_n, box_half_width, eps_quad, sigma_split, eps_split,
 *             sigma_vdw and dmin_cap (so their short-range rows are identical)
 *   flags   : RS_FLAG_* of the new handle (device and the other parameters are part 0's)
 * The new handle's long-range factors are the parts' factors concatenated along the rank,
 * F_a = [F_a^(0) | F_a^(1) | ...] (n x sum_p R_p, no recompression; the O4 tree runs over the
 * concatenated width), its short-range part and vdW distance run over the union of the atoms
 * (part 0's atoms first), and its cell lists are rebuilt for the union.  The parts are not
 * modified and stay owned by the caller; the result is released with rs_free.  Returns NULL on
 * error (mismatched parts, width > 2^20, RS_FLAG_F32_FACTORS with an uncompiled width, no
 * CUDA device unless RS_FLAG_HOST_ONLY, allocation or upload failure).
 */
rs_handle* rs_combine_proteins(const rs_handle* const* parts, int32_t n_parts, int32_t flags);

/*
 * Box-restricted recompression (NEXT row N3; schemes (B)/(C), Table 1
 * the potential restricted to a ligand box Pi has CP rank R_Pi << R_Omega;
 * DESIGN.md reading A25).  Scheme (C), hybrid: the handle's Tucker form of the long-range part
 * (kept from the RHOSVD step S5-S6, factors U_l of n x r_l and core G) is restricted to the
 * cell box lo[l] <= i_l <= hi[l] (0 <= lo <= hi < n, per axis), re-orthonormalised there by an
 * SVD of the restricted rows, and its core recompressed to CP width rank (0: the smallest width
 * within the handle's eps_compress).  The new handle carries these factors in rows inside the
 * box and NaN in every other row, so a pose with a ligand atom outside the box gets E = NaN
 * (its minimum distance is still computed); the short-range part and the vdW distance are the
 * parent's, exactly.  Scoring, forces and scans run unchanged on it.
 *   h     : a handle from rs_build_protein (not from rs_combine_proteins: no Tucker form)
 *   lo, hi: 3 cell indices each (host)
 *   rank  : R_Pi >= 0;   flags: RS_FLAG_* of the new handle
 * With RS_FLAG_BOX_SCHEME_B in flags the box factors come from scheme (B) instead: the
 * randomized RHOSVD (S5) of the long-range sum restricted to the box rows (the side matrices
 * P_box A_l, the other modes' column norms over their box rows), its core (S6) and S7, from the
 * parent's atoms, quadrature and split; any handle with atoms (combined ones too) qualifies.
 * Returns NULL on error (bad box, no Tucker form, RS_FLAG_F32_FACTORS with an uncompiled width,
 * no device unless RS_FLAG_HOST_ONLY, allocation or upload failure).  Release with rs_free.
 */
rs_handle* rs_restrict_box(const rs_handle* h, const int32_t* lo, const int32_t* hi, int32_t rank,
                           int32_t flags);

/*
 * Score P poses of a rigid ligand (Algorithm PLIE + Eq. (22)), synchronously.
 *   q_lig (n_lig), xyz_lig (n_lig x 3) : ligand charges and body-frame coordinates
 *   poses (P x 7)                      : see conventions above
 *   energies_out (P)                   : E_p = sum_l z_l [ P^long_{M,R}(i_l)
 *                                         + sum_{m: |i_l - i_m|_2 <= n_sigma} z_m S(i_l - i_m) ]
 *   mindist_out (P)                    : min_{l,m} |x'_l - x_m| if < dmin_cap, else +inf
 * Pointers may be host (pageable or pinned) or device memory of the handle's device; each
 * is detected with cudaPointerGetAttributes.  Host data are copied in and out inside the
 * call, pipelined: with host poses and outputs and P >= 4e5 one kernel launch scores each
 * pose chunk as soon as its copy lands and each chunk's results are copied back as soon as
 * they are final; otherwise chunks are copied and launched in turn on three
 * streams.  The outputs never depend on the path.  A pose with a zero quaternion, a non-finite value, or any transformed atom outside
 * [-b, b]^3 is invalid: both outputs are NaN.
 * Returns the number of invalid poses (>= 0) or a negative RS_E_* code.
 */
int64_t rs_score_poses(rs_handle* h, const double* q_lig, const double* xyz_lig, int64_t n_lig,
                       const double* poses, int64_t P, double* energies_out, double* mindist_out);

/*
 * Asynchronous variant: all five arrays must be DEVICE memory; the work is enqueued on
 * `cuda_stream` (a cudaStream_t, NULL = legacy default stream) and the call returns at once.
 * If invalid_count_dev is not NULL, the number of invalid poses is written there (int64,
 * device memory) by the same stream.  Returns 0 or a negative RS_E_* code.
 */
int64_t rs_score_poses_async(rs_handle* h, const double* q_lig, const double* xyz_lig,
                             int64_t n_lig, const double* poses, int64_t P,
                             double* energies_out, double* mindist_out,
                             int64_t* invalid_count_dev, void* cuda_stream);

/*
 * Forces on the rigid ligand for P poses (NEXT row N1; §3.3 Eq. (21)
 * "differ_ligand" PAPER.md:1032-1036 and §4 Eqs. (24)-(25), Lemma 4.1 PAPER.md:1612-1640;
 * DESIGN.md reading A22).  Per ligand atom, the backward difference of the long-range CP value
 * on the grid g_a = (phi(i) - phi(i - e_a)) * n/(2b) (forward at i_a = 0) gives the force
 * F_l = -z_l g; per pose forces_out[9 p + 0..8] = (sum_l F_l, sum_l r_l x F_l,
 * sum_l (F_l . r_l / |r_l|^2) r_l) with r_l = x'_l - t: the net force, the torque about the
 * ligand centre t and Eq. (24)'s radial resultant F_0.  Long-range part only, binary64 factors.
 * All pointers are device pointers (P x 7 poses, P x 9 outputs); the work is enqueued on
 * cuda_stream (asynchronous).  Invalid poses (as rs_score_poses) get NaN and are counted in
 * *invalid_count_dev when it is not NULL (zeroed on the stream first).  Returns 0 or a negative
 * RS_E_* code.
 */
int64_t rs_score_forces(rs_handle* h, const double* q_lig, const double* xyz_lig, int64_t n_lig,
                        const double* poses, int64_t P, double* forces_out,
                        int64_t* invalid_count_dev, void* cuda_stream);

/*
 * Which variant of the fused scoring kernel rs_score_poses[_async] runs for this handle and a
 * ligand (host pointer, n_lig x 3 body-frame coordinates; only its radius matters), without
 * launching anything: RS_PATH_WINDOW (H4 rows staged in a shared-memory window per pose tile:
 * the roofline is shared-memory bandwidth), RS_PATH_L2 (rows gathered from L2 with 32-byte
 * loads: the window of one translation does not fit), RS_PATH_L2_RUNTIME (a width without a
 * compiled kernel, L2 rows) or RS_PATH_TUCKER (RS_FLAG_TUCKER_EVAL: the Tucker form).  The measurement (bench.py) picks its roofline from this.  Returns
 * the path (> 0) or a negative RS_E_* code.
 */
#define RS_PATH_WINDOW     1
#define RS_PATH_L2         2
#define RS_PATH_L2_RUNTIME 3
#define RS_PATH_TUCKER     4
int rs_score_path(rs_handle* h, const double* xyz_lig, int64_t n_lig);

/*
 * Handle cache (SPEC.md:207's kernel cache): rs_save_handle writes every host-side table of the
 * handle (parameters, quadrature, split, CP factors, short-range rows, protein atoms and cells,
 * cell lists, Tucker form, setup report) to one binary file with a 64-bit checksum;
 * rs_load_handle reads it back bit for bit and uploads it to `device` (< 0: the saved ordinal),
 * skipping the setup (S1-S9).  flags may hold RS_FLAG_HOST_ONLY.  The file is tied to this
 * library's layout of the rs_params struct; a mismatch is refused.  rs_save_handle returns 0
 * or a negative RS_E_* code; rs_load_handle returns NULL on error (rs_last_error()).
 */
int rs_save_handle(const rs_handle* h, const char* path);
rs_handle* rs_load_handle(const char* path, int32_t device, int32_t flags);

/*
 * Copy the handle's Tucker form of the long-range part (S5-S6; what RS_FLAG_TUCKER_EVAL scores
 * from) to caller buffers (host): r[3] the Tucker ranks; U0, U1, U2 n x r_l each (row-major:
 * row i holds U_l[i, :]); G r0 x r1 x r2 (row-major), charges and quadrature weights folded in.
 * Pass NULL buffers to query r only.  Returns 0 or a negative code (RS_E_INVALID_ARG when the
 * handle keeps no Tucker form, e.g. a combined handle).
 */
int rs_export_tucker(const rs_handle* h, int32_t* r, double* U0, double* U1, double* U2, double* G);

/* Fill *out.  Returns 0 or RS_E_INVALID_ARG. */
int rs_get_info(const rs_handle* h, rs_info* out);

/*
 * Copy the uploaded tables to caller buffers (host), for the oracle and tests:
 *   F1, F2, F3 : n x R each (long-range CP factors, weights folded into F1)
 *   S1, S2, S3 : (2 n_sigma + 1) x R_short each (short-range reference rows, a_k in S1)
 * Any pointer may be NULL to skip it.  Returns 0 or a negative code.
 */
int rs_export_tables(const rs_handle* h, double* F1, double* F2, double* F3, double* S1,
                     double* S2, double* S3);

/*
 * Quadrature and split of the handle: t (K+1), a (K+1), is_long (K+1, 1/0), and the
 * protein cells i_m (n_atoms x 3, int32) the handle snapped.  NULL skips an output.
 */
int rs_export_setup(const rs_handle* h, double* t, double* a, int32_t* is_long,
                    int32_t* protein_cells);

/*
 * PPIEM scan (NEXT row N2; Algorithm PPIEM steps A3-A6; DESIGN.md reading
 * A23).  For every position j (direction dirs[j], unit 3-vector) and ligand orientation k
 * (quats[k], w,x,y,z), the ligand centre starts at centre + s_start dirs[j] and approaches the
 * centre along the line (A3) by sphere tracing on the pose's minimum distance d (a step never
 * exceeds the clearance, so the first contact is never jumped over):
 *     d = +inf (no protein atom within D_cap):  s <- s - (D_cap - sigma_vdw)
 *     d - sigma_vdw <= tol:                      converged (vdW contact)
 *     otherwise:                                 s <- s - (d - sigma_vdw) * 0.999
 * (a later d below sigma_vdw can only come from rounding: contact); all poses advance
 * together, one batched scoring launch per iteration (at most max_iter).  Every dirs[j] must be
 * a unit vector to within 1e-9 (else RS_E_INVALID_ARG: a longer direction could step past the
 * clearance).
 * Outputs (host arrays, row j, column k, m_P x m_L): energy at the final position (A4-A5; NaN
 * unless status is 0 or 4), the final s and a status: 0 contact reached, 1 a ligand atom left
 * the box, 2 clash at s_start, 3 passed the centre without contact (s < 0), 4 max_iter reached
 * (feasible, not converged).  Needs dmin_cap > sigma_vdw (the build's D_cap is the step).
 * The ligand arrays may be host or device pointers.  Returns 0 or a negative RS_E_* code.
 */
int64_t rs_ppiem_scan(rs_handle* h, const double* q_lig, const double* xyz_lig, int64_t n_lig,
                      const double* centre, const double* dirs, int32_t m_P, const double* quats,
                      int32_t m_L, double s_start, double tol, int32_t max_iter,
                      double* energies_out, double* s_out, int32_t* status_out);

/*
 * Local minima of an m_P x m_L landscape (PPIEM step A6): entries strictly below all 8
 * neighbours on the grid periodic in both indices (plateaus: the lexicographically smallest
 * index), NaN entries excluded and never neighbours; sorted by energy, ties by (j, k).  Writes
 * up to top_k flat indices j m_L + k and returns their count (>= 0) or RS_E_INVALID_ARG.
 * Host-only.
 */
int32_t rs_landscape_minima(const double* energies, int32_t m_P, int32_t m_L, int32_t top_k,
                            int32_t* idx_out);

/* Message of the last error on this thread ("" if none). */
const char* rs_last_error(void);

/* Release the handle and its device memory.  NULL is a no-op. */
void rs_free(rs_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* RS_DOCK_H */
