/*
 * oracle_score.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, scalar CPU fp64 implementation of the per-pose quantity the CUDA path
 * computes.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load
 * it.  It shares no source with paper_2510_26611_b200/csrc (no common headers, helpers
 * or constants) and never links against the product library.
 *
 * Build (done by __graft_entry__.build()):
 *   gcc -O2 -ffp-contract=off -fno-tree-vectorize -fopenmp -shared -fPIC \
 *       -o oracle/liboracle.so oracle/oracle_score.c -lm
 * -ffp-contract=off: no implicit a*b+c contraction; every fused multiply-add below is
 * an explicit fma() call (correctly rounded), so each op sequence is exactly as written.
 *
 * What is computed, per pose p (paper notation: protein M = {x_m, z_m}, ligand
 * L = {y_l, z_l}):
 *   E_p = sum_l z_l * [ P^long_{M,R}(i_l) + sum_{m : |i_l - i_m|_2 <= n_sigma} z_m S(i_l - i_m) ]
 *     -- Lemma 3.2 / Eq. (18) gives the long-range sum, Algorithm PLIE
 *        steps 2-3 the <z_L, p_L> form; the RS entry formula of
 *        PAPER.md:460-466 (Def. 2.1) adds the short-range replicas.
 *   d_p = min_{l,m} |x'_l - x_m|  if below D_cap, else +inf
 *     -- the constraint dist(M, F(L)) >= sigma of Eq. (22).
 * The ligand atom positions are x'_l = R(q) y_l + t (F = R o T) and
 * i_l is the cell of x'_l on the piecewise-constant grid.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- O1: unit quaternion (w,x,y,z) -> rotation matrix, row-major R[3][3] ------------
 * Rotation of the ligand about its geometric centre, parametrised by
 * a quaternion (ledger A10).  s = 2/|q|^2 makes a non-unit q act as its normalisation.
 * Returns 0 (invalid pose) when |q|^2 is zero or not finite. */
int oracle_quat_to_rot(const double *q, double *R)
{
    double w = q[0], x = q[1], y = q[2], z = q[3];
    double nn = ((w * w + x * x) + y * y) + z * z;
    if (!(nn > 0.0) || !isfinite(nn)) return 0;
    double s = 2.0 / nn;
    double xs = x * s, ys = y * s, zs = z * s;
    double wx = w * xs, wy = w * ys, wz = w * zs;
    double xx = x * xs, xy = x * ys, xz = x * zs;
    double yy = y * ys, yz = y * zs, zz = z * zs;
    R[0] = 1.0 - (yy + zz); R[1] = xy - wz;          R[2] = xz + wy;
    R[3] = xy + wz;         R[4] = 1.0 - (xx + zz);  R[5] = yz - wx;
    R[6] = xz - wy;         R[7] = yz + wx;          R[8] = 1.0 - (xx + yy);
    return 1;
}

/* ---- O2: rigid transform x' = R y + t ---- */
void oracle_transform(const double *R, const double *y, const double *t, double *xp)
{
    for (int a = 0; a < 3; ++a)
        xp[a] = ((R[3 * a + 0] * y[0] + R[3 * a + 1] * y[1]) + R[3 * a + 2] * y[2]) + t[a];
}

/* ---- O3: snap a coordinate to its grid cell (ledger A3/A4) ----
 * Cells [-b + i h, -b + (i+1) h], i = 0..n-1, h = 2b/n.  u = (x + b) * inv_h with
 * inv_h = n / (2b); i = ceil(u) - 1 clamped to [0, n-1]: an exact cell boundary (u an
 * integer) goes to the lower cell ("ties toward the lower index").
 * Returns -1 when x is outside [-b, b] (or NaN). */
int oracle_snap(double x, double b, double inv_h, int n)
{
    if (!(x >= -b && x <= b)) return -1;
    double u = (x + b) * inv_h;
    double c = ceil(u) - 1.0;
    if (c < 0.0) c = 0.0;
    if (c > (double)(n - 1)) c = (double)(n - 1);
    return (int)c;
}

/* ---- O6: double-double accumulation of exact products (Dekker TwoProduct, Knuth TwoSum) */
typedef struct { double hi, lo; } dd_t;

static void dd_add_product(dd_t *acc, double a, double b)
{
    double p = a * b;
    double e = fma(a, b, -p);               /* a*b = p + e exactly */
    double s = acc->hi + p;                 /* TwoSum(hi, p) */
    double bb = s - acc->hi;
    double err = (acc->hi - (s - bb)) + (p - bb);
    acc->hi = s;
    acc->lo = acc->lo + (err + e);
}

/* exposed for the O6 pin (tests compare with an exact rational sum) */
double oracle_dd_sum_products(const double *a, const double *b, int64_t n)
{
    dd_t acc = {0.0, 0.0};
    for (int64_t i = 0; i < n; ++i) dd_add_product(&acc, a[i], b[i]);
    return acc.hi + acc.lo;
}

/* ---- O4: long-range CP value at cell i (Lemma 3.2 / Eq. (18); entry formula PAPER.md:463)
 * phi = sum_{k<R} F1[i0][k] F2[i1][k] F3[i2][k].  The paper fixes no summation order; the
 * contract (reading A20) is:
 *   q_k = (F1[i0][k] * F2[i1][k]) * F3[i2][k]      for k < R,   q_k = 0 for R <= k < 2C,
 *   C   = smallest power of two >= ceil(R/2)       (number of rank pairs "chunks"),
 *   s_c = q_{2c} + q_{2c+1}                        for c < C,
 *   for m = C/2, C/4, ..., 1:  s_c = s_c + s_{c+m}  for c < m,
 *   phi = s_0.
 * (A pairwise halving tree over rank pairs.) */
double oracle_long_value(const double *F1, const double *F2, const double *F3, int R,
                         int i0, int i1, int i2)
{
    const double *a = F1 + (int64_t)i0 * R, *b = F2 + (int64_t)i1 * R, *c = F3 + (int64_t)i2 * R;
    int C = 1;
    while (2 * C < R) C *= 2;
    double s[C];
    for (int j = 0; j < C; ++j) {
        double q0 = 0.0, q1 = 0.0;
        if (2 * j < R) q0 = (a[2 * j] * b[2 * j]) * c[2 * j];
        if (2 * j + 1 < R) q1 = (a[2 * j + 1] * b[2 * j + 1]) * c[2 * j + 1];
        s[j] = q0 + q1;
    }
    for (int m = C / 2; m >= 1; m /= 2)
        for (int j = 0; j < m; ++j) s[j] = s[j] + s[j + m];
    return s[0];
}

/* ---- O4-f32: the fp32-factor variant of O4 (north_star: "an fp32-factor variant"; DESIGN.md
 * reading A21).  Each factor entry is rounded to binary32, f = fl32(F); then, in binary32,
 *   q_k = (f1[i0][k] * f2[i1][k]) * f3[i2][k]      for k < R,   q_k = 0 for R <= k < 4 C4,
 *   C4  = smallest power of two >= ceil(R/4)       (number of rank quads),
 *   s_c = (q_4c + q_4c+1) + (q_4c+2 + q_4c+3)      for c < C4,
 *   for m = C4/2, ..., 1:  s_c = s_c + s_{c+m}      for c < m,
 *   phi = (double) s_0                              (exact widening).
 * The energy accumulation (O6) stays double-double in binary64. */
double oracle_long_value_f32(const double *F1, const double *F2, const double *F3, int R,
                             int i0, int i1, int i2)
{
    const double *a = F1 + (int64_t)i0 * R, *b = F2 + (int64_t)i1 * R, *c = F3 + (int64_t)i2 * R;
    int C = 1;
    while (4 * C < R) C *= 2;
    float s[C];
    for (int j = 0; j < C; ++j) {
        float q[4];
        for (int t = 0; t < 4; ++t) {
            int k = 4 * j + t;
            q[t] = 0.0f;
            if (k < R) {
                float fa = (float)a[k], fb = (float)b[k], fc = (float)c[k];
                q[t] = (fa * fb) * fc;
            }
        }
        s[j] = (q[0] + q[1]) + (q[2] + q[3]);
    }
    for (int m = C / 2; m >= 1; m /= 2)
        for (int j = 0; j < m; ++j) s[j] = s[j] + s[j + m];
    return (double)s[0];
}

/* ---- O4-T: the long-range value from the Tucker form (NEXT row N5, "Tucker-format
 * evaluation"; the Tucker rank bound PAPER.md:472-484; reading A26).  With the rows
 * u_l = U_l[i_l, :] (U_l: n x r_l, row-major) of the RHOSVD bases and the core G (r0 x r1 x r2,
 * row-major, charges and quadrature weights folded in):
 *   v_ab = sum_c G[a][b][c] * u2[c]          (ascending c, each product rounded, then added)
 *   t_a  = sum_b u1[b] * v_ab                (ascending b)
 *   phi  = sum_a u0[a] * t_a                 (ascending a)
 * each chain starting from +0, no fused multiply-add. */
double oracle_tucker_value(const double *U0, const double *U1, const double *U2, int r0, int r1,
                           int r2, const double *G, int i0, int i1, int i2)
{
    const double *u0 = U0 + (int64_t)i0 * r0, *u1 = U1 + (int64_t)i1 * r1, *u2 = U2 + (int64_t)i2 * r2;
    double phi = 0.0;
    for (int a = 0; a < r0; ++a) {
        double t = 0.0;
        for (int b = 0; b < r1; ++b) {
            const double *g = G + ((int64_t)a * r1 + b) * r2;
            double v = 0.0;
            for (int c = 0; c < r2; ++c) v = v + g[c] * u2[c];
            t = t + u1[b] * v;
        }
        phi = phi + u0[a] * t;
    }
    return phi;
}

/* Tucker tables for mode bit 2 of oracle_score_poses (set before the call; test
 * infrastructure, one scoring call at a time) */
static const double *g_tU[3], *g_tG;
static int g_tr[3];
void oracle_set_tucker(const double *U0, const double *U1, const double *U2, int r0, int r1, int r2,
                       const double *G)
{
    g_tU[0] = U0; g_tU[1] = U1; g_tU[2] = U2;
    g_tr[0] = r0; g_tr[1] = r1; g_tr[2] = r2;
    g_tG = G;
}

/* ---- O5: short-range reference value S(Delta) for |Delta|_2 <= n_sigma (Def. 2.1) ---- */
double oracle_short_value(const double *S1, const double *S2, const double *S3, int Rs,
                          int n_sigma, int d0, int d1, int d2)
{
    const double *a = S1 + (int64_t)(d0 + n_sigma) * Rs;
    const double *b = S2 + (int64_t)(d1 + n_sigma) * Rs;
    const double *c = S3 + (int64_t)(d2 + n_sigma) * Rs;
    double s = 0.0;
    for (int k = 0; k < Rs; ++k) s = s + (a[k] * b[k]) * c[k];
    return s;
}

/*
 * Score P poses.  All arrays host, row-major, fp64 unless stated:
 *   F1,F2,F3 : n x R long-range CP factors (weights folded), exported by the library
 *   S1,S2,S3 : (2 n_sigma + 1) x Rs short-range reference rows (a_k folded into S1)
 *   X (M x 3), zM (M)      : protein atoms (continuous coordinates) and charges
 *   Y (L x 3), zL (L)      : ligand body coordinates (centred) and charges
 *   poses (P x 7)          : w,x,y,z,tx,ty,tz
 *   mode                   : bit 0 = long_only: skip O5 and O7 (Lemma 3.2's cost alone; the CPU
 *                            like-for-like rate); bit 1 = fp32 factors (O4-f32 instead of O4);
 *                            bit 2 = Tucker form (O4-T instead of O4; oracle_set_tucker first)
 * Outputs E (P), dmin (P).  Returns the number of invalid poses (O8: NaN outputs).
 * asum (P, may be NULL): sum over the pose's addends of |addend| (the M8 report's condition
 * number kappa = asum / |E|); NaN for invalid poses.  Report only: E never
 * reads it.
 * Protein cells are recomputed here with oracle_snap (never taken from the library).
 */
int64_t oracle_score_poses(int n, double b, int R, const double *F1, const double *F2,
                           const double *F3, int n_sigma, int Rs, const double *S1,
                           const double *S2, const double *S3, int64_t M, const double *X,
                           const double *zM, int64_t L, const double *Y, const double *zL,
                           int64_t P, const double *poses, double dcap, int mode,
                           double *E, double *dmin, double *asum)
{
    int long_only = mode & 1, f32 = (mode >> 1) & 1, tucker = (mode >> 2) & 1;
    double inv_h = (double)n / (2.0 * b);
    int *iM = (int *)malloc(sizeof(int) * 3 * (size_t)(M > 0 ? M : 1));
    for (int64_t m = 0; m < M; ++m)
        for (int a = 0; a < 3; ++a) iM[3 * m + a] = oracle_snap(X[3 * m + a], b, inv_h, n);
    double dcap2 = dcap * dcap;
    int64_t ns2 = (int64_t)n_sigma * n_sigma;
    int64_t invalid = 0;

#pragma omp parallel for schedule(dynamic, 4) reduction(+ : invalid)
    for (int64_t p = 0; p < P; ++p) {
        const double *pq = poses + 7 * p;
        double Rm[9];
        int ok = oracle_quat_to_rot(pq, Rm);
        dd_t acc = {0.0, 0.0};
        double best = INFINITY, abs_sum = 0.0;
        for (int64_t l = 0; l < L && ok; ++l) {
            double xp[3];
            int il[3];
            oracle_transform(Rm, Y + 3 * l, pq + 4, xp);
            for (int a = 0; a < 3; ++a) {
                il[a] = oracle_snap(xp[a], b, inv_h, n);
                if (il[a] < 0) ok = 0;
            }
            if (!ok) break;
            /* O4 */
            double phi = tucker ? oracle_tucker_value(g_tU[0], g_tU[1], g_tU[2], g_tr[0], g_tr[1],
                                                      g_tr[2], g_tG, il[0], il[1], il[2])
                         : f32 ? oracle_long_value_f32(F1, F2, F3, R, il[0], il[1], il[2])
                               : oracle_long_value(F1, F2, F3, R, il[0], il[1], il[2]);
            dd_add_product(&acc, zL[l], phi);
            abs_sum += fabs(zL[l] * phi);
            if (long_only) continue;
            for (int64_t m = 0; m < M; ++m) {
                /* O7: distance between continuous coordinates */
                double dx0 = xp[0] - X[3 * m + 0];
                double dx1 = xp[1] - X[3 * m + 1];
                double dx2 = xp[2] - X[3 * m + 2];
                double d2 = (dx0 * dx0 + dx1 * dx1) + dx2 * dx2;
                if (d2 < best) best = d2;
                /* O5: short-range replica of protein atom m contains cell i_l */
                int64_t e0 = il[0] - iM[3 * m + 0];
                int64_t e1 = il[1] - iM[3 * m + 1];
                int64_t e2 = il[2] - iM[3 * m + 2];
                if (e0 * e0 + e1 * e1 + e2 * e2 <= ns2) {
                    double s = oracle_short_value(S1, S2, S3, Rs, n_sigma, (int)e0, (int)e1,
                                                  (int)e2);
                    double w = zM[m] * s;
                    dd_add_product(&acc, zL[l], w);
                    abs_sum += fabs(zL[l] * w);
                }
            }
        }
        if (!ok) {
            E[p] = NAN;
            dmin[p] = NAN;
            invalid += 1;
        } else {
            E[p] = acc.hi + acc.lo;
            dmin[p] = (best < dcap2) ? sqrt(best) : INFINITY;
        }
        if (asum) asum[p] = ok ? abs_sum : NAN;
    }
    free(iM);
    return invalid;
}

/*
 * ---- N1: forces on the rigid ligand (NEXT row N1; reading A22) --------------------
 * PAPER.md §3.3: the force on ligand atom l is minus the gradient of the binding energy, taken
 * by one-dimensional finite differences of the long-range CP value on the grid (Eq. (21),
 * "differ_ligand", backward differences); §4 (Eqs. (24)-(25),
 * PAPER.md:1612-1627, Lemma 4.1) sums the atom forces into the resultants on
 * the rigid ligand.  Per ligand atom (cells i from O1-O3, phi from O4):
 *   g_a   = (phi(i) - phi(i - e_a)) * inv_h     (at i_a = 0: (phi(i + e_a) - phi(i)) * inv_h)
 *   F_l   = -(z_l * g)                          (force = minus the energy gradient)
 *   r_l   = x'_l - t                            (from the ligand's geometric centre)
 *   tau_l = (r1 F2 - r2 F1, r2 F0 - r0 F2, r0 F1 - r1 F0)
 *   rad_l = c r_l,  c = ((F0 r0 + F1 r1) + F2 r2) / ((r0 r0 + r1 r1) + r2 r2)   (0 if r_l = 0)
 * and per pose the double-double sums over atoms (O6) of F_l (the net force), tau_l (the torque
 * about t) and rad_l (Eq. (24)'s F_0(x_0), the sum of the radial projections):
 *   out[9 p + 0..2] = F, out[9 p + 3..5] = tau, out[9 p + 6..8] = F_0.  NaN for invalid poses.
 * Every product is rounded as written; no contraction.
 */
int64_t oracle_score_forces(int n, double b, int R, const double *F1, const double *F2,
                            const double *F3, int64_t L, const double *Y, const double *zL,
                            int64_t P, const double *poses, double *out)
{
    double inv_h = (double)n / (2.0 * b);
    int64_t invalid = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : invalid)
    for (int64_t p = 0; p < P; ++p) {
        const double *pq = poses + 7 * p;
        double Rm[9];
        int ok = oracle_quat_to_rot(pq, Rm);
        dd_t acc[9];
        for (int j = 0; j < 9; ++j) { acc[j].hi = 0.0; acc[j].lo = 0.0; }
        for (int64_t l = 0; l < L && ok; ++l) {
            double xp[3];
            int il[3];
            oracle_transform(Rm, Y + 3 * l, pq + 4, xp);
            for (int a = 0; a < 3; ++a) {
                il[a] = oracle_snap(xp[a], b, inv_h, n);
                if (il[a] < 0) ok = 0;
            }
            if (!ok) break;
            double phi = oracle_long_value(F1, F2, F3, R, il[0], il[1], il[2]);
            double g[3], Fl[3], r[3], tau[3], rad[3];
            for (int a = 0; a < 3; ++a) {
                int jm[3] = {il[0], il[1], il[2]};
                if (il[a] > 0) {
                    jm[a] = il[a] - 1;
                    g[a] = (phi - oracle_long_value(F1, F2, F3, R, jm[0], jm[1], jm[2])) * inv_h;
                } else {
                    jm[a] = il[a] + 1;
                    g[a] = (oracle_long_value(F1, F2, F3, R, jm[0], jm[1], jm[2]) - phi) * inv_h;
                }
                Fl[a] = -(zL[l] * g[a]);
                r[a] = xp[a] - pq[4 + a];
            }
            tau[0] = r[1] * Fl[2] - r[2] * Fl[1];
            tau[1] = r[2] * Fl[0] - r[0] * Fl[2];
            tau[2] = r[0] * Fl[1] - r[1] * Fl[0];
            double rr = (r[0] * r[0] + r[1] * r[1]) + r[2] * r[2];
            double c = 0.0;
            if (rr > 0.0) c = ((Fl[0] * r[0] + Fl[1] * r[1]) + Fl[2] * r[2]) / rr;
            for (int a = 0; a < 3; ++a) rad[a] = c * r[a];
            for (int a = 0; a < 3; ++a) {
                dd_add_product(&acc[a], 1.0, Fl[a]);
                dd_add_product(&acc[3 + a], 1.0, tau[a]);
                dd_add_product(&acc[6 + a], 1.0, rad[a]);
            }
        }
        for (int j = 0; j < 9; ++j) out[9 * p + j] = ok ? acc[j].hi + acc[j].lo : NAN;
        if (!ok) invalid += 1;
    }
    return invalid;
}

/* number of OpenMP threads the scorer uses (reported as cpu_baseline.cores) */
int oracle_num_threads(void)
{
    int nt = 1;
#ifdef _OPENMP
#pragma omp parallel
    {
#pragma omp single
        nt = omp_get_num_threads();
    }
#endif
    return nt;
}
