"""RS-tensor docking oracle -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU fp64 implementations of everything the CUDA path
computes, written from PAPER.md (arXiv 2510.26611).  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / `--impl reference` legs may import this module.  It shares
no code with paper_2510_26611_b200/ and never imports it (the library's exported tables
arrive as plain numpy arrays, O11).

Contents (each function cites the passage it follows):
  * grid + snapping                        -- PAPER.md:278-290, ledger A3/A4  (O3)
  * sinc quadrature of 1/r                 -- Eq. (2), ledger A6  (S1)
  * long/short split                       -- Eq. (4), ledger A7  (S2)
  * Galerkin cell averages of Gaussians    -- Eq. (1), ledger A5  (S3)
  * uncompressed RS kernel K_RS(Delta) and the uncompressed long-range CP factors of the
    protein (shift-and-windowing, Eq. (5)-(6) PAPER.md:371-401)
  * brute-force Coulomb binding energy     -- Eq. (13)
  * cell average of the Newton kernel K_h  -- Eq. (1) with p = 1/r
  * ctypes wrappers around oracle_score.c  -- O1-O8 (per-pose energy + min distance)
  * compression-error certificates         -- TEP step 4 PAPER.md:1184-1209, SPEC.md:80:
    dense CP, Gram-identity norms/inner products, unfolding tails, dense HOSVD, dense CP-ALS

Parity status: every function here is pinned by tests/test_oracle_pins.py against closed
forms, library routines (scipy quad / Rotation / cdist, fractions) or brute force.
"""
from __future__ import annotations

import ctypes
import math
import os
from fractions import Fraction

import numpy as np
from scipy import special

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def lib():
    """Load oracle/liboracle.so (built by __graft_entry__.build())."""
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        dp = ctypes.POINTER(ctypes.c_double)
        L.oracle_quat_to_rot.argtypes = [dp, dp]
        L.oracle_quat_to_rot.restype = ctypes.c_int
        L.oracle_transform.argtypes = [dp, dp, dp, dp]
        L.oracle_snap.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int]
        L.oracle_snap.restype = ctypes.c_int
        L.oracle_dd_sum_products.argtypes = [dp, dp, ctypes.c_int64]
        L.oracle_dd_sum_products.restype = ctypes.c_double
        L.oracle_long_value.argtypes = [dp, dp, dp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_int]
        L.oracle_long_value.restype = ctypes.c_double
        L.oracle_long_value_f32.argtypes = L.oracle_long_value.argtypes
        L.oracle_long_value_f32.restype = ctypes.c_double
        L.oracle_score_poses.argtypes = [
            ctypes.c_int, ctypes.c_double, ctypes.c_int, dp, dp, dp, ctypes.c_int, ctypes.c_int,
            dp, dp, dp, ctypes.c_int64, dp, dp, ctypes.c_int64, dp, dp, ctypes.c_int64, dp,
            ctypes.c_double, ctypes.c_int, dp, dp, dp]
        L.oracle_score_poses.restype = ctypes.c_int64
        L.oracle_tucker_value.argtypes = [dp, dp, dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, dp,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.oracle_tucker_value.restype = ctypes.c_double
        L.oracle_set_tucker.argtypes = [dp, dp, dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, dp]
        L.oracle_num_threads.restype = ctypes.c_int
        L.oracle_score_forces.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, dp, dp, dp,
                                          ctypes.c_int64, dp, dp, ctypes.c_int64, dp, dp]
        L.oracle_score_forces.restype = ctypes.c_int64
        _LIB = L
    return _LIB


def build():
    """Compile oracle_score.c (plain scalar C, no FP contraction)."""
    import subprocess
    src = os.path.join(_HERE, "oracle_score.c")
    out = os.path.join(_HERE, "liboracle.so")
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-tree-vectorize", "-fopenmp",
                           "-shared", "-fPIC", "-o", out, src, "-lm"])


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ------------------------------------------------------------------------------------------
# O1-O3 (thin wrappers over the C definitions, used by the pins)
# ------------------------------------------------------------------------------------------

def quat_to_rot(q):
    """O1: 3x3 rotation of quaternion q = (w,x,y,z), or None if |q|^2 == 0."""
    q = _c(q)
    R = np.empty(9)
    ok = lib().oracle_quat_to_rot(_p(q), _p(R))
    return R.reshape(3, 3) if ok else None


def transform(R, y, t):
    """O2: x' = R y + t."""
    R, y, t = _c(R).ravel(), _c(y), _c(t)
    out = np.empty(3)
    lib().oracle_transform(_p(R), _p(y), _p(t), _p(out))
    return out


def snap(x, b, n):
    """O3: cell index of coordinate x on the n-cell grid of [-b, b] (-1 outside)."""
    inv_h = float(n) / (2.0 * b)
    return lib().oracle_snap(float(x), float(b), inv_h, int(n))


def snap_np(x, b, n):
    """O3 vectorised in numpy with the identical op sequence (u = (x+b)*inv_h, ceil-1, clamp)."""
    x = np.asarray(x, dtype=np.float64)
    inv_h = float(n) / (2.0 * b)
    u = (x + b) * inv_h
    i = np.clip(np.ceil(u) - 1.0, 0, n - 1).astype(np.int64)
    i[~((x >= -b) & (x <= b))] = -1
    return i


def dd_sum_products(a, b):
    """O6: double-double sum of exact products a_i*b_i."""
    a, b = _c(a), _c(b)
    return lib().oracle_dd_sum_products(_p(a), _p(b), a.size)


def exact_sum_products(a, b):
    """Exact rational value of sum a_i b_i (the thing O6 approximates), rounded once."""
    s = Fraction(0)
    for x, y in zip(np.asarray(a, float), np.asarray(b, float)):
        s += Fraction(float(x)) * Fraction(float(y))
    return float(s)


# ------------------------------------------------------------------------------------------
# S1: sinc quadrature of the Newton kernel (Eq. (2); ledger A6)
# ------------------------------------------------------------------------------------------

def quadrature(s, K, Ls):
    """Nodes t_k and weights a_k, k = 0..K, with 1/r ~ sum_k a_k exp(-t_k^2 r^2).

    1/r = (2/sqrt(pi)) int_0^inf exp(-r^2 t^2) dt; substitute t = sinh(u)/Ls,
    apply the trapezoid (sinc) rule with step s on the whole real u-axis and fold the
    symmetric terms k and -k together:
        t_0 = 0,                a_0 = s / (sqrt(pi) Ls)
        t_k = sinh(k s)/Ls,     a_k = 2 s cosh(k s) / (sqrt(pi) Ls),   k = 1..K.
    """
    k = np.arange(K + 1, dtype=np.float64)
    t = np.sinh(k * s) / Ls
    a = 2.0 * s * np.cosh(k * s) / (math.sqrt(math.pi) * Ls)
    a[0] = s / (math.sqrt(math.pi) * Ls)
    t[0] = 0.0
    return t, a


def quadrature_rel_error(t, a, rmin, rmax, npts=4000):
    r = np.geomspace(rmin, rmax, npts)
    with np.errstate(over="ignore", invalid="ignore"):
        approx = (a[None, :] * np.exp(-(t[None, :] ** 2) * (r[:, None] ** 2))).sum(axis=1)
    err = np.abs(approx * r - 1.0)
    return float(np.max(np.where(np.isfinite(err), err, np.inf)))


def choose_quadrature(eps, rmin, rmax, Ls):
    """Smallest-K rule (s on a grid) meeting eps on [rmin, rmax] -- the oracle's own search."""
    best = None
    for s in np.arange(0.05, 1.2, 0.01):
        lo, hi = 1, 400
        if quadrature_rel_error(*quadrature(s, hi, Ls), rmin, rmax, 800) > eps:
            continue
        while lo < hi:
            mid = (lo + hi) // 2
            if quadrature_rel_error(*quadrature(s, mid, Ls), rmin, rmax, 800) <= eps:
                hi = mid
            else:
                lo = mid + 1
        if best is None or lo < best[1]:
            best = (float(s), lo)
    return best


# ------------------------------------------------------------------------------------------
# S2: long/short split (Eq. (4); TEP step 2 PAPER.md:1190-1193; ledger A7)
# ------------------------------------------------------------------------------------------

def split_long(t, sigma_s, eps_split):
    """Term k is long-range iff its effective support radius sqrt(ln(1/eps))/t_k >= sigma_s
    (t_0 = 0 has infinite support and is always long)."""
    t = np.asarray(t, dtype=np.float64)
    with np.errstate(divide="ignore"):
        r = np.where(t > 0, math.sqrt(math.log(1.0 / eps_split)) / np.where(t > 0, t, 1.0), np.inf)
    return r >= sigma_s


# ------------------------------------------------------------------------------------------
# S3: 1D Galerkin cell averages (Eq. (1); normalised per ledger A5)
# ------------------------------------------------------------------------------------------

def cell_average(t, h, d):
    """g[d] = (1/h) int_{(d-1/2)h}^{(d+1/2)h} exp(-t^2 x^2) dx  (g = 1 for t = 0).

    Closed form (sqrt(pi)/(2 t h)) (erf(t(d+1/2)h) - erf(t(d-1/2)h)); for cells away from the
    origin the erf difference is rewritten as an erfc difference so it does not cancel,
    and the function is evaluated at |d| so g[-d] == g[d] bitwise.
    """
    d = np.abs(np.asarray(d, dtype=np.float64))
    if t == 0.0:
        return np.ones_like(d)
    lo = t * (d - 0.5) * h
    hi = t * (d + 0.5) * h
    c = math.sqrt(math.pi) / (2.0 * t * h)
    inner = d < 0.5            # the cell containing the origin: integrand symmetric
    out = np.empty_like(d)
    out[inner] = c * 2.0 * special.erf(hi[inner])
    out[~inner] = c * (special.erfc(lo[~inner]) - special.erfc(hi[~inner]))
    return out


def reference_factors(t, h, dmax):
    """Rows d = -dmax..dmax of the 1D reference factors g_k[d] (one column per term)."""
    d = np.arange(-dmax, dmax + 1)
    return np.stack([cell_average(float(tk), h, d) for tk in t], axis=1)


# ------------------------------------------------------------------------------------------
# uncompressed RS kernel and protein potential (Def. 2.1; Eq. (5)-(6))
# ------------------------------------------------------------------------------------------

def K_RS(delta, t, a, long_mask, h, n_sigma):
    """Uncompressed RS kernel value at integer offset Delta:
    sum_{k long} a_k prod_a g_k[Delta_a]  +  [|Delta|_2 <= n_sigma] sum_{k short} a_k prod_a g_k[Delta_a]."""
    delta = np.asarray(delta, dtype=np.int64)
    val = 0.0
    inball = int((delta ** 2).sum()) <= n_sigma * n_sigma
    for k in range(len(t)):
        if not long_mask[k] and not inball:
            continue
        g = cell_average(float(t[k]), h, delta.astype(np.float64))
        val += a[k] * g[0] * g[1] * g[2]
    return val


def uncompressed_long_factors(iM, zM, t, a, long_mask, n, h):
    """Exact long-range CP factors of the protein potential (Eq. (6)):
    column (m, k) of mode l is g_k[i - i_{m,l}] for i = 0..n-1 (shift-and-windowing onto the
    n-grid), and the weight z_m a_k is folded into mode 1.  Rank M * R_l^ref."""
    ks = np.nonzero(long_mask)[0]
    d = np.arange(-(n - 1), n)
    G = np.stack([cell_average(float(t[k]), h, d) for k in ks], axis=1)  # (2n-1, RL)
    M = iM.shape[0]
    F = []
    rows = np.arange(n)
    for ax in range(3):
        Fa = np.empty((n, M * len(ks)))
        for m in range(M):
            off = rows - iM[m, ax] + (n - 1)
            blk = G[off, :]
            if ax == 0:
                blk = blk * (zM[m] * a[ks])[None, :]
            Fa[:, m * len(ks):(m + 1) * len(ks)] = blk
        F.append(np.ascontiguousarray(Fa))
    return F


def short_tables(t, a, long_mask, h, n_sigma):
    """Short-range reference rows S_a[Delta + n_sigma][k], Delta in [-n_sigma, n_sigma],
    k over the short terms, with a_k folded into S_1 (Def. 2.1, A_0)."""
    ks = np.nonzero(~np.asarray(long_mask))[0]
    d = np.arange(-n_sigma, n_sigma + 1)
    if len(ks) == 0:
        z = np.zeros((2 * n_sigma + 1, 0))
        return z, z.copy(), z.copy()
    G = np.stack([cell_average(float(t[k]), h, d) for k in ks], axis=1)
    return np.ascontiguousarray(G * a[ks][None, :]), G.copy(), G.copy()


# ------------------------------------------------------------------------------------------
# Eq. (13): brute-force Coulomb binding energy, and the cell-averaged Newton kernel
# ------------------------------------------------------------------------------------------

def coulomb_binding(X, qM, Y, zL):
    """E(M,L) = sum_m sum_l z_m z_l / |x_m - x_l| (Eq. (13)), math.fsum."""
    X, Y = np.asarray(X, float), np.asarray(Y, float)
    r = np.sqrt(((X[:, None, :] - Y[None, :, :]) ** 2).sum(axis=2))
    return math.fsum((np.asarray(qM)[:, None] * np.asarray(zL)[None, :] / r).ravel())


def coulomb_scale(X, qM, Y, zL):
    """S = sum |z_m z_l| / r_ml, the absolute Coulomb scale used to normalise chain errors."""
    r = np.sqrt(((np.asarray(X)[:, None, :] - np.asarray(Y)[None, :, :]) ** 2).sum(axis=2))
    return float((np.abs(np.asarray(qM))[:, None] * np.abs(np.asarray(zL))[None, :] / r).sum())


K_H0 = 3.0 * math.log(2.0 + math.sqrt(3.0)) - math.pi / 2.0   # h * K_h(0), cube self-average


def K_h(delta, h, order=12):
    """Cell average of 1/|x| over the cell at integer offset Delta (Eq. (1) with p = 1/r,
    normalised): closed form (3 ln(2+sqrt 3) - pi/2)/h at Delta = 0, tensor Gauss-Legendre
    cubature elsewhere (integrand smooth for |Delta|_inf >= 1)."""
    delta = np.asarray(delta, dtype=np.float64)
    if not np.any(delta):
        return K_H0 / h
    xg, wg = np.polynomial.legendre.leggauss(order)
    xg = 0.5 * xg
    wg = 0.5 * wg
    c = [(delta[a] + xg) * h for a in range(3)]
    X0, X1, X2 = np.meshgrid(c[0], c[1], c[2], indexing="ij")
    W = wg[:, None, None] * wg[None, :, None] * wg[None, None, :]
    return float((W / np.sqrt(X0 ** 2 + X1 ** 2 + X2 ** 2)).sum())


# ------------------------------------------------------------------------------------------
# O1-O8 scorer (C) wrapper
# ------------------------------------------------------------------------------------------

def tucker_value(tk: dict, i0, i1, i2) -> float:
    """O4-T at one cell: the long-range value from the Tucker form tk = (U0, U1, U2: n x r_l
    row-major, G: r0 x r1 x r2), the contraction order of oracle_tucker_value (reading A26)."""
    U = [_c(tk[k]) for k in ("U0", "U1", "U2")]
    G = _c(tk["G"])
    r = [u.shape[1] for u in U]
    return lib().oracle_tucker_value(_p(U[0]), _p(U[1]), _p(U[2]), r[0], r[1], r[2], _p(G),
                                     int(i0), int(i1), int(i2))


def score_poses(tables: dict, X, qM, Y, zL, poses, dcap, long_only=False, f32=False,
                abs_sum=False, tucker=None):
    """Per-pose (E, dmin, n_invalid) from exported tables (f32: the O4-f32 long-range part).
    abs_sum: also return sum_addends |addend| per pose (E, dmin, n_invalid, asum), the M8
    report's kappa = asum / |E|.

    tables: n, b, R, F1, F2, F3 (n x R), n_sigma, Rs, S1, S2, S3 ((2 n_sigma+1) x Rs)."""
    n, b = int(tables["n"]), float(tables["b"])
    F1, F2, F3 = (_c(tables[k]) for k in ("F1", "F2", "F3"))
    R = F1.shape[1] if F1.ndim == 2 else int(tables["R"])
    S1, S2, S3 = (_c(tables[k]) for k in ("S1", "S2", "S3"))
    ns = int(tables["n_sigma"])
    Rs = S1.shape[1] if S1.ndim == 2 and S1.size else 0
    X, qM, Y, zL, poses = _c(X), _c(qM), _c(Y), _c(zL), _c(poses)
    P = poses.shape[0]
    E = np.empty(P)
    d = np.empty(P)
    dummy = np.zeros(1)
    asum = np.empty(P) if abs_sum else None
    mode = (1 if long_only else 0) | (2 if f32 else 0)
    if tucker is not None:
        # O4-T (N5): the long range from the Tucker form instead of the CP factors
        U = [_c(tucker[k]) for k in ("U0", "U1", "U2")]
        G = _c(tucker["G"])
        lib().oracle_set_tucker(_p(U[0]), _p(U[1]), _p(U[2]), U[0].shape[1], U[1].shape[1],
                                U[2].shape[1], _p(G))
        mode |= 4
    inv = lib().oracle_score_poses(
        n, b, R, _p(F1), _p(F2), _p(F3), ns, Rs, _p(S1 if S1.size else dummy),
        _p(S2 if S2.size else dummy), _p(S3 if S3.size else dummy), X.shape[0], _p(X), _p(qM),
        Y.shape[0], _p(Y), _p(zL), P, _p(poses), float(dcap), mode, _p(E), _p(d),
        _p(asum) if abs_sum else None)
    if abs_sum:
        return E, d, int(inv), asum
    return E, d, int(inv)


def combine_tables(parts: list) -> dict:
    """Eq. (23) on one grid, reading A24: sum_p P_{M_p} is a CP tensor
    whose terms are all the parts' terms, i.e. the factors concatenated along the rank axis
    (part 0's columns first).  The short-range rows are a property of the shared grid and
    split, so the parts must agree on them."""
    t0 = parts[0]
    for t in parts[1:]:
        assert int(t["n"]) == int(t0["n"]) and float(t["b"]) == float(t0["b"])
        assert int(t["n_sigma"]) == int(t0["n_sigma"])
        for k in ("S1", "S2", "S3"):
            assert np.array_equal(t[k], t0[k])
    out = dict(t0)
    for k in ("F1", "F2", "F3"):
        out[k] = np.concatenate([np.asarray(t[k]).reshape(int(t0["n"]), -1) for t in parts],
                                axis=1)
    out["R"] = out["F1"].shape[1]
    return out


def score_complex(parts: list, proteins: list, Y, zL, poses, dcap):
    """Eq. (23) literally: E = sum_l z_l sum_p P_{M_p}(x_l) = sum_p E_p, each part scored on
    its own tables and atoms; the vdW distance of the complex is the minimum over the parts.
    proteins: list of (X_p, q_p).  Returns (E, dmin, n_invalid)."""
    E = None
    d = None
    inv = 0
    for tb, (X, q) in zip(parts, proteins):
        Ep, dp, inv = score_poses(tb, X, q, Y, zL, poses, dcap)
        E = Ep if E is None else E + Ep
        d = dp if d is None else np.fmin(d, dp)
    if E is not None:
        d = np.where(np.isnan(E), np.nan, d)
    return E, d, inv


def score_forces(tables: dict, Y, zL, poses):
    """Per-pose (P x 9: net force, torque about t, Eq. (24) radial resultant; n_invalid)."""
    n, b = int(tables["n"]), float(tables["b"])
    F1, F2, F3 = (_c(tables[k]) for k in ("F1", "F2", "F3"))
    R = F1.shape[1]
    Y, zL, poses = _c(Y), _c(zL), _c(poses)
    P = poses.shape[0]
    out = np.empty((P, 9))
    inv = lib().oracle_score_forces(n, b, R, _p(F1), _p(F2), _p(F3), Y.shape[0], _p(Y), _p(zL), P,
                                    _p(poses), _p(out))
    return out, int(inv)


def num_threads():
    return int(lib().oracle_num_threads())


# ------------------------------------------------------------------------------------------
# Compression-error certificates for TEP step 4 (the rank bound
# PAPER.md:472-484; SPEC.md:77-80 frobenius_norm by the Gram identity).  A CP tensor is a
# triple (F1, F2, F3) of n x K side matrices (weights folded in), T = sum_k F1_k o F2_k o F3_k.
# ------------------------------------------------------------------------------------------

def cp_dense(F1, F2, F3):
    """The dense n1 x n2 x n3 tensor sum_k F1[:, k] o F2[:, k] o F3[:, k], one mode-3 slice at a
    time: T[:, :, l] = (F1 * F3[l]) F2^T."""
    F1, F2, F3 = _c(F1), _c(F2), _c(F3)
    T = np.empty((F1.shape[0], F2.shape[0], F3.shape[0]))
    for l in range(F3.shape[0]):
        T[:, :, l] = (F1 * F3[l][None, :]) @ F2.T
    return T


def cp_inner(A, B, block=2048):
    """<A, B> of two CP tensors on one grid by the Gram identity:
    sum_{k, k'} prod_a (A_a^T B_a)[k, k'], never forming the dense tensors (blocks of A's
    columns), summed with math.fsum over the blocks."""
    K = A[0].shape[1]
    parts = []
    for s in range(0, K, block):
        e = min(K, s + block)
        G = np.ones((e - s, B[0].shape[1]))
        for a in range(3):
            G *= A[a][:, s:e].T @ B[a]
        parts.append(float(G.sum()))
    return math.fsum(parts)


def cp_norm2(F, block=2048):
    """||T||_F^2 of a CP tensor by the Gram identity, symmetric in (k, k'): the diagonal
    column blocks once, the blocks above it twice."""
    K = F[0].shape[1]
    parts = []
    for s in range(0, K, block):
        e = min(K, s + block)
        G = np.ones((e - s, K - s))
        for a in range(3):
            G *= F[a][:, s:e].T @ F[a][:, s:]
        parts.append(float(G[:, :e - s].sum()) + 2.0 * float(G[:, e - s:].sum()))
    return math.fsum(parts)


def certified_rel_error(F_exact, F_approx):
    """||T - T~||_F / ||T||_F from the factors only: ||T||^2 + ||T~||^2 - 2 <T, T~> (SPEC.md:80,
    certification of the compression error)."""
    n2 = cp_norm2(F_exact)
    d2 = n2 + cp_norm2(F_approx) - 2.0 * cp_inner(F_exact, F_approx)
    return math.sqrt(max(d2, 0.0) / n2)


def unfolding_tails(F, R):
    """Per mode a: the sum of the squared singular values of the mode-a unfolding T_(a) beyond
    the R largest, from T_(a) T_(a)^T = F_a (o_{b != a} F_b^T F_b) F_a^T (Hadamard product of
    the other modes' Grams).  Any approximation of multilinear rank <= R in mode a (every CP
    tensor of width R) is at least sqrt(tail_a) away from T (Eckart-Young on the unfolding)."""
    Gs = [F[a].T @ F[a] for a in range(3)]
    tails = []
    for a in range(3):
        H = np.ones_like(Gs[0])
        for b in range(3):
            if b != a:
                H *= Gs[b]
        lam = np.linalg.eigvalsh(F[a] @ H @ F[a].T)[::-1]
        tails.append(float(np.clip(lam[R:], 0.0, None).sum()))
    return tails


def hosvd_dense(T, R):
    """Truncated HOSVD of a dense tensor (De Lathauwer et al.): U_a = the R dominant left
    singular vectors of the mode-a unfolding, core = T x_1 U_1^T x_2 U_2^T x_3 U_3^T.  Returns
    (U1, U2, U3, core, relative error) with error^2 = ||T||^2 - ||core||^2 (orthogonal
    projection).  Quasi-optimal: its error is at most sqrt(3) x the best Tucker(R) error."""
    U = []
    for a in range(3):
        Ta = np.moveaxis(T, a, 0).reshape(T.shape[a], -1)
        w, V = np.linalg.eigh(Ta @ Ta.T)
        U.append(V[:, ::-1][:, :R])
    core = np.einsum("ijl,ia,jb,lc->abc", T, U[0], U[1], U[2], optimize=True)
    n2 = float(np.sum(T * T))
    return U[0], U[1], U[2], core, math.sqrt(max(n2 - float(np.sum(core * core)), 0.0) / n2)


def cp_als_dense(T, R, iters=100, init=None, seed=0):
    """CP-ALS on a dense tensor (Carroll-Chang / Harshman; Kolda-Bader Alg. 1): each sweep
    solves the three linear least-squares problems F_a = T_(a) KR(others) (o_{b != a} G_b)^+
    in turn.  init: three n x R starting matrices (default: seeded normal).  Returns
    (F1, F2, F3, relative Frobenius error)."""
    rng = np.random.default_rng(seed)
    F = [np.array(f, dtype=np.float64) for f in init] if init is not None else \
        [rng.normal(size=(T.shape[a], R)) for a in range(3)]
    subs = ["ijl,jr,lr->ir", "ijl,ir,lr->jr", "ijl,ir,jr->lr"]
    for _ in range(iters):
        for a in range(3):
            o = [b for b in range(3) if b != a]
            mttkrp = np.einsum(subs[a], T, F[o[0]], F[o[1]], optimize=True)
            V = (F[o[0]].T @ F[o[0]]) * (F[o[1]].T @ F[o[1]])
            F[a] = mttkrp @ np.linalg.pinv(V)
    D = T - cp_dense(*F)
    return F[0], F[1], F[2], math.sqrt(float(np.sum(D * D)) / float(np.sum(T * T)))
