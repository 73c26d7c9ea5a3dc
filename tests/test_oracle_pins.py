"""Pins for the oracle (oracle/): each test ties an oracle function to something other than
itself -- a closed form, a worked example from the paper/SPEC, a library routine (scipy),
exact rational arithmetic, or brute force -- chosen so a dropped term, wrong sign/index or
transposed operand fails.  CPU only (-m "not gpu")."""
import math
import os
from fractions import Fraction

import numpy as np
import pytest
from scipy import integrate
from scipy.spatial.distance import cdist
from scipy.spatial.transform import Rotation

from synth import configs as syn

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    vals = {}
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                k, v = line.split()
                vals[k] = float(v)
    return vals


# ---------------------------------------------------------------------------------- S1
@pytest.mark.parametrize("b,n,eps", [(20.0, 256, 1e-4), (20.0, 256, 1e-6), (64.0, 4096, 1e-6)])
def test_quadrature_approximates_newton_kernel(oracle, b, n, eps):
    """Eq. (2): sum_k a_k exp(-t_k^2 r^2) ~ 1/r on [h/2, 2 sqrt3 b] within eps (relative),
    checked on points the search never saw (random r, not the search's log grid)."""
    h = 2 * b / n
    Ls = 2 * math.sqrt(3) * b
    s, K = oracle.choose_quadrature(eps, h / 2, Ls, Ls)
    t, a = oracle.quadrature(s, K, Ls)
    r = np.exp(np.random.default_rng(0).uniform(math.log(h / 2), math.log(Ls), 20000))
    approx = (a[None, :] * np.exp(-(t[None, :] ** 2) * r[:, None] ** 2)).sum(axis=1)
    assert np.max(np.abs(approx * r - 1)) <= 1.5 * eps
    # the Laplace-Gauss integral itself by adaptive quadrature, one r
    r0 = 1.7
    val, _ = integrate.quad(lambda tt: math.exp(-r0 * r0 * tt * tt), 0, np.inf)
    assert abs(2 / math.sqrt(math.pi) * val - 1 / r0) < 1e-12
    # weights positive, nodes ascending, t_0 = 0 (constant term)
    assert np.all(a > 0) and np.all(np.diff(t) > 0) and t[0] == 0.0


def test_quadrature_table2_rank_trend(oracle):
    """Table 2: the reference CP rank grows slowly with n (20 -> 32 for
    n = 128 -> 16384).  Our rule at eps=1e-4 on the paper-like box grows monotonically and
    stays within the same order."""
    ranks = []
    for n in (128, 1024, 16384):
        b = 20.0
        Ls = 2 * math.sqrt(3) * b
        s, K = oracle.choose_quadrature(1e-4, (2 * b / n) / 2, Ls, Ls)
        ranks.append(2 * K + 1)
    assert ranks[0] <= ranks[1] <= ranks[2]
    assert 15 <= ranks[0] and ranks[2] <= 80


# ---------------------------------------------------------------------------------- S2
def test_split_monotone_and_partition(oracle):
    t, a = oracle.quadrature(0.32, 30, 69.28)
    m2 = oracle.split_long(t, 2.0, 1e-6)
    m4 = oracle.split_long(t, 4.0, 1e-6)
    assert m2[0] and m4[0]                       # constant term always long
    assert np.all(m2[m4])                        # raising sigma never moves short -> long
    # long terms are wide: exp(-t^2 sigma^2) >= eps at sigma; short terms are narrow
    assert np.all(np.exp(-(t[m2] * 2.0) ** 2) >= 1e-6 * (1 - 1e-12))
    assert np.all(np.exp(-(t[~m2] * 2.0) ** 2) < 1e-6)


# ---------------------------------------------------------------------------------- S3
def test_cell_average_closed_form(oracle):
    g = _golden("closed_forms.txt")
    val = oracle.cell_average(1.0, 1.0, np.array([0.0]))[0]
    assert abs(val - g["gauss_cell_t1_h1"]) < 1e-15


def test_cell_average_vs_adaptive_quadrature(oracle):
    rng = np.random.default_rng(3)
    for _ in range(60):
        t = float(np.exp(rng.uniform(-4, 3)))
        h = float(np.exp(rng.uniform(-4, 0)))
        d = int(rng.integers(-40, 41))
        lo, hi = (d - 0.5) * h, (d + 0.5) * h
        ref, _ = integrate.quad(lambda x: math.exp(-t * t * x * x), lo, hi, epsabs=0,
                                epsrel=2e-14, limit=200)
        ref /= h
        val = oracle.cell_average(t, h, np.array([float(d)]))[0]
        if ref > 1e-280:
            assert abs(val - ref) <= 1e-12 * ref, (t, h, d, val, ref)
    assert oracle.cell_average(0.0, 0.3, np.array([0.0, 7.0])).tolist() == [1.0, 1.0]


def test_cell_average_even_bitwise(oracle):
    d = np.arange(-300, 301, dtype=np.float64)
    for t in (0.05, 0.7, 3.0, 20.0):
        g = oracle.cell_average(t, 0.03125, d)
        assert np.array_equal(g, g[::-1])


# ---------------------------------------------------------------------------------- O3
def test_snap_spec_examples(oracle):
    with open(os.path.join(GOLD, "spec_snap.txt")) as f:
        rows = [l.split() for l in f if l.strip() and not l.startswith("#")]
    for r in rows:
        b, n = float(r[0]), int(r[1])
        xyz = [float(v) for v in r[2:5]]
        want = [int(v) for v in r[5:8]]
        got = [oracle.snap(x, b, n) for x in xyz]
        assert got == want, (r, got)


def test_snap_ties_go_low_and_cells_contain_point(oracle):
    b, n = 2.0, 64                        # h = 1/16 exactly representable
    h = 2 * b / n
    for j in range(n + 1):
        x = -b + j * h                    # an exact cell boundary
        assert oracle.snap(x, b, n) == max(j - 1, 0)
    rng = np.random.default_rng(0)
    x = rng.uniform(-b, b, 5000)
    i = oracle.snap_np(x, b, n)
    assert np.all((-b + i * h <= x) & (x <= -b + (i + 1) * h))
    assert oracle.snap(b + 1e-12, b, n) == -1 and oracle.snap(float("nan"), b, n) == -1
    assert [oracle.snap(v, b, n) for v in x[:200]] == i[:200].tolist()


# ---------------------------------------------------------------------------------- O1/O2
def test_quaternion_rotation_vs_scipy(oracle):
    rng = np.random.default_rng(1)
    q = syn.shoemake_quaternions(rng, 2000)
    ref = Rotation.from_quat(q[:, [1, 2, 3, 0]]).as_matrix()     # scipy is scalar-last
    for k in range(q.shape[0]):
        R = oracle.quat_to_rot(q[k])
        assert np.max(np.abs(R - ref[k])) < 2e-15
        assert np.array_equal(R, oracle.quat_to_rot(-q[k]))       # R(q) = R(-q) bitwise
        assert np.max(np.abs(R - oracle.quat_to_rot(3.0 * q[k]))) < 1e-15   # implicit norm
    assert np.array_equal(oracle.quat_to_rot([1, 0, 0, 0]), np.eye(3))
    assert np.array_equal(oracle.quat_to_rot([0, 1, 0, 0]), np.diag([1.0, -1, -1]))
    assert np.array_equal(oracle.quat_to_rot([0, 0, 0, 1]), np.diag([-1.0, -1, 1]))
    assert oracle.quat_to_rot([0, 0, 0, 0]) is None


def test_transform_identity_bitwise_and_isometry(oracle):
    rng = np.random.default_rng(2)
    Y = rng.normal(size=(30, 3)) * 3
    I = oracle.quat_to_rot([1, 0, 0, 0])
    for y in Y:
        assert np.array_equal(oracle.transform(I, y, np.zeros(3)), y)
    R = oracle.quat_to_rot(syn.shoemake_quaternions(rng, 1)[0])
    t = rng.normal(size=3) * 10
    Xp = np.stack([oracle.transform(R, y, t) for y in Y])
    assert np.max(np.abs(cdist(Xp, Xp) - cdist(Y, Y))) < 1e-12
    assert np.max(np.abs(Xp - (Y @ R.T + t))) < 1e-13


# ---------------------------------------------------------------------------------- O6
def test_dd_sum_matches_exact_rational(oracle):
    rng = np.random.default_rng(4)
    exact_hits, n_cases = 0, 300
    for c in range(n_cases):
        n = int(rng.integers(1, 200))
        a = rng.normal(size=n) * np.exp(rng.uniform(-20, 20, n))
        b = rng.normal(size=n)
        if c % 2:     # adversarial: heavy cancellation
            b[n // 2:] = -b[: n - n // 2] * (a[: n - n // 2] / a[n // 2:])[: n - n // 2]
        got = oracle.dd_sum_products(a, b)
        ex = oracle.exact_sum_products(a, b)
        if got == ex:
            exact_hits += (c % 2 == 0)
        else:
            # double-double bound: one final rounding + n * 2^-104 * sum |a_i b_i|
            bound = np.spacing(abs(ex)) + n * 2.0 ** -104 * float(np.sum(np.abs(a * b)))
            assert abs(got - ex) <= bound, (got, ex, bound)
    assert exact_hits >= (n_cases // 2) * 0.98   # well-conditioned sums: correctly rounded


# ---------------------------------------------------------------------------------- O4
def _tables(F, S=None, n_sigma=0, n=None, b=1.0):
    F1, F2, F3 = F
    if S is None:
        S = (np.zeros((2 * n_sigma + 1, 1)),) * 3
    return dict(n=n if n is not None else F1.shape[0], b=b, R=F1.shape[1], F1=F1, F2=F2, F3=F3,
                n_sigma=n_sigma, S1=S[0], S2=S[1], S3=S[2])


def test_long_value_rank1_ones_and_one_hot(oracle):
    n = 8
    ones = np.ones((n, 1))
    assert oracle.lib().oracle_long_value(*(oracle._p(np.ascontiguousarray(ones)),) * 3, 1, 3, 4, 5) == 1.0
    # rank-2, e1 x e1 x e1 (xi=3) and e2 x e2 x e2 (xi=5)
    F = np.zeros((n, 2))
    F[0, 0] = 1
    F[1, 1] = 1
    F1 = F * np.array([3.0, 5.0])
    lv = lambda i: oracle.lib().oracle_long_value(oracle._p(np.ascontiguousarray(F1)),
                                                  oracle._p(F), oracle._p(F), 2, i, i, i)
    assert lv(0) == 3.0 and lv(1) == 5.0 and lv(2) == 0.0


def _lv(oracle, F1, F2, F3, i=(0, 0, 0)):
    c = lambda x: oracle._p(np.ascontiguousarray(x, dtype=np.float64))
    return oracle.lib().oracle_long_value(c(F1), c(F2), c(F3), F1.shape[1], *i)


def test_long_value_summation_order_worked_example(oracle):
    """O4 order contract (reading A20), worked by hand with q = (1e16, 1, 2, -1e16, 3)
    (R = 5, so C = 4 rank pairs, the last two padded with zeros):
      s = (1e16 + 1, 2 - 1e16, 3 + 0, 0) = (1e16, -1e16 + 2, 3, 0)      [1e16 + 1 ties to even]
      m = 2: s0 = 1e16 + 3 = 1e16 + 4 (tie to even), s1 = -1e16 + 2
      m = 1: phi = (1e16 + 4) + (-1e16 + 2) = 6.
    The exact sum is 7 and the ascending sequential chain gives 5, so this pins the tree."""
    q = np.array([[1e16, 1.0, 2.0, -1e16, 3.0]])
    ones = np.ones_like(q)
    assert _lv(oracle, q, ones, ones) == 6.0
    # R = 4 (C = 2): (1e16 + 1) + (-1e16 + 1) = 1e16 - 1e16 = 0, sequential would give 1
    q4 = np.array([[1e16, 1.0, -1e16, 1.0]])
    assert _lv(oracle, q4, np.ones_like(q4), np.ones_like(q4)) == 0.0
    # the triple product is rounded as (F1 F2) F3: 3 * (1/3) * 3 with 1/3 rounded
    t = np.array([[1.0 / 3.0]])
    assert _lv(oracle, np.array([[3.0]]), t, np.array([[3.0]])) == (3.0 * (1.0 / 3.0)) * 3.0


@pytest.mark.parametrize("R", [4, 8, 12, 16, 24, 32])
def test_long_value_cyclic_pair_rotation_invariance(oracle, R):
    """The halving tree is invariant, bitwise, under any cyclic rotation of the C rank pairs
    (pair c is combined with c + C/2 first, i.e. c XOR C/2, which commutes with rotation mod C);
    the kernel relies on this to read chunks in a lane-rotated order.  Also within the
    classical bound |phi - exact| <= gamma_{log2(C) + 3} sum |a b c|."""
    rng = np.random.default_rng(R)
    C = 1
    while 2 * C < R:
        C *= 2
    for trial in range(50):
        F = [rng.normal(size=(1, 2 * C)) * np.exp(rng.normal(0, 3, size=(1, 2 * C))) for _ in range(3)]
        for f in F:
            f[:, R:] = 0.0
        base = _lv(oracle, *[f[:, :R] for f in F])
        for rot in range(1, C):
            perm = np.concatenate([np.arange(2 * ((c + rot) % C), 2 * ((c + rot) % C) + 2) for c in range(C)])
            Fr = [f[:, perm] for f in F]        # width 2C: the padding zeros move with their pair
            assert _lv(oracle, *Fr) == base
        ex = sum(Fraction(float(F[0][0, k])) * Fraction(float(F[1][0, k])) * Fraction(float(F[2][0, k]))
                 for k in range(R))
        mag = float(np.sum(np.abs(F[0][0, :R] * F[1][0, :R] * F[2][0, :R])))
        k = int(np.log2(C)) + 3
        u = 2.0 ** -53
        assert abs(float(Fraction(base) - ex)) <= k * u / (1 - k * u) * mag * (1 + 1e-12)


def test_scorer_long_range_equals_dense_materialisation(oracle):
    """O2-O4+O6 vs numpy: dense tensor T = einsum(F1,F2,F3) indexed at the snapped cells of
    the transformed atoms, summed with weights z (SPEC.md:67 dense materialisation, n<=16)."""
    rng = np.random.default_rng(5)
    n, b, R = 16, 4.0, 5
    F = [rng.normal(size=(n, R)) for _ in range(3)]
    T = np.einsum("ik,jk,lk->ijl", *F)
    Y = rng.normal(size=(6, 3))
    Y -= Y.mean(0)
    z = rng.uniform(-1, 1, 6)
    poses = np.concatenate([syn.shoemake_quaternions(rng, 40), rng.uniform(-1, 1, (40, 3))], 1)
    E, d, inv = oracle.score_poses(_tables(F, b=b), np.zeros((0, 3)), np.zeros(0), Y, z, poses,
                                   1.0, long_only=True)
    assert inv == 0
    for p in range(40):
        R_ = Rotation.from_quat(poses[p, [1, 2, 3, 0]]).as_matrix()
        Xp = Y @ R_.T + poses[p, 4:]
        idx = oracle.snap_np(Xp, b, n)
        ref = math.fsum(z[l] * T[tuple(idx[l])] for l in range(6))
        assert abs(E[p] - ref) <= 1e-13 * (np.abs(z) @ np.abs(T[tuple(idx.T)]) + 1e-300)
    # bitwise linearity in the ligand charges (power-of-two scaling; north_star invariant)
    E2, _, _ = oracle.score_poses(_tables(F, b=b), np.zeros((0, 3)), np.zeros(0), Y, 4.0 * z,
                                  poses, 1.0, long_only=True)
    assert np.array_equal(E2, 4.0 * E)
    # M8's addend magnitude sum: sum_l |z_l T[i_l]| from the same dense tensor, so kappa >= 1
    _, _, _, asum = oracle.score_poses(_tables(F, b=b), np.zeros((0, 3)), np.zeros(0), Y, z,
                                       poses, 1.0, long_only=True, abs_sum=True)
    for p in range(40):
        R_ = Rotation.from_quat(poses[p, [1, 2, 3, 0]]).as_matrix()
        idx = oracle.snap_np(Y @ R_.T + poses[p, 4:], b, n)
        ref = math.fsum(abs(z[l] * T[tuple(idx[l])]) for l in range(6))
        assert abs(asum[p] - ref) <= 1e-13 * ref and asum[p] >= abs(E[p]) * (1 - 1e-15)


# ---------------------------------------------------------------------------------- O7/O8
def test_scorer_min_distance_vs_cdist_and_invalid(oracle):
    rng = np.random.default_rng(6)
    n, b = 32, 8.0
    F = [np.zeros((n, 1))] * 3
    X = rng.uniform(-3, 3, (40, 3))
    q = rng.uniform(-1, 1, 40)
    Y = rng.normal(size=(5, 3))
    Y -= Y.mean(0)
    z = rng.uniform(-1, 1, 5)
    P = 200
    poses = np.concatenate([syn.shoemake_quaternions(rng, P), rng.uniform(-5, 5, (P, 3))], 1)
    poses[7, :4] = 0.0                       # zero quaternion -> invalid
    poses[9, 4] = 7.9                        # atoms leave the box -> invalid
    cap = 2.5
    E, d, inv = oracle.score_poses(_tables(F, b=b), X, q, Y, z, poses, cap)
    for p in range(P):
        if p in (7, 9):
            assert math.isnan(E[p]) and math.isnan(d[p])
            continue
        R_ = Rotation.from_quat(poses[p, [1, 2, 3, 0]]).as_matrix()
        m = cdist(Y @ R_.T + poses[p, 4:], X).min()
        if m < cap - 1e-12:
            assert abs(d[p] - m) < 1e-13
        elif m > cap + 1e-12:
            assert d[p] == np.inf
    assert inv == 2


def test_vdw_threshold_boundary(oracle):
    """SPEC.md:480-481 / Eq. (22) 'dist >= sigma': exactly sigma is feasible, sigma - 1e-9 is a
    clash.  Distances reported exactly below the cap."""
    F = [np.zeros((16, 1))] * 3
    X = np.array([[0.0, 0.0, 0.0]])
    Y = np.array([[0.0, 0.0, 0.0]])
    for dist, clash in ((2.5, False), (2.5 - 1e-9, True)):
        poses = np.array([[1.0, 0, 0, 0, dist, 0, 0]])
        E, d, inv = oracle.score_poses(_tables(F, b=4.0), X, np.ones(1), Y, np.ones(1), poses, 3.0)
        assert d[0] == dist and (d[0] < 2.5) == clash


# ---------------------------------------------------------------------------------- physics chain
def _newton_self_cell_numeric():
    """h*K_h(0) = (1/h^2) int_cube 1/|x| = 0.75 * int_{[-1,1]^2} (1+u^2+v^2)^(-1/2) du dv
    (six pyramids, one per face, each rescaled to the reference face)."""
    I, _ = integrate.dblquad(lambda v, u: 1.0 / math.sqrt(1 + u * u + v * v), -1, 1, -1, 1,
                             epsabs=1e-14, epsrel=2e-14)
    return 0.75 * I


def test_newton_self_cell_closed_form(oracle):
    g = _golden("closed_forms.txt")
    assert abs(oracle.K_H0 - g["newton_self_cell"]) < 1e-12
    assert abs(_newton_self_cell_numeric() - oracle.K_H0) < 1e-12


def test_K_h_cubature_vs_point_kernel(oracle):
    # far cells: cell average -> 1/r with an O(h^2/r^2) midpoint correction
    h = 0.1
    for dl in [(5, 0, 0), (3, 4, 1), (10, 2, 7)]:
        r = h * math.sqrt(sum(v * v for v in dl))
        kh = oracle.K_h(dl, h)
        assert abs(kh * r - 1) < 0.01 * (h / r) ** 2 * 10
    # adjacent cell vs scipy tplquad
    ref, _ = integrate.tplquad(lambda z, y, x: 1 / math.sqrt(x * x + y * y + z * z),
                               0.5, 1.5, -0.5, 0.5, -0.5, 0.5, epsabs=1e-12, epsrel=1e-12)
    assert abs(oracle.K_h((1, 0, 0), 1.0, order=24) - ref) < 1e-10


def _rs_setup(oracle, b, n, eps_q, sigma_s, eps_split=1e-6):
    h = 2 * b / n
    Ls = 2 * math.sqrt(3) * b
    s, K = oracle.choose_quadrature(eps_q, h / 4, Ls, Ls)
    t, a = oracle.quadrature(s, K, Ls)
    lm = oracle.split_long(t, sigma_s, eps_split)
    n_sigma = int(math.ceil(sigma_s / h))
    return h, t, a, lm, n_sigma


def test_K_RS_vs_cell_averaged_newton_kernel(oracle):
    """SURVEY §8(c) C2 vs C1: |K_RS - K_h| / K_h <= ~eps_q off the singular cell; the singular
    cell against the closed form with a looser bound (quadrature weakest there)."""
    b, n = 8.0, 128
    h, t, a, lm, ns = _rs_setup(oracle, b, n, 1e-8, 1.0)
    for dl in [(1, 0, 0), (2, 1, 0), (5, 3, 1), (16, 0, 0), (30, 20, 10)]:
        krs = oracle.K_RS(dl, t, a, lm, h, ns)
        kh = oracle.K_h(dl, h, order=16)
        assert abs(krs - kh) / kh < 2e-7, dl
    k0 = oracle.K_RS((0, 0, 0), t, a, lm, h, ns)
    assert abs(k0 - oracle.K_H0 / h) / (oracle.K_H0 / h) < 1e-2
    # the short part vanishes outside the ball, so K_RS there equals the long-range part
    dl = (ns + 1, 0, 0)
    long_only = sum(a[k] * np.prod(oracle.cell_average(float(t[k]), h, np.array(dl, float)))
                    for k in range(len(t)) if lm[k])
    assert oracle.K_RS(dl, t, a, lm, h, ns) == pytest.approx(long_only, rel=1e-15)


def _chain_case(oracle, seed=0):
    rng = np.random.default_rng(seed)
    b, n = 10.0, 128
    h, t, a, lm, ns = _rs_setup(oracle, b, n, 1e-8, 1.0)
    X = syn.packed_ball(rng, 30, 4.0, 1.2)
    qM = rng.uniform(-1, 1, 30)
    Y = syn.packed_ball(rng, 6, 1.8, 1.2)
    Y -= Y.mean(0)
    zL = rng.uniform(-1, 1, 6)
    iM = oracle.snap_np(X, b, n)
    F = oracle.uncompressed_long_factors(iM, qM, t, a, lm, n, h)
    S = oracle.short_tables(t, a, lm, h, ns)
    tables = dict(n=n, b=b, R=F[0].shape[1], F1=F[0], F2=F[1], F3=F[2], n_sigma=ns,
                  S1=S[0], S2=S[1], S3=S[2])
    return b, n, h, t, a, lm, ns, X, qM, Y, zL, iM, tables, rng


def test_scorer_equals_pairwise_K_RS_sum(oracle):
    """Scorer with uncompressed factors == sum_l sum_m z_l z_m K_RS(i_l - i_m) (double loop):
    pins the shift-and-window factors (Eq. (6)), the short-range ball (Def. 2.1) and the
    scorer's bookkeeping against an independent pairwise evaluation."""
    b, n, h, t, a, lm, ns, X, qM, Y, zL, iM, tables, rng = _chain_case(oracle)
    P = 12
    poses = np.concatenate([syn.shoemake_quaternions(rng, P), rng.uniform(-4, 4, (P, 3))], 1)
    E, d, inv = oracle.score_poses(tables, X, qM, Y, zL, poses, 2.5)
    assert inv == 0
    for p in range(P):
        R_ = oracle.quat_to_rot(poses[p, :4])
        Xp = np.stack([oracle.transform(R_, y, poses[p, 4:]) for y in Y])
        iL = oracle.snap_np(Xp, b, n)
        ref, scale = [], 0.0
        for l in range(len(zL)):
            for m in range(len(qM)):
                k = oracle.K_RS(iL[l] - iM[m], t, a, lm, h, ns)
                ref.append(zL[l] * qM[m] * k)
        ref_sum = math.fsum(ref)
        scale = math.fsum(abs(v) for v in ref)
        assert abs(E[p] - ref_sum) <= 1e-12 * scale


def test_rs_energy_vs_brute_force_coulomb(oracle):
    """Whole-oracle pin (north_star): RS energy (uncompressed) vs the brute-force Coulomb sum
    of Eq. (13), normalised by S = sum |z z|/r (SURVEY §8(c) measured-magnitudes table):
    non-clashing poses within the O(h/r) snapping bound, and E_RS vs point Coulomb at the
    snapped cell centres within the O(h^2/r^2) + eps_q bound."""
    b, n, h, t, a, lm, ns, X, qM, Y, zL, iM, tables, rng = _chain_case(oracle, seed=1)
    P = 40
    u = syn.unit_vectors(rng, P)
    poses = np.concatenate([syn.shoemake_quaternions(rng, P), u * rng.uniform(7.5, 8.0, (P, 1))], 1)
    E, d, inv = oracle.score_poses(tables, X, qM, Y, zL, poses, 2.5)
    assert inv == 0
    centres = lambda i: -b + (i + 0.5) * h
    for p in range(P):
        R_ = oracle.quat_to_rot(poses[p, :4])
        Xp = np.stack([oracle.transform(R_, y, poses[p, 4:]) for y in Y])
        S = oracle.coulomb_scale(X, qM, Xp, zL)
        e_cont = oracle.coulomb_binding(X, qM, Xp, zL)
        e_snap = oracle.coulomb_binding(centres(iM), qM, centres(oracle.snap_np(Xp, b, n)), zL)
        assert abs(E[p] - e_snap) <= 1e-6 * S
        assert abs(E[p] - e_cont) <= 2e-2 * S


def test_swap_symmetry(oracle):
    """Eq. (15): sum_l z_l P_M(x_l) = sum_m z_m P_L(x_m).  With K_RS even
    (g[-d] == g[d]) the uncompressed RS energies agree to roundoff."""
    b, n, h, t, a, lm, ns, X, qM, Y, zL, iM, tables, rng = _chain_case(oracle, seed=2)
    tvec = np.array([3.0, -1.0, 2.0])
    Xl = Y + tvec                                   # ligand placed by a pure translation
    ident = np.array([[1.0, 0, 0, 0, *tvec]])
    E_ml, _, _ = oracle.score_poses(tables, X, qM, Y, zL, ident, 2.5)
    iL = oracle.snap_np(Xl, b, n)
    F = oracle.uncompressed_long_factors(iL, zL, t, a, lm, n, h)
    tab2 = dict(tables, F1=F[0], F2=F[1], F3=F[2], R=F[0].shape[1])
    E_lm, _, _ = oracle.score_poses(tab2, Xl, zL, X, qM, np.array([[1.0, 0, 0, 0, 0, 0, 0]]), 2.5)
    S = oracle.coulomb_scale(X, qM, Xl, zL)
    assert abs(E_ml[0] - E_lm[0]) <= 1e-13 * S


def test_decomposition_identity_brute_force(oracle):
    """E_N(M u L) = E_M + E_L + E_N(M, L), all by Eq. (10)/(13)."""
    rng = np.random.default_rng(7)
    X = rng.normal(size=(20, 3)) * 3
    Y = rng.normal(size=(5, 3)) * 3 + 10
    q, z = rng.uniform(-1, 1, 20), rng.uniform(-1, 1, 5)

    def total(P, c):
        r = cdist(P, P)
        np.fill_diagonal(r, np.inf)
        return 0.5 * math.fsum((c[:, None] * c[None, :] / r).ravel())
    lhs = total(np.vstack([X, Y]), np.concatenate([q, z]))
    rhs = total(X, q) + total(Y, z) + oracle.coulomb_binding(X, q, Y, z)
    assert abs(lhs - rhs) < 1e-12 * (abs(lhs) + 1)


def test_table2_first_order_grid_convergence(oracle):
    """Table 2: two opposite charges ~1.5 A apart; the tensor energy error
    halves per grid doubling (first order: error * n ~ const).  Averaged over placements."""
    rng = np.random.default_rng(8)
    b = 4.0
    sep = 1.5875
    errs = []
    for n in (32, 64, 128, 256):
        h, t, a, lm, ns = _rs_setup(oracle, b, n, 1e-8, 0.3)
        e = []
        for _ in range(24):
            c = rng.uniform(-1, 1, 3)
            u = syn.unit_vectors(rng, 1)[0]
            Xm = (c - 0.5 * sep * u)[None, :]
            Y = np.zeros((1, 3))
            iM = oracle.snap_np(Xm, b, n)
            F = oracle.uncompressed_long_factors(iM, np.array([1.0]), t, a, lm, n, h)
            S = oracle.short_tables(t, a, lm, h, ns)
            tab = dict(n=n, b=b, R=F[0].shape[1], F1=F[0], F2=F[1], F3=F[2], n_sigma=ns,
                       S1=S[0], S2=S[1], S3=S[2])
            pose = np.array([[1.0, 0, 0, 0, *(c + 0.5 * sep * u)]])
            E, _, _ = oracle.score_poses(tab, Xm, np.array([1.0]), Y, np.array([-1.0]), pose, 1.0)
            e.append(abs(E[0] - (-1.0 / sep)))
        errs.append(np.mean(e))
    ratios = [errs[i] / errs[i + 1] for i in range(3)]
    assert all(1.4 < r < 2.9 for r in ratios), (errs, ratios)


# ---------------------------------------------------------------------------------- O4-f32
def _lv32(oracle, F1, F2, F3, i=(0, 0, 0)):
    c = lambda x: oracle._p(np.ascontiguousarray(x, dtype=np.float64))
    return oracle.lib().oracle_long_value_f32(c(F1), c(F2), c(F3), F1.shape[1], *i)


def test_long_value_f32_exact_tables_equal_fp64(oracle):
    """Tables of small integers times powers of two: every product and partial sum is exact in
    binary32, so O4-f32 must equal O4 bit for bit (pins indexing, padding and widening)."""
    rng = np.random.default_rng(3)
    for R in [1, 3, 4, 5, 8, 12, 16, 24, 32]:
        # |entries| <= 8 on a 2^-1 grid: products on a 2^-3 grid below 2^9, sums below 2^14,
        # so every binary32 intermediate is exact
        F = [rng.integers(-4, 5, size=(6, R)).astype(float) * 2.0 ** rng.integers(-1, 2, size=(6, R))
             for _ in range(3)]
        for i in [(0, 1, 2), (5, 5, 5), (3, 0, 4)]:
            assert _lv32(oracle, *F, i=i) == _lv(oracle, *F, i=i)


def test_long_value_f32_order_worked_example(oracle):
    """O4-f32 order (reading A21), worked by hand in binary32 with
    q = (2^24, 1, 1, -2^24, 3) (R = 5, C4 = 2 quads):
      quad 0: (2^24 + 1) + (1 - 2^24) = 2^24 + (-(2^24 - 1)) = 1   [2^24 + 1 ties to 2^24]
      quad 1: (3 + 0) + (0 + 0) = 3;  phi = 1 + 3 = 4.
    The exact sum is 5; the sequential binary32 chain gives 3 (its first three terms round to 2^24)."""
    q = np.array([[2.0 ** 24, 1.0, 1.0, -2.0 ** 24, 3.0]])
    ones = np.ones_like(q)
    assert _lv32(oracle, q, ones, ones) == 4.0
    # inputs are rounded to binary32 first: 1 + 2^-30 becomes 1
    assert _lv32(oracle, np.array([[1.0 + 2.0 ** -30]]), np.ones((1, 1)), np.ones((1, 1))) == 1.0
    # and the product is rounded as (f1 f2) f3 in binary32
    t = float(np.float32(1.0 / 3.0))
    assert _lv32(oracle, np.array([[3.0]]), np.array([[1.0 / 3.0]]), np.array([[3.0]])) == \
        float((np.float32(3.0) * np.float32(t)) * np.float32(3.0))


@pytest.mark.parametrize("R", [4, 8, 12, 16, 24, 32])
def test_long_value_f32_rotation_invariance_and_bound(oracle, R):
    """Invariant under cyclic rotations of the rank quads (the kernel's XOR chunk order relies on
    it) and within gamma_k sum |q| of the exact sum of the products of the binary32-rounded
    factors, k = 2 (products) + 2 (quad) + log2(C4), u = 2^-24."""
    rng = np.random.default_rng(100 + R)
    C = 1
    while 4 * C < R:
        C *= 2
    for trial in range(40):
        F = [rng.normal(size=(1, 4 * C)) * np.exp(rng.normal(0, 2, size=(1, 4 * C))) for _ in range(3)]
        for f in F:
            f[:, R:] = 0.0
        base = _lv32(oracle, *[f[:, :R] for f in F])
        for rot in range(1, C):
            perm = np.concatenate([np.arange(4 * ((c + rot) % C), 4 * ((c + rot) % C) + 4) for c in range(C)])
            assert _lv32(oracle, *[f[:, perm] for f in F]) == base
        g = [np.float32(f[0, :R]).astype(np.float64) for f in F]
        ex = sum(Fraction(float(g[0][k])) * Fraction(float(g[1][k])) * Fraction(float(g[2][k]))
                 for k in range(R))
        mag = float(np.sum(np.abs(g[0] * g[1] * g[2])))
        k = 4 + int(np.log2(C))
        u = 2.0 ** -24
        assert abs(float(Fraction(base) - ex)) <= k * u / (1 - k * u) * mag * (1 + 1e-9)


def test_scorer_f32_mode_matches_long_value_f32(oracle):
    """mode bit 1 routes O4 through O4-f32: a one-atom ligand at the identity pose scores
    z * O4-f32 at its cell, and the fp32 energies stay within 1e-6 of sum |z phi| of fp64's."""
    rng = np.random.default_rng(8)
    n, b, R = 32, 8.0, 12
    F = [rng.normal(size=(n, R)) for _ in range(3)]
    tables = _tables(F, n=n, b=b)
    X = np.array([[7.9, 7.9, 7.9]])
    qM = np.array([0.0])
    Y = np.zeros((1, 3))
    zL = np.array([0.75])
    poses = np.array([[1.0, 0.0, 0.0, 0.0, 1.3, -2.2, 0.4]])
    E, _, _ = oracle.score_poses(tables, X, qM, Y, zL, poses, 1.0, long_only=True, f32=True)
    inv_h = n / (2 * b)
    i = tuple(int(oracle.lib().oracle_snap(float(v), b, inv_h, n)) for v in poses[0, 4:])
    assert E[0] == 0.75 * _lv32(oracle, *F, i=i)
    Yb = rng.normal(size=(40, 3))
    zb = rng.uniform(-1, 1, 40)
    pb = np.c_[np.tile([1.0, 0, 0, 0], (30, 1)), rng.uniform(-3, 3, size=(30, 3))]
    E32, _, _ = oracle.score_poses(tables, X, qM, Yb, zb, pb, 1.0, long_only=True, f32=True)
    E64, _, _ = oracle.score_poses(tables, X, qM, Yb, zb, pb, 1.0, long_only=True)
    for p in range(30):
        S = 0.0
        for l in range(40):
            x = Yb[l] + pb[p, 4:]
            il = tuple(int(oracle.lib().oracle_snap(float(v), b, inv_h, n)) for v in x)
            S += abs(zb[l] * _lv(oracle, *F, i=il))
        assert abs(E32[p] - E64[p]) <= 1e-6 * S


# ---------------------------------------------------------------------------------- N1 forces
def _forces_one_atom(oracle, F, n, b, t, z=1.0):
    tables = _tables(F, n=n, b=b)
    poses = np.array([[1.0, 0.0, 0.0, 0.0, *t]])
    out, inv = oracle.score_forces(tables, np.zeros((1, 3)), np.array([z]), poses)
    assert inv == 0
    return out[0]


def test_forces_linear_potential_exact(oracle):
    """phi = i0 (rank 1: F1[i] = i, F2 = F3 = 1): the backward difference is exactly 1 cell, so
    g = inv_h e0 and F = -z inv_h e0; a single atom at the centre has zero torque and radial
    resultant (r = 0).  At i0 = 0 the forward difference gives the same slope."""
    n, b = 16, 4.0
    inv_h = n / (2 * b)
    F = [np.arange(n, dtype=float)[:, None], np.ones((n, 1)), np.ones((n, 1))]
    for t0 in [0.3, -3.9]:                       # interior cell and cell 0
        out = _forces_one_atom(oracle, F, n, b, (t0, 1.1, -2.0), z=0.5)
        assert np.array_equal(out, [-0.5 * inv_h, 0, 0, 0, 0, 0, 0, 0, 0])


def test_forces_separable_exponential_closed_form(oracle):
    """phi(i) = exp(al i0) exp(be i1) exp(ga i2) (rank 1): the backward differences have the
    closed form g_a = phi(i) (1 - exp(-c_a)) inv_h (forward at i_a = 0: phi (exp(c_a) - 1))."""
    n, b = 16, 4.0
    inv_h = n / (2 * b)
    c = np.array([0.3, -0.2, 0.11])
    idx = np.arange(n)
    F = [np.exp(c[a] * idx)[:, None] for a in range(3)]
    for t in [(0.3, 1.1, -2.0), (-3.9, 2.6, 0.7)]:
        i = [int(oracle.lib().oracle_snap(float(v), b, inv_h, n)) for v in t]
        phi = np.exp(np.dot(c, i))
        g = np.array([phi * (1 - np.exp(-c[a])) if i[a] > 0 else phi * (np.exp(c[a]) - 1)
                      for a in range(3)]) * inv_h
        out = _forces_one_atom(oracle, F, n, b, t, z=-0.7)
        assert np.allclose(out[:3], 0.7 * g, rtol=1e-13, atol=0)


def test_forces_two_atom_torque_and_radial(oracle):
    """Two atoms at t +- d e1 with charges z, -z in phi = i0: atom forces -+z inv_h e0, radial
    projections 0 (F perpendicular to r), net force 0 and torque (0, 0, 2 d z inv_h) by hand."""
    n, b = 32, 8.0
    inv_h = n / (2 * b)
    F = [np.arange(n, dtype=float)[:, None], np.ones((n, 1)), np.ones((n, 1))]
    d, z = 1.25, 0.6
    Y = np.array([[0.0, d, 0.0], [0.0, -d, 0.0]])
    zL = np.array([z, -z])
    poses = np.array([[1.0, 0.0, 0.0, 0.0, 0.1, 0.2, 0.3]])
    out, _ = oracle.score_forces(_tables(F, n=n, b=b), Y, zL, poses)
    assert np.allclose(out[0], [0, 0, 0, 0, 0, 2 * d * z * inv_h, 0, 0, 0], atol=1e-12, rtol=0)
    # a rotation by 90 degrees about e2 maps e1 -> -e0: forces along r, torque 0, radial = net
    q = np.array([np.cos(np.pi / 4), 0, 0, np.sin(np.pi / 4)])
    out2, _ = oracle.score_forces(_tables(F, n=n, b=b), Y, zL, np.r_[q, 0.1, 0.2, 0.3][None])
    assert np.allclose(out2[0, 3:6], 0, atol=1e-12) and np.allclose(out2[0, 6:], out2[0, :3], atol=1e-12)


def test_forces_vs_analytic_coulomb_field(oracle):
    """Physics pin (the analytic field E_M): with the uncompressed long-range
    factors, the FD net force on well-separated ligands matches
    F = sum_l z_l sum_m z_m (x_l - x_m)/|x_l - x_m|^3 within the first-order FD/snapping error
    (relative 8 % of sum |F_l|, h = 0.16 A at 7.5-8 A) and with the right sign."""
    b, n, h, t, a, lm, ns, X, qM, Y, zL, iM, tables, rng = _chain_case(oracle, seed=4)
    P = 20
    u = syn.unit_vectors(rng, P)
    poses = np.concatenate([syn.shoemake_quaternions(rng, P), u * rng.uniform(7.5, 8.0, (P, 1))], 1)
    out, inv = oracle.score_forces(tables, Y, zL, poses)
    assert inv == 0
    for p in range(P):
        R = oracle.quat_to_rot(poses[p, :4])
        xl = Y @ R.T + poses[p, 4:]
        dx = xl[:, None, :] - X[None, :, :]
        r3 = np.linalg.norm(dx, axis=2) ** 3
        Fl = zL[:, None] * np.einsum("m,lmk->lk", qM, dx / r3[:, :, None])
        scale = np.abs(Fl).sum()
        assert np.linalg.norm(out[p, :3] - Fl.sum(0)) <= 0.08 * scale


# ---------------------------------------------------------------------------------- N2 PPIEM
def test_landscape_minima_rules():
    """PPIEM A6 (reading A23): strict minima on the periodic grid, ties toward the smaller
    index, NaN skipped; the oracle's and the library's host implementation agree."""
    from oracle import ppiem_oracle as po
    from paper_2510_26611_b200 import rsdock
    E = np.full((4, 5), 2.0)
    assert list(po.landscape_minima(E, 3)) == [0]            # constant: the smallest index only
    E[2, 3] = -1.0
    E[0, 0] = -0.5                                           # corner: neighbours wrap around
    E[3, 4] = -0.5 + 1e-9
    assert list(po.landscape_minima(E, 5)) == [2 * 5 + 3, 0]
    E[1, 1] = np.nan
    rng = np.random.default_rng(0)
    for trial in range(30):
        L = rng.integers(-3, 3, size=(rng.integers(1, 7), rng.integers(1, 7))).astype(float)
        L[rng.random(L.shape) < 0.2] = np.nan
        assert list(rsdock.rs_landscape_minima(L, 50)) == list(po.landscape_minima(L, 50))
    assert list(rsdock.rs_landscape_minima(E, 5)) == list(po.landscape_minima(E, 5))


def test_ppiem_oracle_two_charges_contact(oracle):
    """Single-atom protein at the origin and single-atom ligand: every direction stops at the
    vdW contact (sigma <= d <= sigma + tol) and the energy approaches z_M z_L / sigma within the
    grid and quadrature error (SPEC ppiem example, 'energy ~ z_M z_L / sigma')."""
    from oracle import ppiem_oracle as po
    b, n = 10.0, 128
    h, t, a, lm, ns = _rs_setup(oracle, b, n, 1e-8, 1.0)
    X = np.array([[0.01, -0.02, 0.03]])
    qM = np.array([0.8])
    iM = oracle.snap_np(X, b, n)
    F = oracle.uncompressed_long_factors(iM, qM, t, a, lm, n, h)
    S = oracle.short_tables(t, a, lm, h, ns)
    tables = dict(n=n, b=b, R=F[0].shape[1], F1=F[0], F2=F[1], F3=F[2], n_sigma=ns,
                  S1=S[0], S2=S[1], S3=S[2])
    dirs, quats = syn.planar_scan(8, 3)
    sigma, dcap, tol = 2.5, 4.5, 1e-3
    E, s, st = po.scan(tables, X, qM, np.zeros((1, 3)), np.array([-0.6]), X[0], dirs, quats,
                       8.0, sigma, dcap, tol)
    assert np.all(st == 0)
    d = np.abs(s)       # the ligand centre is the atom: d = |t - x_M| ~ s (X is the centre)
    assert np.all(d >= sigma) and np.all(d <= sigma + 2 * tol)
    # snapping moves each of the two charges by <= sqrt(3) h / 2, so their distance changes by
    # <= sqrt(3) h: relative error of 1/r <= sqrt(3) h / (sigma - sqrt(3) h)
    bound = math.sqrt(3) * h / (sigma - math.sqrt(3) * h)
    assert np.all(np.abs(E - 0.8 * -0.6 / s) <= (bound + 1e-6) * np.abs(0.8 * 0.6 / s))


# ---------------------------------------------------------------------------------- N4 Eq. (23)
def _two_proteins(oracle, seed):
    b, n, h, t, a, lm, ns, X, qM, Y, zL, iM, tables, rng = _chain_case(oracle, seed=seed)
    XB = syn.packed_ball(rng, 20, 3.5, 1.2) + np.array([0.0, 0.0, 6.5])
    qB = rng.uniform(-1, 1, 20)
    iB = oracle.snap_np(XB, b, n)
    FB = oracle.uncompressed_long_factors(iB, qB, t, a, lm, n, h)
    tB = dict(tables, F1=FB[0], F2=FB[1], F3=FB[2], R=FB[0].shape[1])
    return b, n, h, t, a, lm, ns, (X, qM, iM, tables), (XB, qB, iB, tB), Y, zL, rng


def test_complex_concatenation_is_the_union_protein(oracle):
    """Eq. (23), reading A24: the uncompressed factors of the union of two
    proteins (Eq. (6) over all atoms, A first) are exactly the rank concatenation of the parts'
    factors, so combine_tables reproduces the union tables bit for bit; and the concatenated
    scorer equals the literal sum over proteins, sum_p E_p, within the dd rounding bound."""
    b, n, h, t, a, lm, ns, A, B, Y, zL, rng = _two_proteins(oracle, seed=3)
    X = np.concatenate([A[0], B[0]])
    q = np.concatenate([A[1], B[1]])
    F = oracle.uncompressed_long_factors(np.concatenate([A[2], B[2]]), q, t, a, lm, n, h)
    comb = oracle.combine_tables([A[3], B[3]])
    for k, Fk in zip(("F1", "F2", "F3"), F):
        assert np.array_equal(comb[k], Fk)
    P = 24
    u = syn.unit_vectors(rng, P)
    poses = np.concatenate([syn.shoemake_quaternions(rng, P), u * rng.uniform(3.0, 7.0, (P, 1))], 1)
    E, d, inv = oracle.score_poses(comb, X, q, Y, zL, poses, 2.5)
    Es, ds, invs = oracle.score_complex([A[3], B[3]], [(A[0], A[1]), (B[0], B[1])], Y, zL, poses,
                                        2.5)
    assert inv == invs
    assert np.array_equal(np.isnan(E), np.isnan(Es))
    ok = ~np.isnan(E)
    assert ok.sum() > P // 2
    assert np.array_equal(d[ok], ds[ok])                 # min over the union = min of the mins
    EA, _, _ = oracle.score_poses(A[3], A[0], A[1], Y, zL, poses, 2.5)
    EB, _, _ = oracle.score_poses(B[3], B[0], B[1], Y, zL, poses, 2.5)
    for p in np.nonzero(ok)[0]:
        scale = abs(EA[p]) + abs(EB[p])
        assert abs(E[p] - Es[p]) <= 1e-13 * max(scale, 1e-300)


def test_complex_vs_brute_force_coulomb_of_both_proteins(oracle):
    """Eq. (23) against Eq. (13) summed over both proteins: the complex's RS energy at
    non-clashing poses matches the point-Coulomb energy of the ligand in the field of A and B
    at the snapped cell centres (O(h^2/r^2) + eps_q bound, as for one protein), while leaving
    either protein out misses by far more."""
    b, n, h, t, a, lm, ns, A, B, Y, zL, rng = _two_proteins(oracle, seed=4)
    comb = oracle.combine_tables([A[3], B[3]])
    X = np.concatenate([A[0], B[0]])
    q = np.concatenate([A[1], B[1]])
    P = 16
    u = syn.unit_vectors(rng, P)
    poses = np.concatenate([syn.shoemake_quaternions(rng, P), u * rng.uniform(8.0, 8.5, (P, 1))], 1)
    poses[:, 4:] += np.array([0.0, 0.0, 1.5])
    E, d, inv = oracle.score_poses(comb, X, q, Y, zL, poses, 2.5)
    centres = lambda i: -b + (i + 0.5) * h
    iX = oracle.snap_np(X, b, n)
    n_checked = n_missing_A = n_missing_B = 0
    for p in range(P):
        if np.isnan(E[p]):
            continue
        R_ = oracle.quat_to_rot(poses[p, :4])
        Xp = np.stack([oracle.transform(R_, y, poses[p, 4:]) for y in Y])
        if np.min(np.linalg.norm(Xp[:, None, :] - X[None, :, :], axis=2)) < 2.5:
            continue
        S = oracle.coulomb_scale(X, q, Xp, zL)
        iP = oracle.snap_np(Xp, b, n)
        e_snap = oracle.coulomb_binding(centres(iX), q, centres(iP), zL)
        assert abs(E[p] - e_snap) <= 1e-6 * S
        e_A = oracle.coulomb_binding(centres(A[2]), A[1], centres(iP), zL)
        e_B = oracle.coulomb_binding(centres(B[2]), B[1], centres(iP), zL)
        n_missing_B += abs(E[p] - e_A) > 1e-4 * S        # a dropped part would fail the bound
        n_missing_A += abs(E[p] - e_B) > 1e-4 * S
        n_checked += 1
    assert n_checked >= P // 2
    assert n_missing_A == n_checked and n_missing_B == n_checked


# ------------------------------------------------------- compression certificates (TEP step 4)
def _rand_cp(rng, n, K):
    return [rng.normal(size=(n, K)) for _ in range(3)]


def test_cp_norm_and_inner_gram_identity_vs_dense(oracle):
    """SPEC.md:77-85 frobenius_norm examples: all-ones rank-1 on n = 4 has norm 8; the Gram
    identity equals the dense norm / inner product (numpy on the materialised tensors) on
    random rank-6 and rank-5 tensors, n = 8, to 1e-12; certified error 0 for an exact copy and
    1 against the zero-rank tensor."""
    ones = [np.ones((4, 1))] * 3
    assert abs(math.sqrt(oracle.cp_norm2(ones)) - 8.0) < 1e-14
    rng = np.random.default_rng(41)
    A, B = _rand_cp(rng, 8, 6), _rand_cp(rng, 8, 5)
    TA = np.einsum("ik,jk,lk->ijl", *A)
    TB = np.einsum("ik,jk,lk->ijl", *B)
    assert abs(oracle.cp_norm2(A, block=4) - np.sum(TA * TA)) <= 1e-12 * np.sum(TA * TA)
    assert abs(oracle.cp_inner(A, B, block=4) - np.sum(TA * TB)) <= 1e-12 * np.sum(np.abs(TA * TB))
    assert np.allclose(oracle.cp_dense(*A), TA, rtol=0, atol=1e-12)
    assert oracle.certified_rel_error(A, A) <= 1e-7
    zero = [np.zeros((8, 1))] * 3
    assert abs(oracle.certified_rel_error(A, zero) - 1.0) <= 1e-14
    D = TA - TB
    ref = math.sqrt(np.sum(D * D) / np.sum(TA * TA))
    assert abs(oracle.certified_rel_error(A, B) - ref) <= 1e-10 * ref


def test_unfolding_tails_and_hosvd_vs_numpy_svd(oracle):
    """Unfolding tails from the Grams equal the tail singular values of numpy's SVD of the dense
    unfoldings; HOSVD's error sits between the largest tail and the root sum of the tails
    (the De Lathauwer bounds) and vanishes for a tensor of multilinear rank <= R."""
    rng = np.random.default_rng(42)
    F = _rand_cp(rng, 10, 7)
    T = np.einsum("ik,jk,lk->ijl", *F)
    n2 = float(np.sum(T * T))
    tails = oracle.unfolding_tails(F, 3)
    for a in range(3):
        s = np.linalg.svd(np.moveaxis(T, a, 0).reshape(10, -1), compute_uv=False)
        assert abs(tails[a] - np.sum(s[3:] ** 2)) <= 1e-10 * n2
    e = oracle.hosvd_dense(T, 3)[4]
    assert math.sqrt(max(tails) / n2) - 1e-12 <= e <= math.sqrt(sum(tails) / n2) + 1e-12
    assert oracle.hosvd_dense(T, 7)[4] <= 1e-6


def test_cp_als_recovers_exact_low_rank(oracle):
    """Dense CP-ALS recovers a generic rank-3 tensor (relative error < 1e-8) and its error is
    never below the unfolding lower bound at a smaller width."""
    rng = np.random.default_rng(43)
    F = _rand_cp(rng, 9, 3)
    T = np.einsum("ik,jk,lk->ijl", *F)
    assert oracle.cp_als_dense(T, 3, iters=300, seed=1)[3] < 1e-8
    tails = oracle.unfolding_tails(F, 2)
    e2 = oracle.cp_als_dense(T, 2, iters=100, seed=1)[3]
    assert e2 >= math.sqrt(max(tails) / float(np.sum(T * T))) - 1e-12


# ----------------------------------------------------------------------------- O4-T (N5)

def _tucker(rng, n, r):
    return {"U0": rng.standard_normal((n, r[0])), "U1": rng.standard_normal((n, r[1])),
            "U2": rng.standard_normal((n, r[2])), "G": rng.standard_normal(tuple(r))}


def test_tucker_value_rank_one_closed_form(oracle):
    """O4-T with r = (1, 1, 1) is u0 (u1 (g u2)): exact in binary64 for small integers."""
    tk = {"U0": np.array([[3.0], [5.0]]), "U1": np.array([[-2.0], [7.0]]),
          "U2": np.array([[4.0], [11.0]]), "G": np.array([[[-6.0]]])}
    for i0 in range(2):
        for i1 in range(2):
            for i2 in range(2):
                want = tk["U0"][i0, 0] * (tk["U1"][i1, 0] * (tk["G"][0, 0, 0] * tk["U2"][i2, 0]))
                assert oracle.tucker_value(tk, i0, i1, i2) == want


def test_tucker_value_dense_materialisation(oracle):
    """O4-T equals the dense Tucker tensor sum_abc G_abc U0[i,a] U1[j,b] U2[k,c] (numpy einsum)
    at every cell of a small grid with unequal ranks, to rounding."""
    rng = np.random.default_rng(11)
    n, r = 6, (2, 3, 4)
    tk = _tucker(rng, n, r)
    T = np.einsum("abc,ia,jb,kc->ijk", tk["G"], tk["U0"], tk["U1"], tk["U2"])
    got = np.array([[[oracle.tucker_value(tk, i, j, k) for k in range(n)] for j in range(n)]
                    for i in range(n)])
    assert np.max(np.abs(got - T)) <= 1e-13 * np.max(np.abs(T))


def test_tucker_value_order_hand_worked(oracle):
    """The contraction order of reading A26, by hand: with G[0,0,:] = (1e16, 1, -1e16) and
    u2 = (1, 1, 1) the innermost chain is ((0 + 1e16) + 1) + (-1e16) = 0 in binary64 (the exact
    value is 1; a chain in the other order, (-1e16 + 1) + 1e16, also gives 0, and the tree
    (1e16 + -1e16) + 1 gives 1): O4-T is the ascending chain."""
    tk = {"U0": np.array([[1.0]]), "U1": np.array([[1.0]]), "U2": np.array([[1.0, 1.0, 1.0]]),
          "G": np.array([[[1e16, 1.0, -1e16]]])}
    assert oracle.tucker_value(tk, 0, 0, 0) == 0.0
    tk["G"] = np.array([[[1e16, -1e16, 1.0]]])
    assert oracle.tucker_value(tk, 0, 0, 0) == 1.0


def test_tucker_scorer_is_zL_weighted_sum(oracle):
    """The scorer's long-range part with a Tucker form (mode bit 2) is the double-double sum of
    z_l O4-T(i_l) over the ligand atoms: one atom at the identity pose reproduces the cell value."""
    rng = np.random.default_rng(5)
    n, b = 16, 4.0
    tk = _tucker(rng, n, (2, 2, 3))
    tb = {"n": n, "b": b, "R": 1, "F1": np.zeros((n, 1)), "F2": np.zeros((n, 1)),
          "F3": np.zeros((n, 1)), "n_sigma": 0, "S1": np.zeros((1, 0)), "S2": np.zeros((1, 0)),
          "S3": np.zeros((1, 0))}
    Y = np.array([[0.3, -1.1, 2.2]])
    zL = np.array([0.75])
    poses = np.array([[1.0, 0, 0, 0, 0.0, 0.0, 0.0]])
    E, d, inv = oracle.score_poses(tb, np.zeros((0, 3)), np.zeros(0), Y, zL, poses, 2.5,
                                   long_only=True, tucker=tk)
    c = [oracle.snap_np(Y[0], b, n)[a] for a in range(3)]
    assert inv == 0 and E[0] == 0.75 * oracle.tucker_value(tk, *c)
