"""Seeded synthetic workloads C1..C5 (BASELINE.json `configs`, recipes in SURVEY.md §8(d) M2).

This module is INPUT GENERATION ONLY: it holds none of the method's arithmetic (no
quadrature, no snapping, no tensor evaluation, no energy).  Both the oracle and the CUDA
path consume what it produces, which is the only thing they share.

The paper measures on no public dataset: its workloads are synthetic flat clusters with
random charges (Table 1 caption PAPER.md:739-740) and an unidentified
379-atom protein that is not available.  The five BASELINE configs
stand in for them; every unstated detail is fixed by the rule cited beside it
(DESIGN.md "Input recipe").

Units: Angstrom and elementary charge.  Every cluster is centred at the origin.
Poses are (w, x, y, z, tx, ty, tz): unit quaternion (scalar first) + translation of the
ligand's geometric centre (the ligand body coordinates are centred at their mean), which
is the paper's q = (x_0, phi), widened to full SO(3).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

SIGMA_VDW = 2.5          # vdW threshold [A], BASELINE C1; used for all configs (ledger A11)
D_CAP = 2.5              # min-distance reporting cap [A] (= sigma_vdw)
SIGMA_SPLIT = 2.0        # range-split radius sigma_s [A] (ledger A2)
EPS_SPLIT = 1e-6         # Gaussian effective-support threshold (ledger A7)
EPS_QUAD = 1e-6          # sinc quadrature target relative error (ledger A6)
MIN_SEP = 1.2            # RSA minimum separation [A] (BASELINE C1)


@dataclasses.dataclass
class Workload:
    name: str
    protein_xyz: np.ndarray   # (M, 3) float64
    protein_q: np.ndarray     # (M,)   float64
    ligand_xyz: np.ndarray    # (L, 3) float64, body frame (mean-centred)
    ligand_q: np.ndarray      # (L,)   float64
    poses: np.ndarray         # (P, 7) float64  (w,x,y,z,tx,ty,tz)
    grid_n: int
    box_half_width: float
    rank_R: int
    sigma_split: float = SIGMA_SPLIT
    sigma_vdw: float = SIGMA_VDW
    dmin_cap: float = D_CAP
    eps_split: float = EPS_SPLIT
    eps_quad: float = EPS_QUAD
    n_rot: int = 0            # poses are translation-major products when n_rot > 0
    note: str = ""

    @property
    def M(self) -> int:
        return int(self.protein_q.shape[0])

    @property
    def L(self) -> int:
        return int(self.ligand_q.shape[0])

    @property
    def P(self) -> int:
        return int(self.poses.shape[0])

    def params(self) -> dict:
        return dict(grid_n=self.grid_n, rank_R=self.rank_R, sigma_split=self.sigma_split,
                    sigma_vdw=self.sigma_vdw, dmin_cap=self.dmin_cap, eps_split=self.eps_split,
                    eps_quad=self.eps_quad)

    def with_poses(self, poses: np.ndarray, suffix: str = "") -> "Workload":
        return dataclasses.replace(self, poses=np.ascontiguousarray(poses, dtype=np.float64),
                                   name=self.name + suffix)


# --------------------------------------------------------------------------------------
# geometry samplers
# --------------------------------------------------------------------------------------

def _rsa(rng: np.random.Generator, n: int, propose, min_sep: float, max_rounds: int = 400):
    """Random sequential addition: accept proposals at >= min_sep from every accepted point.

    `propose(rng, k)` returns k candidate points (k, 3).  Spatial hash with cell = min_sep.
    """
    cell = min_sep
    grid: dict = {}
    pts = np.empty((n, 3), dtype=np.float64)
    cnt = 0
    sep2 = min_sep * min_sep
    offs = [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)]
    for _ in range(max_rounds):
        cand = propose(rng, max(256, 2 * (n - cnt)))
        keys = np.floor(cand / cell).astype(np.int64)
        for p, k in zip(cand, keys):
            kx, ky, kz = int(k[0]), int(k[1]), int(k[2])
            ok = True
            for (a, b, c) in offs:
                lst = grid.get((kx + a, ky + b, kz + c))
                if lst is None:
                    continue
                for j in lst:
                    d = pts[j] - p
                    if d[0] * d[0] + d[1] * d[1] + d[2] * d[2] < sep2:
                        ok = False
                        break
                if not ok:
                    break
            if ok:
                pts[cnt] = p
                grid.setdefault((kx, ky, kz), []).append(cnt)
                cnt += 1
                if cnt == n:
                    return pts
    raise RuntimeError(f"RSA could not place {n} points (placed {cnt})")


def _ball_proposer(radius: float, center=(0.0, 0.0, 0.0)):
    c = np.asarray(center, dtype=np.float64)

    def propose(rng, k):
        v = rng.normal(size=(k, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        r = radius * rng.random(k) ** (1.0 / 3.0)
        return c + v * r[:, None]
    return propose


def _ellipsoid_proposer(axes, centers):
    axes = np.asarray(axes, dtype=np.float64)
    centers = [np.asarray(c, dtype=np.float64) for c in centers]

    def propose(rng, k):
        v = rng.normal(size=(k, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        r = rng.random(k) ** (1.0 / 3.0)
        pts = v * r[:, None] * axes
        which = rng.integers(0, len(centers), size=k)
        return pts + np.stack(centers)[which]
    return propose


def packed_ball(rng, n, radius, min_sep=MIN_SEP):
    return _rsa(rng, n, _ball_proposer(radius), min_sep)


def ligand_body(rng, L, min_sep=MIN_SEP):
    """Packed ball with the tiny ligand's density, r = 3 A (L/20)^(1/3), mean-centred (M2)."""
    r = 3.0 * (L / 20.0) ** (1.0 / 3.0)
    x = packed_ball(rng, L, r, min_sep)
    return x - x.mean(axis=0)


def shoemake_quaternions(rng, k):
    """Uniform random unit quaternions (Shoemake), returned scalar-first (w, x, y, z)."""
    u1, u2, u3 = rng.random(k), rng.random(k), rng.random(k)
    a, b = np.sqrt(1.0 - u1), np.sqrt(u1)
    x = a * np.sin(2 * np.pi * u2)
    y = a * np.cos(2 * np.pi * u2)
    z = b * np.sin(2 * np.pi * u3)
    w = b * np.cos(2 * np.pi * u3)
    return np.stack([w, x, y, z], axis=1)


def unit_vectors(rng, k):
    v = rng.normal(size=(k, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def partial_charges(rng, n, std, clip=1.0):
    return np.clip(rng.normal(0.0, std, size=n), -clip, clip)


def set_net_charge(q, target, clip=1.0, tol=1e-12, iters=200):
    """Shift all charges by (target - sum q)/M, re-clip, iterate (ledger A14)."""
    q = q.copy()
    for _ in range(iters):
        d = target - q.sum()
        if abs(d) < tol:
            return q
        q = np.clip(q + d / q.size, -clip, clip)
    raise RuntimeError("net charge did not converge")


def product_poses(quats, trans):
    """Translation-major product: pose p = i_t * n_rot + i_r (M2)."""
    nr, nt = quats.shape[0], trans.shape[0]
    poses = np.empty((nt * nr, 7), dtype=np.float64)
    poses[:, :4] = np.tile(quats, (nt, 1))
    poses[:, 4:] = np.repeat(trans, nr, axis=0)
    return poses


_POSE_STREAM = 0


def _streams(seed):
    ss = np.random.SeedSequence(seed).spawn(6)
    # fixed order: protein xyz, protein q, ligand xyz, ligand q, rotations, translations
    g = [np.random.default_rng(s) for s in ss]
    if _POSE_STREAM:
        # an independent pose batch (weak-scaling shard) for the same protein and ligand
        r = np.random.SeedSequence([seed, _POSE_STREAM]).spawn(2)
        g[4], g[5] = np.random.default_rng(r[0]), np.random.default_rng(r[1])
    return g


# --------------------------------------------------------------------------------------
# the five configs
# --------------------------------------------------------------------------------------

def config_c1(seed=0, n_poses=1000) -> Workload:
    """tiny: 200 charges in a 10 A ball (sep 1.2), q~U[-1,1]; 20-atom ligand in a 3 A ball;
    n=256, b=20, R=8; 1000 poses = Shoemake q x t~U([-7.5,7.5]^3)."""
    g_px, g_pq, g_lx, g_lq, g_rot, g_tr = _streams(seed)
    X = packed_ball(g_px, 200, 10.0)
    q = g_pq.uniform(-1.0, 1.0, size=200)
    Y = ligand_body(g_lx, 20)
    z = g_lq.uniform(-1.0, 1.0, size=20)
    quats = shoemake_quaternions(g_rot, n_poses)
    t = g_tr.uniform(-7.5, 7.5, size=(n_poses, 3))
    poses = np.concatenate([quats, t], axis=1)
    return Workload("C1", X, q, Y, z, poses, grid_n=256, box_half_width=20.0, rank_R=8,
                    note="tiny; '15 A cube' read as edge 15 A centred on the protein")


def config_c2(seed=0, n_rot=100) -> Workload:
    """2000-atom packed ball (3.5 A mean spacing), q~N(0,0.4) clip, net +5; 50-atom ligand
    q~N(0,0.3); n=1024, b=40, R=12; 100 rotations x 10x10x10 lattice (1 A) near the surface."""
    g_px, g_pq, g_lx, g_lq, g_rot, g_tr = _streams(seed)
    M = 2000
    radius = (M * 3.5 ** 3 * 3.0 / (4.0 * math.pi)) ** (1.0 / 3.0)
    X = packed_ball(g_px, M, radius)
    q = set_net_charge(partial_charges(g_pq, M, 0.4), 5.0)
    Y = ligand_body(g_lx, 50)
    z = partial_charges(g_lq, 50, 0.3)
    quats = shoemake_quaternions(g_rot, n_rot)
    Rp = float(np.linalg.norm(X, axis=1).max())
    rL = float(np.linalg.norm(Y, axis=1).max())
    c = (Rp + rL) * np.ones(3) / math.sqrt(3.0)
    j = np.arange(10, dtype=np.float64) - 4.5
    lat = np.stack(np.meshgrid(j, j, j, indexing="ij"), axis=-1).reshape(-1, 3)
    trans = c + lat
    return Workload("C2", X, q, Y, z, product_poses(quats, trans), grid_n=1024,
                    box_half_width=40.0, rank_R=12, n_rot=n_rot)


def _ellipsoid_surface_shell(rng, k, axes, dmin, dmax):
    u = unit_vectors(rng, k)
    s = u / np.sqrt(((u / np.asarray(axes)) ** 2).sum(axis=1, keepdims=True))
    delta = rng.uniform(dmin, dmax, size=(k, 1))
    return s + delta * u


def config_c3(seed=0, n_rot=1000, n_trans=1000) -> Workload:
    """10,000-atom ellipsoid (30/25/20 A), q~N(0,0.4); 60-atom ligand q~N(0,0.3); n=4096,
    b=64, R=16; 1000 rotations x 1000 translations on a 2-8 A shell outside the surface."""
    g_px, g_pq, g_lx, g_lq, g_rot, g_tr = _streams(seed)
    M = 10000
    axes = (30.0, 25.0, 20.0)
    X = _rsa(g_px, M, _ellipsoid_proposer(axes, [(0, 0, 0)]), MIN_SEP)
    q = partial_charges(g_pq, M, 0.4)
    Y = ligand_body(g_lx, 60)
    z = partial_charges(g_lq, 60, 0.3)
    quats = shoemake_quaternions(g_rot, n_rot)
    trans = _ellipsoid_surface_shell(g_tr, n_trans, axes, 2.0, 8.0)
    return Workload("C3", X, q, Y, z, product_poses(quats, trans), grid_n=4096,
                    box_half_width=64.0, rank_R=16, n_rot=n_rot)


def config_c4(seed=0, n_poses=10_000_000) -> Workload:
    """Two-protein complex: 2 x 25,000-atom ellipsoids (40.7/33.9/27.1 A) centred (+-41.7,0,0),
    q~N(0,0.4); 200-atom ligand; n=16384, b=128, R=24; Shoemake q x t uniform in the box
    shrunk by r_max + h (ledger A16).  Built as ONE RS tensor (ledger A15)."""
    g_px, g_pq, g_lx, g_lq, g_rot, g_tr = _streams(seed)
    s = 2.5 ** (1.0 / 3.0)
    axes = (30.0 * s, 25.0 * s, 20.0 * s)
    X = _rsa(g_px, 50000, _ellipsoid_proposer(axes, [(-41.7, 0, 0), (41.7, 0, 0)]), MIN_SEP)
    q = partial_charges(g_pq, 50000, 0.4)
    Y = ligand_body(g_lx, 200)
    z = partial_charges(g_lq, 200, 0.3)
    b, n = 128.0, 16384
    rmax = float(np.linalg.norm(Y, axis=1).max())
    lim = b - rmax - 2 * b / n
    quats = shoemake_quaternions(g_rot, n_poses)
    t = g_tr.uniform(-lim, lim, size=(n_poses, 3))
    return Workload("C4", X, q, Y, z, np.concatenate([quats, t], axis=1), grid_n=n,
                    box_half_width=b, rank_R=24)


def config_c5(seed=0, rank_R=16, sigma_mult=1, n_poses=100_000) -> Workload:
    """Protein-protein: receptor 5,000 atoms (ball r=19.58 A), rigid partner 5,000 atoms (same
    generator, independent stream), q~N(0,0.4); n=8192, b=96; R in {8,16,32} x sigma_s in
    {2,4,6} A; t = (R_rec + R_par + delta) u, delta~U[0,10]."""
    g_px, g_pq, g_lx, g_lq, g_rot, g_tr = _streams(seed)
    r = 19.58
    X = packed_ball(g_px, 5000, r)
    q = partial_charges(g_pq, 5000, 0.4)
    Y = packed_ball(g_lx, 5000, r)
    Y = Y - Y.mean(axis=0)
    z = partial_charges(g_lq, 5000, 0.4)
    Rr = float(np.linalg.norm(X, axis=1).max())
    Rp = float(np.linalg.norm(Y, axis=1).max())
    quats = shoemake_quaternions(g_rot, n_poses)
    u = unit_vectors(g_tr, n_poses)
    delta = g_tr.uniform(0.0, 10.0, size=(n_poses, 1))
    t = (Rr + Rp + delta) * u
    return Workload(f"C5_R{rank_R}_s{sigma_mult}", X, q, Y, z,
                    np.concatenate([quats, t], axis=1), grid_n=8192, box_half_width=96.0,
                    rank_R=rank_R, sigma_split=SIGMA_SPLIT * sigma_mult)


CONFIGS = {"C1": config_c1, "C2": config_c2, "C3": config_c3, "C4": config_c4, "C5": config_c5}


def make(name: str, pose_stream: int = 0, **kw) -> Workload:
    """Config `name`; pose_stream > 0 draws an independent pose batch (same protein/ligand)."""
    global _POSE_STREAM
    _POSE_STREAM = int(pose_stream)
    try:
        return CONFIGS[name](**kw)
    finally:
        _POSE_STREAM = 0


def subsample(poses: np.ndarray, k: int, seed: int = 1) -> tuple[np.ndarray, np.ndarray]:
    """Seeded subsample of k pose indices (sorted), for oracle-sized parity / CPU baselines."""
    P = poses.shape[0]
    if k >= P:
        idx = np.arange(P)
    else:
        idx = np.sort(np.random.default_rng(seed).choice(P, size=k, replace=False))
    return idx, np.ascontiguousarray(poses[idx])


def random_small(seed=0, M=30, L=7, n=32, b=8.0, R=4, P=64, protein_radius=3.0,
                 trans=3.0) -> Workload:
    """Small random workload for parity tests (several tiles + ragged tail at tiny sizes)."""
    g = _streams(seed)
    X = packed_ball(g[0], M, protein_radius, 0.8)
    q = g[1].uniform(-1, 1, M)
    Y = packed_ball(g[2], L, 1.5, 0.8)
    Y = Y - Y.mean(axis=0)
    z = g[3].uniform(-1, 1, L)
    quats = shoemake_quaternions(g[4], P)
    t = g[5].uniform(-trans, trans, size=(P, 3))
    return Workload(f"small{seed}", X, q, Y, z, np.concatenate([quats, t], axis=1), grid_n=n,
                    box_half_width=b, rank_R=R, sigma_split=1.0, sigma_vdw=1.0, dmin_cap=1.5)


def planar_scan(m_P: int, m_L: int):
    """PPIEM scan grid in the z = 0 plane (A0): m_P directions
    (cos phi_j, sin phi_j, 0), phi_j = 2 pi j / m_P, and m_L ligand self-rotations about e_z,
    quaternions (cos(phi_k / 2), 0, 0, sin(phi_k / 2)), phi_k = 2 pi k / m_L."""
    phi = 2.0 * math.pi * np.arange(m_P) / m_P
    dirs = np.stack([np.cos(phi), np.sin(phi), np.zeros(m_P)], axis=1)
    psi = 2.0 * math.pi * np.arange(m_L) / m_L
    quats = np.stack([np.cos(psi / 2), np.zeros(m_L), np.zeros(m_L), np.sin(psi / 2)], axis=1)
    return dirs, quats


def complex_parts(w: Workload, axis: int = 0) -> list:
    """The proteins of a two-protein complex whose members lie on either side of the plane
    x_axis = 0 (C4's two ellipsoids; complex_small): [(X_A, q_A), (X_B, q_B)], A at x < 0."""
    left = w.protein_xyz[:, axis] < 0.0
    return [(np.ascontiguousarray(w.protein_xyz[m]), np.ascontiguousarray(w.protein_q[m]))
            for m in (left, ~left)]


def complex_small(seed=0, M=(30, 24), L=7, n=64, b=8.0, R=4, P=160, radius=2.5,
                  trans=4.0) -> Workload:
    """Small two-protein complex for Eq. (23) parity: balls of M[0] and M[1] atoms (radius
    2.5 A) centred at (-3.2, 0, 0) and (+3.2, 0, 0) (in general +-(radius + 0.7)); ligand and
    poses as random_small, the translations uniform in [-trans, trans]^3 (many poses clash with
    one protein or sit between)."""
    g = _streams(seed + 100)
    c = radius + 0.7
    XA = packed_ball(g[0], M[0], radius, 0.8) + np.array([-c, 0.0, 0.0])
    XB = packed_ball(g[1], M[1], radius, 0.8) + np.array([c, 0.0, 0.0])
    q = g[2].uniform(-1, 1, M[0] + M[1])
    Y = packed_ball(g[3], L, 1.5, 0.8)
    Y = Y - Y.mean(axis=0)
    z = g[4].uniform(-1, 1, L)
    quats = shoemake_quaternions(g[5], P)
    t = g[5].uniform(-trans, trans, size=(P, 3))
    return Workload(f"complex{seed}", np.concatenate([XA, XB]), q, Y, z,
                    np.concatenate([quats, t], axis=1), grid_n=n, box_half_width=b, rank_R=R,
                    sigma_split=1.0, sigma_vdw=1.0, dmin_cap=1.5)
