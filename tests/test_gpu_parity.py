"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same seeded inputs.

Bar (north_star / SURVEY.md §8(c) M8): per-pose energy within 1e-12 relative (expected
bitwise), min distance bitwise, identical NaN (invalid-pose) pattern and count.  Small cases
compare every pose; full-size configs run the whole batch in the launch configuration
bench.py times and compare a seeded sample of poses the oracle scores one by one."""
import math
import os
import sys

import numpy as np
import pytest

from synth import configs as syn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu

REL = 1e-12


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build_library()
    from paper_2510_26611_b200 import rsdock
    from oracle import rs_oracle
    rs_oracle.lib()
    return torch, rsdock, rs_oracle


def build(rsdock, w, **kw):
    prm = dict(w.params())
    prm.update(kw)
    return rsdock.Protein(w.protein_q, w.protein_xyz, w.box_half_width, **prm)


def gpu_score(torch, rsdock, prot, w, poses, async_api=False):
    dev = torch.device("cuda:0")
    q = torch.tensor(w.ligand_q, device=dev)
    y = torch.tensor(w.ligand_xyz, device=dev).contiguous()
    ps = torch.tensor(poses, device=dev).contiguous()
    P = ps.shape[0]
    E = torch.empty(P, dtype=torch.float64, device=dev)
    D = torch.empty(P, dtype=torch.float64, device=dev)
    if async_api:
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        prot.score_async(q, y, ps, E, D, cnt)
        torch.cuda.synchronize()
        inv = int(cnt.item())
    else:
        inv = rsdock.rs_score_poses(prot.handle, q, y, w.L, ps, P, E, D)
    return E.cpu().numpy(), D.cpu().numpy(), inv


def compare(Eg, Dg, Eo, Do, invg=None, invo=None):
    assert np.array_equal(np.isnan(Eg), np.isnan(Eo))
    assert np.array_equal(np.isnan(Dg), np.isnan(Do))
    ok = ~np.isnan(Eo)
    rel = np.abs(Eg[ok] - Eo[ok]) / np.maximum(np.abs(Eo[ok]), 1e-300)
    assert np.all((rel <= REL) | (Eg[ok] == Eo[ok])), f"max rel {rel.max():.3e}"
    assert np.array_equal(Dg[ok], Do[ok])
    if invg is not None:
        assert invg == invo
    return float(np.mean(Eg[ok] == Eo[ok])) if ok.any() else 1.0


def oracle_score(rs_oracle, prot, w, poses, idx=None):
    tb = prot.export_tables()
    ps = poses if idx is None else poses[idx]
    return rs_oracle.score_poses(tb, w.protein_xyz, w.protein_q, w.ligand_xyz, w.ligand_q, ps,
                                 w.dmin_cap)


# ----------------------------------------------------------------------------- widths / tiles

@pytest.mark.parametrize("R", [4, 8, 12, 16, 24, 32, 10])
def test_small_random_all_widths(env, R):
    """Every compiled width (and a runtime width, 10), several tiles and a ragged tail
    (P = 333 = 5 tiles of 64 + 13)."""
    torch, rsdock, rs_oracle = env
    w = syn.random_small(seed=R, M=40, L=9, n=64, b=8.0, R=R, P=333)
    prot = build(rsdock, w)
    Eg, Dg, inv = gpu_score(torch, rsdock, prot, w, w.poses)
    Eo, Do, invo = oracle_score(rs_oracle, prot, w, w.poses)
    compare(Eg, Dg, Eo, Do, inv, invo)


def test_score_path_plan(env):
    """rs_score_path reports the variant the launcher picks: the shared-memory window when the
    whole factor set fits (C1), L2 rows when one translation's rows do not (C5: a 5,000-atom
    partner at n = 8192), the runtime-width kernel for an uncompiled width; scoring agrees with
    the oracle on each."""
    torch, rsdock, rs_oracle = env
    w = syn.config_c1(n_poses=64)
    prot = build(rsdock, w)
    assert rsdock.rs_score_path(prot.handle, w.ligand_xyz) == rsdock.RS_PATH_WINDOW
    w10 = syn.random_small(seed=3, M=40, L=9, n=64, b=8.0, R=10, P=40)
    p10 = build(rsdock, w10)
    assert rsdock.rs_score_path(p10.handle, w10.ligand_xyz) == rsdock.RS_PATH_L2_RUNTIME
    w5 = syn.config_c5(rank_R=8, sigma_mult=1, n_poses=64)
    p5 = build(rsdock, w5)
    assert rsdock.rs_score_path(p5.handle, w5.ligand_xyz) == rsdock.RS_PATH_L2
    # a small ligand on the same handle fits the window again
    assert rsdock.rs_score_path(p5.handle, w5.ligand_xyz[:20] * 0.1) == rsdock.RS_PATH_WINDOW
    with pytest.raises(ValueError):      # the plan reads a host ligand
        rsdock.rs_score_path(p5.handle, torch.tensor(w5.ligand_xyz, device="cuda:0"))


_STALL_SCRIPT = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2510_26611_b200 import rsdock
from synth import configs as syn
w = syn.config_c1(n_poses=1000)
prot = rsdock.Protein(w.protein_q, w.protein_xyz, w.box_half_width, **w.params())
poses = np.ascontiguousarray(np.tile(w.poses, (3, 1)))
E = np.empty(len(poses)); D = np.empty(len(poses))
inv = rsdock.rs_score_poses(prot.handle, w.ligand_q, w.ligand_xyz, w.L, poses, len(poses), E, D)
np.save(sys.argv[2], np.stack([E, D]))
print("invalid", inv)
'''


@pytest.mark.parametrize("fault", [False, True])
def test_streamed_pipeline_stall_falls_back(env, tmp_path, fault):
    """The streamed host pipeline (one launch waiting on copy-engine arrival flags) on a small
    batch (RS_STREAM_MIN_POSES): bitwise the device-resident results; with the arrival flags
    withheld (fault injection: the copies never run beside the kernel) the launch gives up after
    its wall-time bound and the call recomputes with chunked launches, still bitwise equal."""
    import subprocess
    torch, rsdock, rs_oracle = env
    envv = dict(os.environ, RS_STREAM_MIN_POSES="1000")
    if fault:
        envv["RS_STREAM_FAULT_DROP_FLAGS"] = "1"
    out = tmp_path / "ed.npy"
    r = subprocess.run([sys.executable, "-c", _STALL_SCRIPT, ROOT, str(out)], env=envv,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert ("stalled" in r.stderr) == fault
    Eh, Dh = np.load(out)
    w = syn.config_c1(n_poses=1000)
    prot = build(rsdock, w)
    Eg, Dg, inv = gpu_score(torch, rsdock, prot, w, np.tile(w.poses, (3, 1)))
    assert np.array_equal(Eh, Eg, equal_nan=True) and np.array_equal(Dh, Dg, equal_nan=True)


def test_loaded_handle_scores_identically(env, tmp_path):
    """A handle written by rs_save_handle and read back by rs_load_handle scores every pose
    bit for bit like the handle it came from (the setup is skipped, S10 runs)."""
    torch, rsdock, rs_oracle = env
    w = syn.config_c2(n_rot=2)
    prot = build(rsdock, w)
    path = tmp_path / "c2.rsh"
    prot.save(path)
    again = rsdock.Protein.load(path, device=0)
    Ea, Da, ia = gpu_score(torch, rsdock, prot, w, w.poses)
    Eb, Db, ib = gpu_score(torch, rsdock, again, w, w.poses)
    assert ia == ib and np.array_equal(Ea, Eb, equal_nan=True) and np.array_equal(Da, Db, equal_nan=True)


def test_c1_all_poses(env):
    torch, rsdock, rs_oracle = env
    w = syn.config_c1()
    prot = build(rsdock, w)
    Eg, Dg, inv = gpu_score(torch, rsdock, prot, w, w.poses)
    Eo, Do, invo = oracle_score(rs_oracle, prot, w, w.poses)
    frac = compare(Eg, Dg, Eo, Do, inv, invo)
    assert frac > 0.99
    assert np.mean(Dg < w.sigma_vdw) > 0.5           # C1 is the clash-heavy config


def test_c1_host_pointers_and_async_agree(env):
    torch, rsdock, rs_oracle = env
    w = syn.config_c1()
    prot = build(rsdock, w)
    Ed, Dd, invd = gpu_score(torch, rsdock, prot, w, w.poses)
    Eh, Dh, invh = prot.score(w.ligand_q, w.ligand_xyz, w.poses)     # numpy: host path
    Ea, Da, inva = gpu_score(torch, rsdock, prot, w, w.poses, async_api=True)
    assert np.array_equal(Ed, Eh) and np.array_equal(Dd, Dh) and invd == invh
    assert np.array_equal(Ed, Ea) and np.array_equal(Dd, Da) and invd == inva


# ----------------------------------------------------------------------------- edge cases

def test_edge_cases(env):
    torch, rsdock, rs_oracle = env
    w = syn.random_small(seed=11, M=40, L=7, n=64, b=8.0, R=8, P=64)
    prot = build(rsdock, w)
    poses = w.poses.copy()
    poses[3, :4] = 0.0                      # zero quaternion
    poses[5, 4] = np.nan                    # NaN translation
    poses[7, 5] = 7.9                       # leaves the box
    poses[9, :4] = [2.0, 0.0, 0.0, 0.0]     # non-unit quaternion == identity
    poses[10, 4:] = [-7.0, 7.0, -7.0]       # far corner, valid or not by the rule
    Eg, Dg, inv = gpu_score(torch, rsdock, prot, w, poses)
    Eo, Do, invo = oracle_score(rs_oracle, prot, w, poses)
    compare(Eg, Dg, Eo, Do, inv, invo)
    assert np.isnan(Eg[[3, 5, 7]]).all() and inv >= 3
    # P = 0
    E0, D0, inv0 = gpu_score(torch, rsdock, prot, w, poses[:0])
    assert E0.size == 0 and inv0 == 0
    # L = 0: E = 0, d = +inf
    wl = syn.Workload(w.name, w.protein_xyz, w.protein_q, np.zeros((0, 3)), np.zeros(0), poses,
                      w.grid_n, w.box_half_width, w.rank_R, w.sigma_split, w.sigma_vdw, w.dmin_cap)
    E1, D1, inv1 = gpu_score(torch, rsdock, prot, wl, w.poses)
    assert np.all(E1 == 0.0) and np.all(np.isinf(D1)) and inv1 == 0
    # L = 1
    w1 = syn.Workload(w.name, w.protein_xyz, w.protein_q, np.zeros((1, 3)), np.array([0.7]),
                      w.poses, w.grid_n, w.box_half_width, w.rank_R, w.sigma_split, w.sigma_vdw,
                      w.dmin_cap)
    Eg, Dg, inv = gpu_score(torch, rsdock, prot, w1, w.poses)
    Eo, Do, invo = oracle_score(rs_oracle, prot, w1, w.poses)
    compare(Eg, Dg, Eo, Do, inv, invo)


def test_large_ligand_and_scattered_tiles(env):
    """L > 256 (ligand read from global memory) and tiles whose poses are far apart (the
    shared-memory window does not fit -> per-tile halving and the L2 fallback)."""
    torch, rsdock, rs_oracle = env
    rng = np.random.default_rng(4)
    w = syn.random_small(seed=12, M=60, L=5, n=256, b=16.0, R=16, P=300, trans=10.0)
    Y = syn.packed_ball(rng, 300, 4.0, 0.6)
    Y -= Y.mean(0)
    wl = syn.Workload("bigL", w.protein_xyz, w.protein_q, Y, rng.uniform(-1, 1, 300), w.poses,
                      w.grid_n, w.box_half_width, 16, w.sigma_split, w.sigma_vdw, w.dmin_cap)
    prot = build(rsdock, wl)
    Eg, Dg, inv = gpu_score(torch, rsdock, prot, wl, wl.poses)
    Eo, Do, invo = oracle_score(rs_oracle, prot, wl, wl.poses)
    compare(Eg, Dg, Eo, Do, inv, invo)
    # alternate two distant translations pose by pose
    poses = w.poses.copy()
    poses[0::2, 4:] = [-9.0, -9.0, -9.0]
    poses[1::2, 4:] = [9.0, 9.0, 9.0]
    Eg, Dg, inv = gpu_score(torch, rsdock, prot, w, poses)
    Eo, Do, invo = oracle_score(rs_oracle, prot, w, poses)
    compare(Eg, Dg, Eo, Do, inv, invo)


def test_order_invariance(env):
    """O9 freedoms: pose order and ligand atom order do not change a pose's result."""
    torch, rsdock, rs_oracle = env
    w = syn.config_c1(n_poses=400)
    prot = build(rsdock, w)
    E, D, _ = gpu_score(torch, rsdock, prot, w, w.poses)
    perm = np.random.default_rng(0).permutation(w.P)
    E2, D2, _ = gpu_score(torch, rsdock, prot, w, w.poses[perm])
    assert np.array_equal(E2, E[perm]) and np.array_equal(D2, D[perm])
    ap = np.random.default_rng(1).permutation(w.L)
    wa = syn.Workload(w.name, w.protein_xyz, w.protein_q, w.ligand_xyz[ap], w.ligand_q[ap],
                      w.poses, w.grid_n, w.box_half_width, w.rank_R, w.sigma_split, w.sigma_vdw,
                      w.dmin_cap)
    E3, D3, _ = gpu_score(torch, rsdock, prot, wa, w.poses)
    assert np.array_equal(D3, D)
    assert np.all(np.abs(E3 - E) <= 1e-14 * np.abs(E) + 1e-300)


def test_linearity_in_ligand_charges(env):
    torch, rsdock, rs_oracle = env
    w = syn.config_c1(n_poses=300)
    prot = build(rsdock, w)
    E, D, _ = gpu_score(torch, rsdock, prot, w, w.poses)
    w2 = syn.Workload(w.name, w.protein_xyz, w.protein_q, w.ligand_xyz, 2.0 * w.ligand_q, w.poses,
                      w.grid_n, w.box_half_width, w.rank_R, w.sigma_split, w.sigma_vdw, w.dmin_cap)
    E2, D2, _ = gpu_score(torch, rsdock, prot, w2, w.poses)
    assert np.array_equal(E2, 2.0 * E) and np.array_equal(D2, D)


def test_repeated_and_concurrent_streams(env):
    """Each launch takes a fresh dynamic-schedule work counter (stream-ordered reset): repeated
    calls and concurrent calls on two streams give the same bits as one synchronous call."""
    torch, rsdock, rs_oracle = env
    w = syn.config_c1()
    prot = build(rsdock, w)
    E0, D0, inv0 = gpu_score(torch, rsdock, prot, w, w.poses)
    dev = torch.device("cuda:0")
    q = torch.tensor(w.ligand_q, device=dev)
    y = torch.tensor(w.ligand_xyz, device=dev).contiguous()
    ps = torch.tensor(w.poses, device=dev).contiguous()
    h = w.P // 2
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for st in streams:
        st.wait_stream(torch.cuda.current_stream())
    for _ in range(3):
        outs = []
        for k, (lo, hi) in enumerate([(0, h), (h, w.P)]):
            E = torch.empty(hi - lo, dtype=torch.float64, device=dev)
            D = torch.empty(hi - lo, dtype=torch.float64, device=dev)
            cnt = torch.zeros(1, dtype=torch.int64, device=dev)
            streams[k].wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(streams[k]):
                prot.score_async(q, y, ps[lo:hi], E, D, cnt, stream=streams[k])
            outs.append((E, D, cnt))
        torch.cuda.synchronize()
        E = torch.cat([o[0] for o in outs]).cpu().numpy()
        D = torch.cat([o[1] for o in outs]).cpu().numpy()
        assert np.array_equal(E, E0) and np.array_equal(D, D0)
        assert sum(int(o[2].item()) for o in outs) == inv0


def test_many_unsynchronised_launches_on_streams(env):
    """100 launches in flight at once on three streams, none synchronised with another (more
    than any fixed pool of work counters): every launch has its own counter, so every output
    equals the one-call result bit for bit."""
    torch, rsdock, rs_oracle = env
    w = syn.config_c1()
    prot = build(rsdock, w)
    E0, D0, inv0 = gpu_score(torch, rsdock, prot, w, w.poses)
    dev = torch.device("cuda:0")
    q = torch.tensor(w.ligand_q, device=dev)
    y = torch.tensor(w.ligand_xyz, device=dev).contiguous()
    ps = torch.tensor(w.poses, device=dev).contiguous()
    streams = [torch.cuda.Stream() for _ in range(3)]
    for st in streams:
        st.wait_stream(torch.cuda.current_stream())
    outs = []
    for k in range(100):
        st = streams[k % 3]
        E = torch.empty(w.P, dtype=torch.float64, device=dev)
        D = torch.empty(w.P, dtype=torch.float64, device=dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        with torch.cuda.stream(st):
            prot.score_async(q, y, ps, E, D, cnt, stream=st)
        outs.append((E, D, cnt))
    torch.cuda.synchronize()
    for E, D, cnt in outs:
        assert np.array_equal(E.cpu().numpy(), E0) and np.array_equal(D.cpu().numpy(), D0)
        assert int(cnt.item()) == inv0


def test_ppiem_rejects_non_unit_directions(env):
    """A direction longer than 1 would let a step exceed the clearance: refused."""
    torch, rsdock, rs_oracle = env
    w = syn.config_c1(n_poses=4)
    prot = build(rsdock, w, dmin_cap=4.5)
    dirs, quats = syn.planar_scan(4, 2)
    centre = w.protein_xyz.mean(0)
    with pytest.raises(RuntimeError, match="unit vector"):
        rsdock.rs_ppiem_scan(prot.handle, w.ligand_q, w.ligand_xyz, centre, 1.5 * dirs, quats, 15.0)


# ----------------------------------------------------------------------------- physics on GPU

def test_tolerance_mode_gpu_vs_coulomb(env):
    """Tolerance-mode build (rank_R = 0, eps 1e-6, runtime-width kernel): parity with the
    oracle, and the GPU energies of non-clashing poses against brute-force Coulomb (Eq. (13))
    within the chain tolerance of SURVEY §8(c) (x S = sum |z z|/r)."""
    torch, rsdock, rs_oracle = env
    w0 = syn.config_c1()
    rng = np.random.default_rng(5)
    P = 60
    u = syn.unit_vectors(rng, P)
    poses = np.concatenate([syn.shoemake_quaternions(rng, P), u * rng.uniform(14, 16, (P, 1))], 1)
    w = w0.with_poses(poses)
    prot = build(rsdock, w, rank_R=0, eps_compress=1e-6)
    Eg, Dg, inv = gpu_score(torch, rsdock, prot, w, poses)
    Eo, Do, invo = oracle_score(rs_oracle, prot, w, poses)
    compare(Eg, Dg, Eo, Do, inv, invo)
    for p in range(P):
        R_ = rs_oracle.quat_to_rot(poses[p, :4])
        Xp = w.ligand_xyz @ R_.T + poses[p, 4:]
        S = rs_oracle.coulomb_scale(w.protein_xyz, w.protein_q, Xp, w.ligand_q)
        e = rs_oracle.coulomb_binding(w.protein_xyz, w.protein_q, Xp, w.ligand_q)
        assert abs(Eg[p] - e) <= 1e-3 * S


# ----------------------------------------------------------------------------- full sizes

def record(report, key, Eg, Dg, Eo, Do, asum, sigma):
    """M8 report row: sample size, bitwise-equal fraction of the energies,
    max relative difference, the condition number kappa = sum|addends| / |E| (oracle side)
    distribution, and the clash counts (d < sigma_vdW; none within 1e-9 A of sigma unless a
    test puts them there)."""
    ok = ~np.isnan(Eo)
    rel = np.abs(Eg[ok] - Eo[ok]) / np.maximum(np.abs(Eo[ok]), 1e-300)
    kap = asum[ok] / np.maximum(np.abs(Eo[ok]), 1e-300)
    q = (lambda a, f: float(np.quantile(a, f)) if a.size else None)
    report[key] = {
        "n": int(Eo.size), "valid": int(ok.sum()),
        "bitwise_frac": float(np.mean(Eg[ok] == Eo[ok])) if ok.any() else 1.0,
        "max_rel": float(rel.max()) if rel.size else 0.0,
        "kappa": {"median": q(kap, 0.5), "p99": q(kap, 0.99), "p999": q(kap, 0.999),
                  "max": float(kap.max()) if kap.size else None},
        "clash": int(np.sum(Do[ok] < sigma)),
        "near_sigma_1e9": int(np.sum(np.abs(Do[ok] - sigma) <= 1e-9)),
    }
    return report[key]


def sampled_parity(env, report, key, w, prot, k, seed):
    """The whole batch through the async API in the bench launch configuration; the oracle
    re-scores a seeded sample of k poses one by one (with its kappa)."""
    torch, rsdock, rs_oracle = env
    Eg, Dg, inv = gpu_score(torch, rsdock, prot, w, w.poses, async_api=True)
    idx, _ = syn.subsample(w.poses, k, seed=seed)
    tb = prot.export_tables()
    Eo, Do, invo, asum = rs_oracle.score_poses(tb, w.protein_xyz, w.protein_q, w.ligand_xyz,
                                               w.ligand_q, w.poses[idx], w.dmin_cap, abs_sum=True)
    compare(Eg[idx], Dg[idx], Eo, Do)
    assert inv == int(np.isnan(Eg).sum())
    return record(report, key, Eg[idx], Dg[idx], Eo, Do, asum, w.sigma_vdw)


@pytest.mark.parametrize("name,k", [("C2", 10000), ("C3", 10000)])
def test_full_size_sampled(env, parity_report, name, k):
    """Whole batch on the GPU in the bench launch configuration (async API, device tensors);
    the oracle re-scores a seeded sample of poses (M8 sizes: 10^4)."""
    torch, rsdock, rs_oracle = env
    w = syn.make(name)
    prot = build(rsdock, w)
    row = sampled_parity(env, parity_report, name, w, prot, k, 3)
    assert row["clash"] > 0 and row["valid"] > 0.9 * k


@pytest.mark.slow
def test_c4_full_size_sampled(env, parity_report):
    """C4: n = 16384, 50,000 atoms, R = 24 (L2 path: the ligand spans more rows than fit in
    shared memory), 10^7 poses on the GPU, 10^4 sampled poses re-scored by the oracle; the
    sample holds hundreds of clashing poses (C4's ~5% clash rate) on the L2 path."""
    torch, rsdock, rs_oracle = env
    w = syn.make("C4")
    prot = build(rsdock, w)
    assert prot.info["R"] == 24
    row = sampled_parity(env, parity_report, "C4", w, prot, 10000, 4)
    assert row["clash"] >= 100


@pytest.mark.slow
@pytest.mark.parametrize("R,mult", [(R, m) for R in (8, 16, 32) for m in (1, 2, 3)])
def test_c5_full_size_sampled(env, parity_report, R, mult):
    """C5 protein-protein, the whole R x sigma_s grid (R in {8, 16, 32}, sigma_s in {2, 4, 6} A):
    5000-atom rigid partner (ligand from global memory), n = 8192; 10^3 sampled poses per point."""
    torch, rsdock, rs_oracle = env
    w = syn.config_c5(rank_R=R, sigma_mult=mult)
    prot = build(rsdock, w)
    sampled_parity(env, parity_report, f"C5_R{R}_s{2 * mult}", w, prot, 1000, 5)


def test_snap_ties_on_cell_boundaries(env, parity_report):
    """H3/O3 ties: protein atoms, ligand atoms and translations on exact multiples of h, so
    with the identity and the axis half-turns (exact rotation matrices, O1) every transformed
    ligand coordinate falls exactly on a cell boundary (u = (x + b)/h an integer); the
    protein's cells (S4) tie too.  The kernel and the oracle must take the same side of every
    tie (A3: cell = ceil(u) - 1 clamped), so the results are compared element by element."""
    torch, rsdock, rs_oracle = env
    w0 = syn.random_small(seed=21, M=40, L=9, n=64, b=8.0, R=8, P=1)
    h = 2.0 * w0.box_half_width / w0.grid_n
    X = np.round(w0.protein_xyz / h) * h
    X = X[np.unique(X, axis=0, return_index=True)[1]]
    Y = np.round(w0.ligand_xyz / h) * h
    g = np.random.default_rng(5)
    halfturns = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 1, 0], [0, 0, 0, 1]], float)
    q = halfturns[g.integers(0, 4, 600)]
    t = np.round(g.uniform(-3.0, 3.0, (600, 3)) / h) * h
    poses = np.concatenate([q, t], axis=1)
    w = syn.Workload("ties", X, w0.protein_q[:X.shape[0]], Y, w0.ligand_q, poses, w0.grid_n,
                     w0.box_half_width, w0.rank_R, w0.sigma_split, w0.sigma_vdw, w0.dmin_cap)
    u = (w.protein_xyz + w.box_half_width) / h
    assert np.all(u == np.round(u))                       # protein atoms on boundaries
    prot = build(rsdock, w)
    Eg, Dg, inv = gpu_score(torch, rsdock, prot, w, poses)
    tb = prot.export_tables()
    Eo, Do, invo, asum = rs_oracle.score_poses(tb, X, w.protein_q, Y, w.ligand_q, poses,
                                               w.dmin_cap, abs_sum=True)
    compare(Eg, Dg, Eo, Do, inv, invo)
    row = record(parity_report, "snap_ties", Eg, Dg, Eo, Do, asum, w.sigma_vdw)
    assert row["valid"] > 500


def test_poses_at_vdw_and_cap_thresholds(env, parity_report):
    """H6 thresholds: poses whose closest ligand-protein pair sits at sigma_vdW +- 1e-9 A (the
    clash flag's edge, M8) and at D_cap +- 1e-9 A (the edge of the reported distance: +inf
    beyond, reading A11; this test builds with D_cap = 4 A so the two edges differ).  A one-atom ligand is placed along the outward radial
    direction of each of the 12 outermost protein atoms at the chosen distance (for the
    outermost atom no other atom is closer, so its poses sit exactly at the edge); the kernel
    must report the same distance bit for bit and the same inf/finite split."""
    torch, rsdock, rs_oracle = env
    w0 = syn.random_small(seed=31, M=40, L=3, n=64, b=8.0, R=8, P=1, protein_radius=2.5)
    X = w0.protein_xyz
    c = X.mean(0)
    Y = np.zeros((1, 3))                  # one atom: the pose's distance is the placed one
    eps = 1e-9
    dists = []
    for base in (w0.sigma_vdw, 4.0):
        dists += [base - eps, base, base + eps, base - 4 * eps, base + 4 * eps]
    poses = []
    for m in np.argsort(-np.linalg.norm(X - c, axis=1))[:12]:     # the outermost atoms
        u = (X[m] - c) / np.linalg.norm(X[m] - c)
        for d in dists:
            poses.append([1.0, 0.0, 0.0, 0.0, *(X[m] + d * u)])   # identity: x'_0 = t
    poses = np.array(poses)
    w = syn.Workload("thresholds", X, w0.protein_q, Y, w0.ligand_q[:1], poses, w0.grid_n,
                     w0.box_half_width, w0.rank_R, w0.sigma_split, w0.sigma_vdw, 4.0)
    prot = build(rsdock, w)
    Eg, Dg, inv = gpu_score(torch, rsdock, prot, w, poses)
    tb = prot.export_tables()
    Eo, Do, invo, asum = rs_oracle.score_poses(tb, X, w.protein_q, Y, w.ligand_q, poses,
                                               w.dmin_cap, abs_sum=True)
    compare(Eg, Dg, Eo, Do, inv, invo)
    row = record(parity_report, "vdw_cap_thresholds", Eg, Dg, Eo, Do, asum, w.sigma_vdw)
    assert row["near_sigma_1e9"] >= 3                       # poses really sit at the edge
    top = Do[len(dists) // 2:len(dists)]                    # outermost atom, at D_cap +- eps
    assert np.isfinite(top[[0, 3]]).all() and np.isinf(top[[2, 4]]).all()


# ----------------------------------------------------------------------------- fp32 factors (N5)

def _atom_scale(rs_oracle, prot, w, poses):
    """S_p = sum_l |z_l phi(x_l)| per pose (the north_star's scale for the fp32-factor variant),
    from the oracle with one-atom ligands."""
    tb = prot.export_tables()
    S = np.zeros(len(poses))
    for l in range(w.L):
        El, _, _ = rs_oracle.score_poses(tb, w.protein_xyz, w.protein_q, w.ligand_xyz[l:l + 1],
                                         w.ligand_q[l:l + 1], poses, w.dmin_cap)
        S += np.abs(El)
    return S


@pytest.mark.parametrize("name,k", [("C1", None), ("C2", 300), ("C3", 200)])
def test_f32_factors_parity_and_accuracy(env, name, k):
    """RS_FLAG_F32_FACTORS (reading A21): the kernel matches the O4-f32 oracle to the
    1e-12 parity bar, and stays within 1e-6 * sum_l |z_l phi(x_l)| of the binary64 path."""
    torch, rsdock, rs_oracle = env
    w = syn.make(name)
    prot32 = build(rsdock, w, flags=rsdock.RS_FLAG_F32_FACTORS)
    assert prot32.info["factor_bits"] == 32
    idx = None if k is None else syn.subsample(w.poses, k, seed=3)[0]
    poses = w.poses if idx is None else w.poses[idx]
    E32, D32, inv32 = gpu_score(torch, rsdock, prot32, w, poses)
    tb = prot32.export_tables()
    Eo, Do, invo = rs_oracle.score_poses(tb, w.protein_xyz, w.protein_q, w.ligand_xyz, w.ligand_q,
                                         poses, w.dmin_cap, f32=True)
    compare(E32, D32, Eo, Do, inv32, invo)
    E64, D64, _ = oracle_score(rs_oracle, prot32, w, poses)       # same tables, binary64 O4
    S = _atom_scale(rs_oracle, prot32, w, poses[:100])
    assert np.array_equal(D32, D64)
    assert np.all(np.abs(E32[:100] - E64[:100]) <= 1e-6 * S)


@pytest.mark.parametrize("R", [4, 8, 12, 16, 24, 32])
def test_f32_factors_all_widths(env, R):
    torch, rsdock, rs_oracle = env
    w = syn.random_small(seed=20 + R, M=40, L=20, n=64, b=8.0, R=R, P=333)
    prot = build(rsdock, w, flags=rsdock.RS_FLAG_F32_FACTORS)
    Eg, Dg, inv = gpu_score(torch, rsdock, prot, w, w.poses)
    tb = prot.export_tables()
    Eo, Do, invo = rs_oracle.score_poses(tb, w.protein_xyz, w.protein_q, w.ligand_xyz, w.ligand_q,
                                         w.poses, w.dmin_cap, f32=True)
    compare(Eg, Dg, Eo, Do, inv, invo)


# ----------------------------------------------------------------------------- forces (N1)

def gpu_forces(torch, prot, w, poses):
    dev = torch.device("cuda:0")
    q = torch.tensor(w.ligand_q, device=dev)
    y = torch.tensor(w.ligand_xyz, device=dev).contiguous()
    ps = torch.tensor(poses, device=dev).contiguous()
    out = torch.empty((ps.shape[0], 9), dtype=torch.float64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    prot.forces_async(q, y, ps, out, cnt)
    torch.cuda.synchronize()
    return out.cpu().numpy(), int(cnt.item())


def compare_forces(Fg, Fo, ig, io):
    assert ig == io
    assert np.array_equal(np.isnan(Fg), np.isnan(Fo))
    ok = ~np.isnan(Fo)
    scale = np.maximum(np.abs(Fo), 1e-300)
    # per component: bitwise expected; 1e-12 relative to the pose's largest component otherwise
    big = np.max(np.where(ok, np.abs(Fo), 0.0), axis=1, keepdims=True) * np.ones_like(Fo)
    assert np.all((Fg[ok] == Fo[ok]) | (np.abs(Fg[ok] - Fo[ok]) <= 1e-12 * big[ok])), \
        float(np.max(np.where(ok, np.abs(Fg - Fo) / scale, 0.0)))
    return float(np.mean(Fg[ok] == Fo[ok]))


@pytest.mark.parametrize("R", [4, 8, 12, 16, 24, 32, 10])
def test_forces_all_widths(env, R):
    """rs_score_forces (NEXT row N1) vs oracle_score_forces, every compiled width and a runtime
    width; invalid poses (zero quaternion, NaN, leaving the box) give NaN rows and are counted."""
    torch, rsdock, rs_oracle = env
    w = syn.random_small(seed=40 + R, M=40, L=20, n=64, b=8.0, R=R, P=333)
    prot = build(rsdock, w)
    poses = w.poses.copy()
    poses[3, :4] = 0.0
    poses[5, 4] = np.nan
    poses[7, 5] = 7.9
    Fg, ig = gpu_forces(torch, prot, w, poses)
    Fo, io = rs_oracle.score_forces(prot.export_tables(), w.ligand_xyz, w.ligand_q, poses)
    compare_forces(Fg, Fo, ig, io)
    assert np.isnan(Fg[[3, 5, 7]]).all() and ig >= 3


@pytest.mark.parametrize("name,k", [("C1", None), ("C3", 2000)])
def test_forces_configs(env, name, k):
    torch, rsdock, rs_oracle = env
    w = syn.make(name)
    prot = build(rsdock, w)
    poses = w.poses if k is None else w.poses[syn.subsample(w.poses, k, seed=9)[0]]
    Fg, ig = gpu_forces(torch, prot, w, poses)
    Fo, io = rs_oracle.score_forces(prot.export_tables(), w.ligand_xyz, w.ligand_q, poses)
    frac = compare_forces(Fg, Fo, ig, io)
    assert frac > 0.99


def test_forces_c3_contiguous_window(env):
    """The windowed force kernel on C3's launch order (16 translations x 1000 rotations,
    contiguous: each block restages its window per translation) against the oracle."""
    torch, rsdock, rs_oracle = env
    w = syn.config_c3()
    prot = build(rsdock, w)
    poses = w.poses[:16000]
    Fg, ig = gpu_forces(torch, prot, w, poses)
    Fo, io = rs_oracle.score_forces(prot.export_tables(), w.ligand_xyz, w.ligand_q, poses)
    assert compare_forces(Fg, Fo, ig, io) > 0.99


@pytest.mark.parametrize("R", [8, 16])
def test_forces_window_and_fallback_mix(env, R):
    """n = 2048 (h = 1/128 A): tiles of one translation fit the window, tiles of scattered
    translations do not and read L2; atoms beyond the window edge read L2 too."""
    torch, rsdock, rs_oracle = env
    w = syn.random_small(seed=60 + R, M=40, L=20, n=2048, b=8.0, R=R, P=400, trans=3.0)
    poses = w.poses.copy()
    poses[:200, 4:] = poses[0, 4:]                     # 200 poses at one translation
    prot = build(rsdock, w)
    Fg, ig = gpu_forces(torch, prot, w, poses)
    Fo, io = rs_oracle.score_forces(prot.export_tables(), w.ligand_xyz, w.ligand_q, poses)
    compare_forces(Fg, Fo, ig, io)


# ----------------------------------------------------------------------------- PPIEM scan (N2)

@pytest.mark.parametrize("mP,mL", [(12, 8), (5, 3)])
def test_ppiem_scan_matches_oracle(env, mP, mL):
    """rs_ppiem_scan (NEXT row N2, reading A23) vs the PPIEM oracle on C1 geometry with a
    D_cap > sigma build: the same statuses and contact distances bit for bit (the minimum
    distances are bitwise equal), energies within 1e-12, and the same landscape minima."""
    torch, rsdock, rs_oracle = env
    from oracle import ppiem_oracle as po
    w = syn.config_c1(n_poses=4)
    prot = build(rsdock, w, dmin_cap=4.5)
    dirs, quats = syn.planar_scan(mP, mL)
    centre = w.protein_xyz.mean(0)
    s_start = float(np.max(np.linalg.norm(w.protein_xyz - centre, axis=1)) + 6.0)
    E, s, st = rsdock.rs_ppiem_scan(prot.handle, w.ligand_q, w.ligand_xyz, centre, dirs, quats,
                                    s_start, tol=1e-3, max_iter=64)
    Eo, so, sto = po.scan(prot.export_tables(), w.protein_xyz, w.protein_q, w.ligand_xyz,
                          w.ligand_q, centre, dirs, quats, s_start, w.sigma_vdw, 4.5, 1e-3, 64)
    assert np.array_equal(st, sto)
    assert np.array_equal(s, so)
    ok = ~np.isnan(Eo)
    assert np.array_equal(np.isnan(E), np.isnan(Eo))
    assert np.all(np.abs(E[ok] - Eo[ok]) <= 1e-12 * np.abs(Eo[ok]) + 1e-300)
    assert (st == 0).mean() > 0.9
    assert list(rsdock.rs_landscape_minima(E, 10)) == list(po.landscape_minima(Eo, 10))


def test_ppiem_scan_statuses(env):
    """Every status of rs_ppiem_scan against the oracle: 2 (clash at the start: s_start inside
    the protein), 1 (a ligand atom leaves the box: s_start beyond b), 3 (the line misses the
    protein, s goes below 0: the centre is offset from a small protein), 4 (max_iter reached)."""
    torch, rsdock, rs_oracle = env
    from oracle import ppiem_oracle as po
    w = syn.random_small(seed=77, M=12, L=6, n=64, b=8.0, R=8, P=4, protein_radius=1.5)
    prot = build(rsdock, w, dmin_cap=4.0, sigma_vdw=1.5)
    dirs, quats = syn.planar_scan(6, 2)
    tb = prot.export_tables()
    cases = [(w.protein_xyz.mean(0), 0.5, 64),                   # clash at the start
             (w.protein_xyz.mean(0), 9.0, 64),                   # starts outside the box
             (w.protein_xyz.mean(0) + [0.0, 0.0, 3.5], 4.0, 64),  # lines above the protein
             (w.protein_xyz.mean(0), 6.0, 1)]                    # one iteration only
    seen = set()
    for centre, s0, it in cases:
        E, s, st = rsdock.rs_ppiem_scan(prot.handle, w.ligand_q, w.ligand_xyz, centre, dirs, quats,
                                        s0, tol=1e-3, max_iter=it)
        Eo, so, sto = po.scan(tb, w.protein_xyz, w.protein_q, w.ligand_xyz, w.ligand_q, centre,
                              dirs, quats, s0, 1.5, 4.0, 1e-3, it)
        assert np.array_equal(st, sto) and np.array_equal(s, so)
        assert np.array_equal(np.isnan(E), np.isnan(Eo))
        ok = ~np.isnan(Eo)
        assert np.all(np.abs(E[ok] - Eo[ok]) <= 1e-12 * np.abs(Eo[ok]) + 1e-300)
        seen |= set(np.unique(st).tolist())
    assert {1, 2, 3, 4} <= seen


def test_window_too_small_takes_l2_path(env):
    """A ligand whose rows for one translation exceed the shared memory left for the window
    (n = 4096 grid, 5.6 A ligand radius): the launch falls back to the L2 path for the whole
    batch instead of one-pose tiles; results still match the oracle."""
    torch, rsdock, rs_oracle = env
    rng = np.random.default_rng(31)
    X = syn.packed_ball(rng, 80, 6.0, 1.2)
    q = rng.uniform(-1, 1, 80)
    Y = syn.packed_ball(rng, 40, 5.6, 1.2)
    Y -= Y.mean(0)
    Y *= 5.6 / np.max(np.linalg.norm(Y, axis=1))
    P = 150
    poses = np.concatenate([syn.shoemake_quaternions(rng, P), rng.uniform(-12, 12, (P, 3))], 1)
    w = syn.Workload("bigwin", X, q, Y, rng.uniform(-1, 1, 40), poses, 4096, 64.0, 16)
    prot = build(rsdock, w)
    Eg, Dg, inv = gpu_score(torch, rsdock, prot, w, w.poses)
    Eo, Do, invo = oracle_score(rs_oracle, prot, w, w.poses)
    compare(Eg, Dg, Eo, Do, inv, invo)


# ----------------------------------------------------------------------------- N4: Eq. (23) complex

def _complex(rsdock, w, R=(4, 8), flags=0):
    parts = syn.complex_parts(w)
    prm = dict(w.params())
    prots = [rsdock.Protein(q, X, w.box_half_width, **dict(prm, rank_R=r,
                                                           flags=rsdock.RS_FLAG_HOST_ONLY))
             for (X, q), r in zip(parts, R)]
    return parts, prots, rsdock.Protein.combine(prots, flags=flags)


@pytest.mark.parametrize("seed,R", [(0, (4, 8)), (1, (8, 8)), (2, (12, 12)), (3, (5, 6))])
def test_complex_parity(env, seed, R):
    """rs_combine_proteins (reading A24): the kernel on the combined handle matches the oracle on
    the concatenated tables (1e-12, D bitwise) for compiled and runtime widths, and the literal
    Eq. (23) sum over the proteins, sum_p E_p (oracle.score_complex), within the dd bound."""
    torch, rsdock, rs_oracle = env
    w = syn.complex_small(seed=seed, P=333)
    parts, prots, C = _complex(rsdock, w, R)
    Eg, Dg, inv = gpu_score(torch, rsdock, C, w, w.poses)
    tabs = [p.export_tables() for p in prots]
    comb = rs_oracle.combine_tables(tabs)
    Xu = np.concatenate([X for X, _ in parts])
    qu = np.concatenate([q for _, q in parts])
    Eo, Do, invo = rs_oracle.score_poses(comb, Xu, qu, w.ligand_xyz, w.ligand_q, w.poses,
                                         w.dmin_cap)
    compare(Eg, Dg, Eo, Do, inv, invo)
    Es, Ds, _ = rs_oracle.score_complex(tabs, parts, w.ligand_xyz, w.ligand_q, w.poses, w.dmin_cap)
    ok = ~np.isnan(Eo)
    assert np.array_equal(Dg[ok], Ds[ok])
    scale = sum(np.abs(rs_oracle.score_poses(t, X, q, w.ligand_xyz, w.ligand_q, w.poses,
                                             w.dmin_cap)[0]) for t, (X, q) in zip(tabs, parts))
    assert np.all(np.abs(Eg[ok] - Es[ok]) <= 1e-13 * np.maximum(scale[ok], 1e-300))


def test_complex_f32_parity(env):
    torch, rsdock, rs_oracle = env
    w = syn.complex_small(seed=5, P=257)
    parts, prots, C = _complex(rsdock, w, (8, 8), flags=rsdock.RS_FLAG_F32_FACTORS)
    assert C.info["factor_bits"] == 32
    Eg, Dg, inv = gpu_score(torch, rsdock, C, w, w.poses)
    comb = rs_oracle.combine_tables([p.export_tables() for p in prots])
    Xu = np.concatenate([X for X, _ in parts])
    qu = np.concatenate([q for _, q in parts])
    Eo, Do, invo = rs_oracle.score_poses(comb, Xu, qu, w.ligand_xyz, w.ligand_q, w.poses,
                                         w.dmin_cap, f32=True)
    compare(Eg, Dg, Eo, Do, inv, invo)


def test_complex_mid_size_sample(env):
    """A 700 + 500-atom complex at n = 256 (several windows of tiles, 20,000 poses in one launch),
    a seeded sample of poses scored by the oracle one by one."""
    torch, rsdock, rs_oracle = env
    w = syn.complex_small(seed=7, M=(700, 500), L=24, n=256, b=24.0, R=8, P=20000, radius=7.0,
                          trans=14.0)
    parts, prots, C = _complex(rsdock, w, (8, 8))
    Eg, Dg, inv = gpu_score(torch, rsdock, C, w, w.poses)
    idx, _ = syn.subsample(w.poses, 600)
    comb = rs_oracle.combine_tables([p.export_tables() for p in prots])
    Xu = np.concatenate([X for X, _ in parts])
    qu = np.concatenate([q for _, q in parts])
    Eo, Do, _ = rs_oracle.score_poses(comb, Xu, qu, w.ligand_xyz, w.ligand_q, w.poses[idx],
                                      w.dmin_cap)
    compare(Eg[idx], Dg[idx], Eo, Do)


# ----------------------------------------------------------------------------- N3: box restriction

def _site_poses(w, centre, spread, P, seed):
    rng = np.random.default_rng(seed)
    quats = syn.shoemake_quaternions(rng, P)
    return np.concatenate([quats, centre + rng.uniform(-spread, spread, (P, 3))], axis=1)


def _box_cells(w, lo_x, hi_x):
    inv_h = w.grid_n / (2 * w.box_half_width)
    lo = np.clip(np.ceil((lo_x + w.box_half_width) * inv_h) - 1, 0, w.grid_n - 1).astype(np.int32)
    hi = np.clip(np.ceil((hi_x + w.box_half_width) * inv_h) - 1, 0, w.grid_n - 1).astype(np.int32)
    return lo, hi


@pytest.mark.parametrize("R,f32,scheme_b", [(4, False, False), (8, False, False), (6, False, False),
                                            (8, True, False), (8, False, True), (4, True, True)])
def test_restricted_box_parity(env, R, f32, scheme_b):
    """rs_restrict_box (reading A25): the kernel on the box handle matches the oracle on its
    exported tables; poses with an atom outside the box give NaN on both sides, their minimum
    distance still bitwise equal."""
    torch, rsdock, rs_oracle = env
    w = syn.config_c1()
    parent = build(rsdock, w, rank_R=0, eps_compress=1e-4, flags=rsdock.RS_FLAG_HOST_ONLY)
    c = w.protein_xyz.mean(0) + np.array([12.0, 0.0, 0.0])
    rl = float(np.linalg.norm(w.ligand_xyz, axis=1).max())
    lo, hi = _box_cells(w, c - 2.0 - rl, c + 2.0 + rl)
    box = parent.restrict_box(lo, hi, R, flags=(rsdock.RS_FLAG_F32_FACTORS if f32 else 0) |
                              (rsdock.RS_FLAG_BOX_SCHEME_B if scheme_b else 0))
    poses = _site_poses(w, c, 3.0, 517, seed=R)
    Eg, Dg, inv = gpu_score(torch, rsdock, box, w, poses)
    Eo, Do, invo = rs_oracle.score_poses(box.export_tables(), w.protein_xyz, w.protein_q,
                                         w.ligand_xyz, w.ligand_q, poses, w.dmin_cap, f32=f32)
    compare(Eg, Dg, Eo, Do, inv, invo)
    assert np.array_equal(Dg, Do, equal_nan=True)
    nan = np.isnan(Eg)
    assert 0.1 < nan.mean() < 0.9                      # both kinds present


def test_restricted_box_c2_site_sample(env):
    """C2's docking site (1000-translation lattice x 100 rotations) on a box handle of width 8
    from a parent with a rank-64 Tucker form: the full 10^5-pose launch, a seeded sample against the oracle;
    every pose lies inside the box, so no energy is NaN."""
    torch, rsdock, rs_oracle = env
    w = syn.config_c2()
    parent = build(rsdock, w, eps_compress=1e-4, tucker_rank_max=64,
                   flags=rsdock.RS_FLAG_HOST_ONLY)
    rl = float(np.linalg.norm(w.ligand_xyz, axis=1).max())
    t = w.poses[:, 4:]
    lo, hi = _box_cells(w, t.min(0) - rl - 0.5, t.max(0) + rl + 0.5)
    box = parent.restrict_box(lo, hi, 8)
    Eg, Dg, inv = gpu_score(torch, rsdock, box, w, w.poses)
    assert not np.isnan(Eg).any()
    idx, sample = syn.subsample(w.poses, 300)
    Eo, Do, _ = rs_oracle.score_poses(box.export_tables(), w.protein_xyz, w.protein_q,
                                      w.ligand_xyz, w.ligand_q, sample, w.dmin_cap)
    compare(Eg[idx], Dg[idx], Eo, Do)


def test_shards_concatenate_bitwise(env):
    """§8(e): the G-way sharded outputs (shard.shard_bounds, each shard its own launch)
    concatenate to the 1-launch output bit for bit (per-pose arithmetic never depends on the
    tiling, chunking or launch)."""
    torch, rsdock, rs_oracle = env
    from paper_2510_26611_b200.shard import shard_bounds
    w = syn.config_c2()
    prot = build(rsdock, w)
    poses = w.poses[:30011]
    E, D, inv = gpu_score(torch, rsdock, prot, w, poses)
    for G in (2, 3, 8):
        parts = [gpu_score(torch, rsdock, prot, w, poses[a:b])
                 for a, b in (shard_bounds(len(poses), G, r) for r in range(G))]
        assert np.array_equal(np.concatenate([p[0] for p in parts]), E, equal_nan=True)
        assert np.array_equal(np.concatenate([p[1] for p in parts]), D, equal_nan=True)
        assert sum(p[2] for p in parts) == inv


# ----------------------------------------------------------------------------- maximum sizes

def test_max_grid_no_window(env):
    """n = 32768 (the largest grid; cells need all 15 bits of the packed entries), h = 1/256 A:
    n_sigma = 256 (a 136 MB short-range memo); a translation's rows exceed shared memory, so
    H4 reads L2."""
    torch, rsdock, rs_oracle = env
    w = syn.random_small(seed=90, M=60, L=12, n=32768, b=64.0, R=8, P=200, protein_radius=4.0,
                         trans=3.0)
    prot = build(rsdock, w)
    assert prot.info["n_sigma"] == 256
    Eg, Dg, inv = gpu_score(torch, rsdock, prot, w, w.poses)
    Eo, Do, invo = oracle_score(rs_oracle, prot, w, w.poses)
    compare(Eg, Dg, Eo, Do, inv, invo)


def test_large_ligand_beyond_smem_staging(env):
    """L = 300 ligand atoms (more than the 256 a windowed launch stages in shared memory: the
    rest read L2) with the whole factor set in the window; R = 16 and a runtime width."""
    torch, rsdock, rs_oracle = env
    import dataclasses
    rng = np.random.default_rng(5)
    Y = syn.ligand_body(rng, 300)
    Y = Y - Y.mean(0)
    for R in (16, 10):
        w = syn.random_small(seed=91, M=40, L=7, n=64, b=12.0, R=R, P=150, trans=2.0)
        w = dataclasses.replace(w, ligand_xyz=Y, ligand_q=rng.uniform(-1, 1, 300))
        prot = build(rsdock, w)
        Eg, Dg, inv = gpu_score(torch, rsdock, prot, w, w.poses)
        Eo, Do, invo = oracle_score(rs_oracle, prot, w, w.poses)
        compare(Eg, Dg, Eo, Do, inv, invo)
        Fg, ig = gpu_forces(torch, prot, w, w.poses)
        Fo, io = rs_oracle.score_forces(prot.export_tables(), w.ligand_xyz, w.ligand_q, w.poses)
        compare_forces(Fg, Fo, ig, io)


@pytest.mark.parametrize("name,k", [("C2", None), ("C3", 450000)])
def test_streamed_host_pipeline_bitwise(env, name, k):
    """rs_score_poses on pinned host buffers (P >= 4e5, C3 here: one launch that waits for each pose
    chunk's arrival flag while the copies land, per-chunk completion counters releasing the
    result copies; C2: the per-chunk launches) returns exactly the device-resident launch's
    outputs."""
    torch, rsdock, rs_oracle = env
    w = syn.make(name)
    poses = w.poses if k is None else np.ascontiguousarray(w.poses[:k])
    prot = build(rsdock, w)
    Ed, Dd, invd = gpu_score(torch, rsdock, prot, w, poses, async_api=True)
    hp = torch.from_numpy(poses).pin_memory()
    hE = torch.empty(len(poses), dtype=torch.float64).pin_memory()
    hD = torch.empty(len(poses), dtype=torch.float64).pin_memory()
    for _ in range(3):
        hE.fill_(0.0)
        inv = rsdock.rs_score_poses(prot.handle, w.ligand_q, w.ligand_xyz, w.L, hp, len(poses), hE, hD)
        assert inv == invd
        assert np.array_equal(hE.numpy(), Ed, equal_nan=True)
        assert np.array_equal(hD.numpy(), Dd, equal_nan=True)
    # pageable numpy buffers take the same path (copies staged by the driver)
    Eh, Dh, invh = prot.score(w.ligand_q, w.ligand_xyz, poses)
    assert invh == invd and np.array_equal(Eh, Ed, equal_nan=True)
    assert np.array_equal(Dh, Dd, equal_nan=True)


@pytest.mark.parametrize("R", [12, 24, 16])
def test_f32_no_window_l2_path(env, R):
    """The fp32-factor variant without a window (n = 8192, h = 1/256 A: a translation's rows
    exceed shared memory): H4 reads the binary32 rows from L2, only the quads that hold ranks
    (R = 12, 24 pad to 4, 8 quads) -- against the O4-f32 oracle."""
    torch, rsdock, rs_oracle = env
    w = syn.random_small(seed=95 + R, M=50, L=10, n=8192, b=16.0, R=R, P=300, trans=3.0)
    prot = build(rsdock, w, flags=rsdock.RS_FLAG_F32_FACTORS)
    Eg, Dg, inv = gpu_score(torch, rsdock, prot, w, w.poses)
    Eo, Do, invo = rs_oracle.score_poses(prot.export_tables(), w.protein_xyz, w.protein_q,
                                         w.ligand_xyz, w.ligand_q, w.poses, w.dmin_cap, f32=True)
    compare(Eg, Dg, Eo, Do, inv, invo)


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_device_core_setup_bitwise(env, name):
    """S6 on the device (setup_device.cu, N4 part): a handle built with a device and the host
    convolutions (RS_FLAG_HOST_FFT) forms the Tucker core there with the host loop's exact op
    sequence, so its exported tables are bitwise the host-only build's."""
    torch, rsdock, rs_oracle = env
    w = syn.make(name)
    dev = build(rsdock, w, flags=rsdock.RS_FLAG_HOST_FFT)
    host = build(rsdock, w, flags=rsdock.RS_FLAG_HOST_ONLY)
    td, th = dev.export_tables(), host.export_tables()
    for k in ("F1", "F2", "F3", "S1", "S2", "S3"):
        assert np.array_equal(td[k], th[k]), k
    assert dev.info["cp_core_err"] == host.info["cp_core_err"]


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_device_fft_setup(env, name):
    """The default device build (N4 part): the RHOSVD and core convolutions with cuFFT.  The CP it builds
    agrees with the host-only build's at sampled cells to 1e-6 of their max (the FFT rounding
    moves the randomized bases, not the accuracy: the same sampled error to 1e-3 relative), and
    the kernel on its tables matches the oracle as always."""
    torch, rsdock, rs_oracle = env
    w = syn.make(name)
    host = build(rsdock, w, flags=rsdock.RS_FLAG_HOST_ONLY)
    dev = build(rsdock, w)
    th, td = host.export_tables(), dev.export_tables()
    rng = np.random.default_rng(3)
    idx = rng.integers(0, w.grid_n, size=(2000, 3))
    vh = np.einsum("pk,pk,pk->p", th["F1"][idx[:, 0]], th["F2"][idx[:, 1]], th["F3"][idx[:, 2]])
    vd = np.einsum("pk,pk,pk->p", td["F1"][idx[:, 0]], td["F2"][idx[:, 1]], td["F3"][idx[:, 2]])
    assert np.max(np.abs(vh - vd)) <= 1e-6 * np.max(np.abs(vh))
    assert abs(dev.info["sampled_max_err"] - host.info["sampled_max_err"]) <= 1e-3 * host.info["sampled_max_err"]
    ks, sample = syn.subsample(w.poses, 300)
    Eg, Dg, inv = gpu_score(torch, rsdock, dev, w, sample)
    Eo, Do, invo = oracle_score(rs_oracle, dev, w, sample)
    compare(Eg, Dg, Eo, Do, inv, invo)


@pytest.mark.parametrize("name,k", [("C1", 1000), ("C2", 2000)])
def test_tucker_eval_matches_oracle(env, name, k):
    """RS_FLAG_TUCKER_EVAL (NEXT row N5, reading A26): the fused kernel with the long range from
    the Tucker form (rows of the RHOSVD bases from L2, core in shared memory) matches the
    oracle's O4-T scorer pose by pose (1e-12, distances bitwise), the plan reports the Tucker
    path, and a saved / reloaded handle keeps scoring the same."""
    torch, rsdock, rs_oracle = env
    w = syn.make(name)
    prot = build(rsdock, w, flags=rsdock.RS_FLAG_TUCKER_EVAL)
    assert rsdock.rs_score_path(prot.handle, w.ligand_xyz) == rsdock.RS_PATH_TUCKER
    _, sample = syn.subsample(w.poses, k)
    Eg, Dg, inv = gpu_score(torch, rsdock, prot, w, sample)
    Eo, Do, invo = rs_oracle.score_poses(prot.export_tables(), w.protein_xyz, w.protein_q,
                                         w.ligand_xyz, w.ligand_q, sample, w.dmin_cap,
                                         tucker=prot.export_tucker())
    compare(Eg, Dg, Eo, Do, inv, invo)

