#!/usr/bin/env python
"""Small invocations of every device path of librsdock.so, for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck, one tool per run):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py [CASE ...]

Cases: window (C1, shared-memory window, device and async API), stream (the streamed host
pipeline: one launch spinning on copy-engine arrival flags, per-chunk completion counters; the
threshold lowered with RS_STREAM_MIN_POSES), chunked (host buffers below the threshold), l2
(C5 geometry: rows from L2), runtime (an uncompiled width), f32 (binary32 factors), forces
(window and L2 force kernels), ppiem (the approach loop), memo (the device fill of the
short-range memo and setup S6 run inside every build).  Prints one line per case."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("RS_STREAM_MIN_POSES", "1000")


def main(cases):
    import torch
    from paper_2510_26611_b200 import rsdock
    from synth import configs as syn
    dev = torch.device("cuda:0")

    def build(w, **kw):
        prm = dict(w.params())
        prm.update(kw)
        return rsdock.Protein(w.protein_q, w.protein_xyz, w.box_half_width, **prm)

    def device_score(prot, w, poses):
        q = torch.tensor(w.ligand_q, device=dev)
        y = torch.tensor(w.ligand_xyz, device=dev).contiguous()
        ps = torch.tensor(poses, device=dev).contiguous()
        E = torch.empty(len(poses), dtype=torch.float64, device=dev)
        D = torch.empty_like(E)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        prot.score_async(q, y, ps, E, D, cnt)
        inv = rsdock.rs_score_poses(prot.handle, q, y, w.L, ps, len(poses), E, D)
        torch.cuda.synchronize()
        return E.cpu().numpy(), inv

    def host_score(prot, w, poses):
        E = np.empty(len(poses))
        D = np.empty(len(poses))
        inv = rsdock.rs_score_poses(prot.handle, w.ligand_q, w.ligand_xyz, w.L,
                                    np.ascontiguousarray(poses), len(poses), E, D)
        return E, inv

    w1 = syn.config_c1(n_poses=1000)
    for case in cases:
        if case == "window":
            prot = build(w1)
            E, inv = device_score(prot, w1, w1.poses)
        elif case == "stream":
            prot = build(w1)
            poses = np.tile(w1.poses, (5, 1))          # 5000 >= RS_STREAM_MIN_POSES: streamed
            E, inv = host_score(prot, w1, poses)
        elif case == "chunked":
            prot = build(w1)
            E, inv = host_score(prot, w1, w1.poses[:600])
        elif case == "l2":
            w = syn.config_c5(rank_R=8, sigma_mult=1, n_poses=48)
            prot = build(w)
            assert rsdock.rs_score_path(prot.handle, w.ligand_xyz) == rsdock.RS_PATH_L2
            E, inv = device_score(prot, w, w.poses)
        elif case == "runtime":
            w = syn.random_small(seed=2, M=40, L=9, n=64, b=8.0, R=10, P=200)
            prot = build(w)
            E, inv = device_score(prot, w, w.poses)
        elif case == "f32":
            prot = build(w1, flags=rsdock.RS_FLAG_F32_FACTORS)
            E, inv = device_score(prot, w1, w1.poses)
        elif case == "forces":
            prot = build(w1)
            for R, w in ((8, w1), (10, syn.random_small(seed=4, M=40, L=9, n=64, b=8.0, R=10, P=100))):
                p = prot if R == 8 else build(w)
                q = torch.tensor(w.ligand_q, device=dev)
                y = torch.tensor(w.ligand_xyz, device=dev).contiguous()
                ps = torch.tensor(w.poses, device=dev).contiguous()
                F = torch.empty((len(w.poses), 9), dtype=torch.float64, device=dev)
                cnt = torch.zeros(1, dtype=torch.int64, device=dev)
                p.forces_async(q, y, ps, F, cnt)
            torch.cuda.synchronize()
            E, inv = F[:, 0].cpu().numpy(), int(cnt.item())
        elif case == "ppiem":
            w = syn.config_c1(n_poses=4)
            prot = build(w, dmin_cap=4.5)
            dirs, quats = syn.planar_scan(8, 4)
            centre = w.protein_xyz.mean(0)
            s0 = float(np.max(np.linalg.norm(w.protein_xyz - centre, axis=1)) + 6.0)
            E, s, st = rsdock.rs_ppiem_scan(prot.handle, w.ligand_q, w.ligand_xyz, centre, dirs,
                                            quats, s0, tol=1e-3, max_iter=64)
            inv = int(np.sum(st != 0))
        elif case == "memo":
            w = syn.config_c2(n_rot=1)
            prot = build(w)
            E, inv = device_score(prot, w, w.poses[:200])
        else:
            raise SystemExit(f"unknown case {case}")
        print(f"case {case}: {E.size} results, {int(np.sum(np.isnan(E)))} NaN, invalid {inv}, "
              f"finite sum {float(np.nansum(E)):.6e}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["window", "stream", "chunked", "l2", "runtime", "f32", "forces",
                          "ppiem", "memo"])
