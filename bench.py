#!/usr/bin/env python
"""Benchmark of the RS-tensor pose-rescoring hot path (Algorithm PLIE + Eq. (22)) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl reference]

One "step" = one pass of the whole hot path (H1-H8) over the config's full pose batch
(C3: 10^6 poses x 60 atoms, n = 4096, R = 16), inputs resident in HBM, through the C ABI
(rs_score_poses_async on device tensors).  L2 is flushed (256 MiB write) between timed
steps, outside the timed events.  Prints ONE JSON line on rank 0.

Multi-GPU (torchrun, one process per GPU): poses are independent units, so each rank scores
its own batch with its own replica of the protein handle and no data-path collective
("scaling": "weak"); the step time is the max over ranks (NCCL all-reduce of the timings).

--impl reference times the oracle (oracle/, plain scalar C, OpenMP over poses) on the host
cores on a bounded sample of the same workload (rank 0 only)."""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "poses/sec and ligand-atom evals/sec at 1 B200; fraction of FP64/L2 roofline"


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return json.load(f)
    except OSError:
        return {}


def run_microbench():
    exe = os.path.join(ROOT, "tools", "microbench")
    if not os.path.exists(exe):
        return None
    try:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=120).stdout
        return json.loads(out.strip().splitlines()[-1])
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                "sw_power_cap"), f[4:8]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def load_workload(name, pose_stream=0, **kw):
    from synth import configs as syn
    return syn.make(name, pose_stream=pose_stream, **kw)


def workload_kw(args):
    """C5's sweep point (BASELINE: R in {8, 16, 32} x short-range cutoff {1, 2, 3} x default)."""
    if args.config == "C5":
        return {"rank_R": args.c5_rank, "sigma_mult": args.c5_sigma_mult}
    return {}


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(n):
    """`bench.py --gpus N` outside a launcher: re-run this command under torch.distributed.run
    with N processes on this node (one per GPU, rendezvous on 127.0.0.1); rank 0 prints the
    line.  Returns the launcher's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)]
    cmd += sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")            # communicator init lines (nranks) on stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(cmd, env=env)


def rank_batch(args, world, rank):
    """This rank's poses: weak scaling -- an independent batch of the config's size per rank
    (pose_stream = rank; rank 0 holds the canonical batch); strong scaling -- the contiguous
    slice shard_bounds(P, world, rank) of the one canonical batch (translation tiles stay
    compact).  Returns (workload, lo, hi, global P)."""
    from paper_2510_26611_b200.shard import shard_bounds
    if args.scaling == "weak":
        w = load_workload(args.config, pose_stream=rank, **workload_kw(args))
        return w, 0, w.P, w.P * world
    w = load_workload(args.config, **workload_kw(args))
    lo, hi = shard_bounds(w.P, world, rank)
    return w, lo, hi, w.P


def bench_dry_run(args):
    """The multi-rank plumbing of the bench without a GPU (gloo): per-rank batches, barrier,
    max-over-ranks step time, rank-0 line.  For the CPU tests of the launcher."""
    import hashlib
    import torch
    world, rank = _env_int("WORLD_SIZE", 1), _env_int("RANK", 0)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    w, lo, hi, Pg = rank_batch(args, world, rank)
    digest = int(hashlib.sha1(np.ascontiguousarray(w.poses[lo:hi]).tobytes()).hexdigest()[:12], 16)
    ms = torch.tensor([1.0 + 0.25 * rank], dtype=torch.float64)      # stand-in per-rank times
    digests = [torch.tensor([digest], dtype=torch.int64) for _ in range(world)]
    if dist:
        dist.barrier()
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        dist.all_gather(digests, torch.tensor([digest], dtype=torch.int64))
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "scaling": args.scaling,
                          "ms_per_step": float(ms.item()),
                          "value": Pg / (float(ms.item()) * 1e-3), "poses_per_rank": hi - lo,
                          "global_poses": Pg, "rank_digests": [int(d.item()) for d in digests]}),
              flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def cpu_reference_rate(w, tables, budget_s=12.0, max_poses=200000, seed=7, f32=False, tucker=None):
    """Time the oracle (as it stands) on a bounded seeded sample of the workload's poses."""
    from oracle import rs_oracle
    from synth import configs as syn
    _, probe = syn.subsample(w.poses, 64, seed=seed)
    t0 = time.perf_counter()
    rs_oracle.score_poses(tables, w.protein_xyz, w.protein_q, w.ligand_xyz, w.ligand_q, probe,
                          w.dmin_cap, f32=f32, tucker=tucker)
    dt = time.perf_counter() - t0
    k = int(min(max_poses, max(64, 64 * budget_s / max(dt, 1e-6))))
    idx, sample = syn.subsample(w.poses, k, seed=seed + 1)
    t0 = time.perf_counter()
    rs_oracle.score_poses(tables, w.protein_xyz, w.protein_q, w.ligand_xyz, w.ligand_q, sample,
                          w.dmin_cap, f32=f32, tucker=tucker)
    dt = time.perf_counter() - t0
    return k, dt, rs_oracle.num_threads()


def impl_reference(args):
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0
    w = load_workload(args.config, **workload_kw(args))
    from paper_2510_26611_b200 import rsdock
    flags = 0
    try:
        import torch
        if not torch.cuda.is_available():
            flags = rsdock.RS_FLAG_HOST_ONLY
    except Exception:
        flags = rsdock.RS_FLAG_HOST_ONLY
    prot = rsdock.Protein(w.protein_q, w.protein_xyz, w.box_half_width, **w.params(), flags=flags)
    tables = prot.export_tables()
    from oracle import rs_oracle
    from synth import configs as syn
    per_step = max(16, args.ref_poses)
    times = []
    for s in range(args.warmup + args.steps):
        _, sample = syn.subsample(w.poses, per_step, seed=100 + s)
        t0 = time.perf_counter()
        rs_oracle.score_poses(tables, w.protein_xyz, w.protein_q, w.ligand_xyz, w.ligand_q, sample,
                              w.dmin_cap)
        if s >= args.warmup:
            times.append(time.perf_counter() - t0)
    t = float(np.sum(times))
    val = per_step * args.steps / t
    cores = rs_oracle.num_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "poses/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "atom_evals_per_s": val * w.L,
        "config": config_dict(w, args),
        "cpu_baseline": {"value": val, "unit": "poses/s", "cores": cores, "kind": "oracle",
                         "sample": f"{per_step} seeded poses of {w.name} per step "
                                   f"(brute-force short-range/vdW over all {w.M} protein atoms)"},
        "e2e": {"value": val, "unit": "poses/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(w, args):
    return {"workload": f"{w.name}: protein M={w.M}, ligand L={w.L}, grid n={w.grid_n}, "
                        f"box b={w.box_half_width}, R={w.rank_R}, P={w.P} poses",
            "config": args.config, "M": w.M, "L": w.L, "n": w.grid_n, "R": w.rank_R,
            "poses": w.P, "sigma_split": w.sigma_split, "sigma_vdw": w.sigma_vdw,
            "parallelism": (f"dp{_env_int('WORLD_SIZE', 1)}: " +
                            ("an independent pose batch per rank" if getattr(args, "scaling", "weak") == "weak"
                             else "the batch split into contiguous slices") +
                            ", replicated handle, no data-path collective"),
            "mode": ("forces (rs_score_forces, N1)" if getattr(args, "forces", False) else "energy + mindist")
                    + (", fp32 factors (A21)" if getattr(args, "f32", False) else "")
                    + (", Tucker-format evaluation (N5, A26)" if getattr(args, "tucker", False) else "")
                    + (", Eq. (23) complex: 2 proteins x R/2, rank-concatenated (A24)"
                       if getattr(args, "complex", False) else "")
                    + (f", box-restricted width {args.box}, scheme "
                       f"({getattr(args, 'box_scheme', 'b').upper()}) (N3, A25)"
                       if getattr(args, "box", 0) else ""),
            "l2": "flushed between timed steps (256 MiB write, outside the events)"}


def bench_ppiem(args):
    """PPIEM scan (rs_ppiem_scan, reading A23) on the config's protein and ligand: planar grid of
    M positions x M self-rotations, approach to vdW contact by sphere tracing on the device
    (D_cap = sigma + 2 A), landscape and minima.  Wall time of the synchronous call.  Under
    torchrun the positions are split over the ranks (shard.ppiem_sharded: one all-gather of the
    landscape rows, minima on the whole landscape); the time is the max over ranks."""
    import torch
    from paper_2510_26611_b200 import rsdock
    from paper_2510_26611_b200.shard import ppiem_sharded
    from synth import configs as syn
    import __graft_entry__
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        dist_mod.init_process_group("nccl", device_id=dev)
        dist = dist_mod
    if rank == 0:
        __graft_entry__.build_library()
    if dist:
        dist.barrier()
    w = load_workload(args.config, **workload_kw(args))
    prm = dict(w.params())
    prm["dmin_cap"] = w.sigma_vdw + 2.0
    prot = rsdock.Protein(w.protein_q, w.protein_xyz, w.box_half_width, **prm, device=local)
    dirs, quats = syn.planar_scan(args.ppiem, args.ppiem)
    centre = w.protein_xyz.mean(0)
    rl = float(np.max(np.linalg.norm(w.ligand_xyz, axis=1)))
    s_start = float(np.max(np.linalg.norm(w.protein_xyz - centre, axis=1))) + rl + 3.0
    s_start = min(s_start, w.box_half_width - rl - 1.0)
    q = torch.tensor(w.ligand_q, device=dev)
    y = torch.tensor(w.ligand_xyz, device=dev).contiguous()

    def scan(d, qs):
        return rsdock.rs_ppiem_scan(prot.handle, q, y, centre, d, qs, s_start)

    ppiem_sharded(scan, dirs, quats)                                         # warm-up
    times = []
    for _ in range(max(1, args.steps)):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        E, sv, st, mins = ppiem_sharded(scan, dirs, quats, rsdock.rs_landscape_minima, 10)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if dist:
            tt = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        times.append(dt)
    t = float(np.median(times))
    if rank == 0:
        line = {"metric": "PPIEM scan landscape entries/s (approach + energy)", "value": E.size / t,
                "unit": "entries/s", "n_gpus": world, "steps": len(times), "ms_per_scan": 1e3 * t,
                "higher_is_better": True, "scaling": "strong", "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": w.name, "m_P": args.ppiem, "m_L": args.ppiem,
                           "s_start": s_start, "dmin_cap": prm["dmin_cap"],
                           "parallelism": f"positions split over {world} rank(s), one all-gather"},
                "status_counts": {str(k): int((st == k).sum()) for k in range(5)},
                "best": [{"j": int(i // args.ppiem), "k": int(i % args.ppiem),
                          "E": float(E.flat[i]), "s": float(sv.flat[i])} for i in mins[:3]]}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--c5-rank", type=int, default=16, choices=[8, 16, 32],
                    help="C5 sweep: CP width R")
    ap.add_argument("--c5-sigma-mult", type=int, default=1, choices=[1, 2, 3],
                    help="C5 sweep: short-range cutoff sigma_s = k x 2 A")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-poses", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-microbench", action="store_true")
    ap.add_argument("--ppiem", type=int, default=0, metavar="M",
                    help="time a PPIEM scan (NEXT row N2) with M positions x M self-rotations")
    ap.add_argument("--forces", action="store_true",
                    help="time rs_score_forces (NEXT row N1) instead of the energy path")
    ap.add_argument("--box", type=int, default=0, metavar="R_PI",
                    help="score on a box-restricted handle of width R_PI covering the poses "
                         "(N3, scheme (C): rs_restrict_box)")
    ap.add_argument("--box-scheme", default="b", choices=["b", "c"],
                    help="N3 scheme: (B) new RHOSVD over the box rows, or (C) from a rank-64 "
                         "Tucker form of the whole potential")
    ap.add_argument("--complex", action="store_true",
                    help="build the config's protein as a two-protein complex (Eq. (23), N4): "
                         "one RS tensor of width R/2 per protein, rank-concatenated")
    ap.add_argument("--tucker", action="store_true",
                    help="Tucker-format evaluation of the long range (RS_FLAG_TUCKER_EVAL, NEXT row N5)")
    ap.add_argument("--f32", action="store_true",
                    help="the fp32-factor variant (RS_FLAG_F32_FACTORS, DESIGN.md reading A21)")
    ap.add_argument("--nbr-cell", type=float, default=0.0,
                    help="edge [A] of the neighbour-list cells (0 = the library's automatic choice)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: an independent batch of the config's size per rank; strong: the "
                         "one batch split into contiguous slices over the ranks")
    ap.add_argument("--dry-run", action="store_true",
                    help="the multi-rank plumbing only (gloo, no GPU): per-rank batches, max-over-"
                         "ranks timing, rank-0 line (used by the CPU tests)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.dry_run:
        return bench_dry_run(args)
    if args.impl == "reference":
        return impl_reference(args)
    if args.ppiem:
        return bench_ppiem(args)

    import torch
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        dist_mod.init_process_group("nccl", device_id=dev)
        dist = dist_mod

    import __graft_entry__
    if rank == 0:
        __graft_entry__.build_library()        # one rank (re)builds if stale; the others wait
    if dist:
        dist.barrier()
    from paper_2510_26611_b200 import rsdock

    w, lo, hi, P_global = rank_batch(args, world, rank)
    if rank == 0 and dist:
        print(f"bench: NCCL communicator initialised, nranks={world}, scaling={args.scaling}",
              file=sys.stderr, flush=True)
    ncpu = os.cpu_count() or 1
    t0 = time.perf_counter()
    fl = (rsdock.RS_FLAG_F32_FACTORS if args.f32 else 0) | (rsdock.RS_FLAG_TUCKER_EVAL if args.tucker else 0)
    box_info = None
    if args.complex:
        # NEXT row N4 (Eq. (23)): one RS tensor per protein (R/2 each), combined on the device
        from synth import configs as syn
        prm = dict(w.params(), rank_R=w.rank_R // 2)
        parts = [rsdock.Protein(qp, Xp, w.box_half_width, **prm, device=local,
                                n_threads=max(1, ncpu // max(world, 1)), nbr_cell=args.nbr_cell,
                                flags=rsdock.RS_FLAG_HOST_ONLY)
                 for Xp, qp in syn.complex_parts(w)]
        prot = rsdock.Protein.combine(parts, flags=fl)
        del parts
    elif args.box:
        # NEXT row N3: the box that covers every pose's atoms, width args.box; scheme (B) (a new
        # RHOSVD over the box rows, from the ordinary handle) or (C) (from a parent with a
        # rank-64 Tucker form)
        scheme_b = args.box_scheme == "b"
        parent = rsdock.Protein(w.protein_q, w.protein_xyz, w.box_half_width, **w.params(),
                                tucker_rank_max=0 if scheme_b else 64, device=local,
                                n_threads=max(1, ncpu // max(world, 1)), nbr_cell=args.nbr_cell,
                                flags=rsdock.RS_FLAG_HOST_ONLY)
        rl = float(np.linalg.norm(w.ligand_xyz, axis=1).max())
        tr = w.poses[:, 4:]
        inv_h = w.grid_n / (2 * w.box_half_width)
        cell = lambda x: np.clip(np.ceil((x + w.box_half_width) * inv_h) - 1, 0, w.grid_n - 1)
        blo = cell(tr.min(0) - rl - 0.5).astype(np.int32)
        bhi = cell(tr.max(0) + rl + 0.5).astype(np.int32)
        t1 = time.perf_counter()
        prot = parent.restrict_box(blo, bhi, args.box,
                                   flags=fl | (rsdock.RS_FLAG_BOX_SCHEME_B if scheme_b else 0))
        box_info = {"scheme": args.box_scheme.upper(), "restrict_seconds": time.perf_counter() - t1,
                    "lo": blo.tolist(), "hi": bhi.tolist(), "R_pi": args.box,
                    "box_cp_core_err": prot.info["cp_core_err"],
                    "parent_cp_core_err": parent.info["cp_core_err"],
                    "parent_sampled_max_err": parent.info["sampled_max_err"],
                    "parent_tucker_r": parent.info["tucker_r"]}
        del parent
    else:
        prot = rsdock.Protein(w.protein_q, w.protein_xyz, w.box_half_width, **w.params(),
                              device=local, n_threads=max(1, ncpu // max(world, 1)),
                              nbr_cell=args.nbr_cell, flags=fl)
    setup_s = time.perf_counter() - t0
    info = prot.info

    q = torch.tensor(w.ligand_q, device=dev)
    y = torch.tensor(w.ligand_xyz, device=dev).contiguous()
    poses = torch.tensor(w.poses[lo:hi], device=dev).contiguous()
    P, L = hi - lo, w.L
    E = torch.empty(P, dtype=torch.float64, device=dev)
    D = torch.empty(P, dtype=torch.float64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    Fout = torch.empty((P, 9), dtype=torch.float64, device=dev) if args.forces else None

    def step():
        if args.forces:
            prot.forces_async(q, y, poses, Fout, cnt, stream=stream)
        else:
            prot.score_async(q, y, poses, E, D, cnt, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(np.sum(step_ms))
    if dist:
        tt = torch.tensor([total_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms = total_ms / args.steps
    value = P_global / (ms * 1e-3)           # every rank's poses / the slowest rank's time
    invalid = int(cnt.item())

    # end to end through the same C ABI with pinned HOST buffers (copies inside the call)
    e2e = None
    if not args.no_e2e:
        hp = torch.from_numpy(np.ascontiguousarray(w.poses[lo:hi])).pin_memory()
        hq = torch.from_numpy(w.ligand_q).pin_memory()
        hy = torch.from_numpy(np.ascontiguousarray(w.ligand_xyz)).pin_memory()
        hE = torch.empty(P, dtype=torch.float64).pin_memory()
        hD = torch.empty(P, dtype=torch.float64).pin_memory()
        rsdock.rs_score_poses(prot.handle, hq, hy, L, hp, P, hE, hD)
        tl = []
        for _ in range(max(3, min(args.steps, 5))):
            t1 = time.perf_counter()
            rsdock.rs_score_poses(prot.handle, hq, hy, L, hp, P, hE, hD)
            tl.append(time.perf_counter() - t1)
        te = float(np.median(tl))
        if dist:
            tt = torch.tensor([te], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        # the pinned host-to-device copy rate of this box (the pose upload bounds e2e)
        dbuf = torch.empty_like(hp, device=dev)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        hts = []
        for _ in range(3):
            ev0.record()
            dbuf.copy_(hp, non_blocking=True)
            ev1.record()
            torch.cuda.synchronize()
            hts.append(ev0.elapsed_time(ev1) * 1e-3)
        h2d_gbs = hp.numel() * 8 / min(hts) / 1e9
        del dbuf
        e2e = {"value": P_global / te, "unit": "poses/s",
               "h2d_bytes_per_step": int(P * 7 * 8 + L * 4 * 8), "d2h_bytes_per_step": int(P * 2 * 8),
               "h2d_pinned_gbs": h2d_gbs,
               "upload_bound_poses_per_s": world * h2d_gbs * 1e9 / 56.0,
               "path": "rs_score_poses, pinned host buffers: one launch streaming behind chunked H2D (arrival flags), per-chunk D2H released by completion counters"}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0

    mb = None if args.no_microbench else run_microbench()
    peaks = _peaks()
    R = info["R"]
    fbytes = 4.0 if args.f32 else 8.0
    # H4: 3 rows x R factors per atom evaluation; forces (N1): 6 rows (phi(i), phi(i - e_a))
    rows = 6.0 if args.forces else 3.0
    gather_bytes = rows * fbytes * R * P * L
    t_s = ms * 1e-3
    achieved = gather_bytes / t_s / 1e9
    smem_peak = mb.get("lds128_random_row_rotated_gbs") if mb else None
    l2_peak = mb.get("l2_gather_cg_9p4MB_gbs") if mb else None          # L2 service rate, C4 size
    l2_peak_c3 = mb.get("l2_gather_cg_1p6MB_gbs") if mb else None       # the same at C3's size
    fp64_rate = mb.get("dfma_instr_per_s") if mb else None
    dp_instr = ((0.0 if args.f32 else 3.0 * R) + 25.0) * P * L   # 2R DMUL + R DADD + ~25 per atom
    if args.forces:
        dp_instr = (12.0 * R + 80.0) * P * L      # four values (8R DMUL + 4R DADD) + resultants
    # the variant the library runs for this ligand: a shared-memory window of the tile's rows
    # (bound: shared-memory bandwidth) or rows from L2 (bound: L2 gather bandwidth)
    path = rsdock.RS_PATH_WINDOW if args.forces else rsdock.rs_score_path(prot.handle, w.ligand_xyz)
    on_l2 = path != rsdock.RS_PATH_WINDOW
    peak = l2_peak if on_l2 else smem_peak
    traffic = None
    tfile = os.path.join(ROOT, "profiles", f"ncu_traffic_{args.config}.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    if args.tucker:
        # N5: the Tucker contraction is FP64 issue (2 r0 r1 r2 + 2 r0 r1 + 2 r0 DMUL/DADD per atom)
        tr = info["tucker_r"]
        dp_instr = (2.0 * tr[0] * tr[1] * tr[2] + 2.0 * tr[0] * tr[1] + 2.0 * tr[0] + 25.0) * P * L
    roofline = {
        "bound": "l2" if on_l2 else "smem", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": (achieved / peak) if peak else None, "traffic": traffic,
        "kernel": (f"force_window_kernel<{R}>" if R in (4, 8, 16, 32) else f"force_kernel<{R}>")
                  if args.forces else f"score_kernel<{R}>" + (" (L2 rows)" if on_l2 else " (smem window)"),
        "peak_source": ("tools/microbench (same run): random 32-byte-sector row gathers with "
                        "ld.global.cg (L2 only) over a 9.4 MB table, 148 SMs" if on_l2 else
                        "tools/microbench (same run): conflict-free random-row LDS.128 "
                        "(lane-rotated chunks), 148 SMs"),
        "algorithmic_bytes_per_launch": gather_bytes,
        "fp64_frac": (dp_instr / t_s / fp64_rate) if fp64_rate else None,
        "l2_literal_frac": (achieved / (l2_peak if on_l2 else l2_peak_c3)) if (l2_peak and l2_peak_c3) else None,
        "hbm_peak_measured_gbs": peaks.get("hbm_gbs"),
    }
    if args.tucker:
        roofline.update({"bound": "fp64", "achieved": dp_instr / t_s / 1e9,
                         "peak": fp64_rate / 1e9 if fp64_rate else None, "unit": "G DP instr/s",
                         "frac": (dp_instr / t_s / fp64_rate) if fp64_rate else None,
                         "kernel": "score_kernel<Tucker>",
                         "peak_source": "tools/microbench (same run): DFMA issue rate, 148 SMs",
                         "algorithmic_dp_instr_per_launch": dp_instr})
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        k, dt, cores = cpu_reference_rate(w, prot.export_tables(), f32=args.f32,
                                          tucker=prot.export_tucker() if args.tucker else None)
        cpu = {"value": k / dt, "unit": "poses/s", "cores": cores, "kind": "oracle",
               "sample": f"{k} seeded poses of {w.name} ({dt:.1f} s; brute-force short-range/vdW "
                         f"over all {w.M} protein atoms)"}
    line = {
        "metric": METRIC, "value": value, "unit": "poses/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f32-factors/f64" if args.f32 else "f64",
        "data": "synthetic", "atom_evals_per_s": value * L,
        "config": config_dict(w, args),
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": args.steps, "clocks": clk.summary(),
        "invalid_poses": invalid, "setup_seconds": setup_s,
        "setup": {k: info[k] for k in ("R", "tucker_r", "quad_K", "R_long_ref", "R_short",
                                       "n_sigma", "sampled_max_err", "sampled_rms_err",
                                       "cp_core_err", "nbr_entries", "device_bytes")},
        "step_ms_min": float(np.min(step_ms)), "step_ms_max": float(np.max(step_ms)),
    }
    if box_info:
        line["box"] = box_info
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
