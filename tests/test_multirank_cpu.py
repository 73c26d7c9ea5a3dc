"""World-size-2 gloo tests of the multi-GPU host logic (pose sharding + gather), on CPU: the
per-rank scorer is the oracle, so the test exercises exactly the sharding/gather code the GPU
path uses, without a GPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_26611_b200.shard import ppiem_sharded, score_sharded, shard_bounds
from synth import configs as syn


def test_shard_bounds_partition():
    for P in (0, 1, 7, 64, 1000, 1001):
        for world in (1, 2, 3, 8):
            got = [shard_bounds(P, world, r) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == P
            assert all(got[i][1] == got[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in got]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import rs_oracle
    w = syn.random_small(seed=21, M=30, L=6, n=32, b=8.0, R=4, P=101)
    rng = np.random.default_rng(0)
    tb = dict(n=32, b=8.0, R=4, F1=rng.normal(size=(32, 4)), F2=rng.normal(size=(32, 4)),
              F3=rng.normal(size=(32, 4)), n_sigma=2, S1=rng.normal(size=(5, 3)),
              S2=rng.normal(size=(5, 3)), S3=rng.normal(size=(5, 3)))
    poses = w.poses.copy()
    poses[5, :4] = 0.0                      # one invalid pose (in rank 0's shard)
    poses[77, 4] = 50.0                     # one invalid pose (in rank 1's shard)

    def score(ps):
        return rs_oracle.score_poses(tb, w.protein_xyz, w.protein_q, w.ligand_xyz, w.ligand_q,
                                     np.ascontiguousarray(ps), 1.5)

    E, D, inv, rng_ = score_sharded(score, poses, gather=True)
    E1, D1, inv1 = score(poses)
    ok = (np.array_equal(E.numpy(), E1, equal_nan=True) and
          np.array_equal(D.numpy(), D1, equal_nan=True) and inv == inv1 == 2)
    El, Dl, invl, (lo, hi) = score_sharded(score, poses, gather=False)
    ok = ok and np.array_equal(El.numpy(), E1[lo:hi], equal_nan=True) and invl == 2
    out[rank] = bool(ok)
    dist.destroy_process_group()


def test_sharded_scoring_gloo_world2():
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] and out[1]


def _ppiem_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import ppiem_oracle as po
    from oracle import rs_oracle
    w = syn.random_small(seed=31, M=30, L=5, n=64, b=10.0, R=4, P=1)
    rng = np.random.default_rng(3)
    tb = dict(n=64, b=10.0, R=4, F1=rng.normal(size=(64, 4)) * 0.1, F2=rng.normal(size=(64, 4)),
              F3=rng.normal(size=(64, 4)), n_sigma=2, S1=rng.normal(size=(5, 3)) * 0.1,
              S2=rng.normal(size=(5, 3)), S3=rng.normal(size=(5, 3)))
    dirs, quats = syn.planar_scan(7, 4)
    centre = w.protein_xyz.mean(0)
    args = (tb, w.protein_xyz, w.protein_q, w.ligand_xyz, w.ligand_q, centre)

    def scan(d, q):
        return po.scan(*args, d, q, 7.0, 1.0, 2.5, 1e-3, 40)

    E, s, st, mins = ppiem_sharded(scan, dirs, quats, po.landscape_minima, 5)
    E1, s1, st1 = scan(dirs, quats)
    ok = (np.array_equal(E, E1, equal_nan=True) and np.array_equal(s, s1) and
          np.array_equal(st, st1) and list(mins) == list(po.landscape_minima(E1, 5)) and
          (st1 == 0).sum() > 0)
    out[rank] = bool(ok)
    dist.destroy_process_group()


def test_ppiem_sharded_gloo_world2():
    """PPIEM rows split over two ranks (7 positions: 4 + 3), one all-gather: the landscape,
    distances, statuses and minima equal the 1-rank scan bit for bit."""
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_ppiem_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] and out[1]


def _run_bench(*extra):
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    env.pop("LOCAL_RANK", None)
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--dry-run", *extra],
                         capture_output=True, text=True, env=env, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    import json
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_launcher_weak_scaling_spawns_ranks():
    """`bench.py --gpus 2` outside a launcher re-runs itself under torch.distributed.run with 2
    ranks (gloo here): each rank scores an independent batch of the config's size, the step
    time is the max over ranks, the value counts every rank's poses, one line from rank 0."""
    d = _run_bench("--gpus", "2", "--config", "C1")
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["ms_per_step"] == 1.25                       # max of the ranks' stand-in times
    assert d["global_poses"] == 2 * d["poses_per_rank"] == 2000
    assert len(set(d["rank_digests"])) == 2               # independent batches


def test_bench_launcher_strong_scaling_splits_one_batch():
    d = _run_bench("--gpus", "2", "--config", "C1", "--scaling", "strong")
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["global_poses"] == 1000 and d["poses_per_rank"] == 500
    assert len(set(d["rank_digests"])) == 2
    one = _run_bench("--config", "C1", "--scaling", "strong")
    assert one["n_gpus"] == 1 and one["global_poses"] == 1000
