"""Multi-GPU pose sharding: poses are independent units, so N ranks (one
process per GPU, torch.distributed) each score a contiguous slice with their own replica of
the protein handle.  No collective touches the data path; results are all-gathered only when
a consumer asks for them (gather=True)."""
from __future__ import annotations


def shard_bounds(P: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of P poses for `rank`; the first P % world ranks get one more."""
    if world <= 0 or not (0 <= rank < world) or P < 0:
        raise ValueError("bad shard arguments")
    q, r = divmod(P, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def score_sharded(score_fn, poses, group=None, gather: bool = False):
    """Score this rank's slice of the global pose array with `score_fn(poses) -> (E, D, inv)`.

    Returns (E_local, D_local, invalid_total, (lo, hi)) or, with gather=True, the global E and D
    (rank order == pose order) on every rank.  Works with any torch.distributed backend (NCCL on
    GPUs, gloo on CPU); tensors are moved to the backend's device as needed."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_bounds(int(poses.shape[0]), world, rank)
    E, D, inv = score_fn(poses[lo:hi])
    E = torch.as_tensor(E)
    D = torch.as_tensor(D)
    if world == 1:
        return (E, D, int(inv), (lo, hi))
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    cnt = torch.tensor([int(inv)], dtype=torch.int64, device=dev)
    dist.all_reduce(cnt, group=group)
    if not gather:
        return (E, D, int(cnt.item()), (lo, hi))
    P = int(poses.shape[0])
    n_max = P // world + (1 if P % world else 0)
    pad = torch.full((2, n_max), float("nan"), dtype=torch.float64, device=dev)
    pad[0, : hi - lo] = E.to(dev)
    pad[1, : hi - lo] = D.to(dev)
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    Es, Ds = [], []
    for r, t in enumerate(parts):
        a, b = shard_bounds(P, world, r)
        Es.append(t[0, : b - a])
        Ds.append(t[1, : b - a])
    return (torch.cat(Es), torch.cat(Ds), int(cnt.item()), (0, P))


def ppiem_sharded(scan_fn, dirs, quats, minima_fn=None, top_k: int = 0, group=None):
    """PPIEM over N ranks (Algorithm PPIEM): the m_P
    positions (rows of the landscape) are split into contiguous slices, each rank scans its
    rows against every orientation with `scan_fn(dirs_slice, quats) -> (E, s, status)` (the
    rs_ppiem_scan call on its own device), and one all-gather assembles the m_P x m_L landscape
    on every rank: the minima search (A6) needs it whole, since its 8-neighbourhood wraps around
    the row index across slice boundaries.  Every trajectory is independent, so the gathered
    landscape is bitwise the 1-rank result.  Returns (E, s, status, minima or None)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    m_P, m_L = int(dirs.shape[0]), int(quats.shape[0])
    lo, hi = shard_bounds(m_P, world, rank)
    if hi > lo:
        E, s, st = scan_fn(np.ascontiguousarray(dirs[lo:hi]), quats)
    else:
        E, s, st = (np.empty((0, m_L)), np.empty((0, m_L)), np.empty((0, m_L), dtype=np.int32))
    if world > 1:
        backend = dist.get_backend(group)
        dev = (torch.device("cuda", torch.cuda.current_device()) if backend == "nccl"
               else torch.device("cpu"))
        rows = m_P // world + (1 if m_P % world else 0)
        pad = torch.full((3, rows, m_L), float("nan"), dtype=torch.float64, device=dev)
        pad[0, : hi - lo] = torch.as_tensor(np.asarray(E, dtype=np.float64))
        pad[1, : hi - lo] = torch.as_tensor(np.asarray(s, dtype=np.float64))
        pad[2, : hi - lo] = torch.as_tensor(np.asarray(st, dtype=np.float64))
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
        blocks = []
        for r, t in enumerate(parts):
            a, b = shard_bounds(m_P, world, r)
            blocks.append(t[:, : b - a].cpu().numpy())
        full = np.concatenate(blocks, axis=1)
        E, s, st = full[0], full[1], full[2].astype(np.int32)
    mins = minima_fn(E, top_k) if minima_fn is not None and top_k > 0 else None
    return E, s, st, mins
