"""Multi-GPU ECM stage 1: curves shard across ranks, one gather of the per-curve results.

Curves are independent, so rank r of W takes the contiguous curve range
[r*C/W, (r+1)*C/W) and runs ecm_stage1_batch on its own GPU with no communication.  The only
exchange step is at the end: an all-gather of the uint8 status per curve
(padded to equal shard sizes) and of a compacted list (curve index, g) of the curves that found
a proper factor.  With NCCL over NVLink these are KB-sized messages; the same code runs under
gloo on CPU tensors for the world-size-2 tests (the per-shard compute is injectable there).
"""
from __future__ import annotations

import numpy as np


def shard_bounds(count: int, rank: int, world: int) -> tuple[int, int]:
    return rank * count // world, (rank + 1) * count // world


def _default_compute(N, L, B1, sigmas_shard):
    from . import ecm_stage1_batch
    return ecm_stage1_batch(N, L, B1, sigmas_shard, want=("g",))


def ecm_stage1_distributed(N: int, L: int, B1: int, sigmas, *, group=None, compute=None, device=None):
    """Run this rank's shard of `sigmas` (the FULL per-job seed array, host numpy) and gather.

    Returns (status, factors): status is a uint8 tensor of all `count` curves in curve order
    (identical on every rank), factors a list of (curve_index, g_int) for status-1 curves.
    `compute(N, L, B1, sigma_tensor) -> {"status": u8[count_local], "g": u32[count_local, L]}`.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    sig = np.asarray(sigmas, dtype=np.uint64)
    count = sig.size
    lo, hi = shard_bounds(count, rank, world)
    # the shard is computed on this rank's GPU (or wherever `compute` wants it); the gather runs
    # on `device` (the NCCL device by default, CPU tensors under gloo)
    compute_dev = "cuda" if (compute is None and torch.cuda.is_available()) else "cpu"
    device = device or ("cuda" if torch.cuda.is_available() else "cpu")
    local = torch.from_numpy(sig[lo:hi].copy()).to(compute_dev)
    res = (compute or _default_compute)(N, L, B1, local)
    st = res["status"].to(device)
    g = res["g"]
    if g.dtype == torch.uint32:
        g = g.to(torch.int64)
    g = g.to(device)
    if world == 1:
        status = st
        idx = torch.nonzero(st == 1).flatten()
        return status, [(int(i), _limbs_to_int(g[i])) for i in idx.tolist()]
    # 1) statuses, padded to the largest shard
    shard = (count + world - 1) // world
    pad = torch.zeros(shard, dtype=torch.uint8, device=device)
    pad[: hi - lo] = st
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    status = torch.cat([parts[r][: shard_bounds(count, r, world)[1] - shard_bounds(count, r, world)[0]]
                        for r in range(world)])
    # 2) compacted (index, g) of found factors, capacity = max flagged count over ranks
    idx = torch.nonzero(st == 1).flatten()
    nf = torch.tensor([idx.numel()], dtype=torch.int64, device=device)
    dist.all_reduce(nf, op=dist.ReduceOp.MAX, group=group)
    cap = int(nf.item())
    factors = []
    if cap:
        rec = torch.full((cap, 1 + L), -1, dtype=torch.int64, device=device)
        if idx.numel():
            rec[: idx.numel(), 0] = idx.to(torch.int64) + lo
            rec[: idx.numel(), 1:] = g[idx].to(torch.int64)
        recs = [torch.empty_like(rec) for _ in range(world)]
        dist.all_gather(recs, rec, group=group)
        for r in recs:
            for row in r.cpu().numpy():
                if row[0] >= 0:
                    factors.append((int(row[0]), sum(int(w) << (32 * j) for j, w in enumerate(row[1:]))))
    return status, sorted(factors)


def _limbs_to_int(row) -> int:
    return sum(int(w) << (32 * j) for j, w in enumerate(row.cpu().numpy().astype(np.uint64)))
