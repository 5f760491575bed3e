"""Multi-GPU ECM stage 1: curves shard across ranks, one gather of the per-curve results.

Curves are independent, so rank r of W takes the contiguous curve range
[r*C/W, (r+1)*C/W) and runs ecm_stage1_batch on its own GPU with no communication.  The only
exchange step is at the end, two fixed-size all-gathers enqueued back to back
on the stream the shard ran on, with no host synchronisation between them:

  1. the uint8 status of every curve (`all_gather_into_tensor`, shards padded to ceil(C/W));
  2. a fixed-capacity compacted list of the curves that found a proper factor (status 1, or 4
     = the setup gcd was a proper factor): row 0 = (number of such curves on the rank, 0, ...),
     rows 1..cap = (global curve index, g limbs).  The compaction runs on the device (prefix sum
     + scatter, fixed shapes), so nothing waits for the host.

After both collectives each rank reads the gathered counts once; only if some rank found more
factors than the capacity (never at the paper's configs: ~1 % of curves) does a second, exact
gather run.  Rank 0 decodes the records into Python integers; the other ranks return the device
tensors only.  With NCCL over NVLink the messages are KB-sized; the same code runs under gloo on
CPU tensors for the world-size-2 tests (the per-shard compute is injectable there).
"""
from __future__ import annotations

import numpy as np

FACTOR_STATUSES = (1, 4)  # ECM_CURVE_FACTOR, ECM_CURVE_SETUP_FACTOR


def shard_bounds(count: int, rank: int, world: int) -> tuple[int, int]:
    return rank * count // world, (rank + 1) * count // world


def default_capacity(shard: int) -> int:
    """Records per rank in the fixed-capacity gather: 1/64 of the shard (the paper-shaped configs
    flag < 1 %: C3 ≈ 0.8 %, C5 ≈ 0.3 %), at least 64."""
    return max(64, -(-shard // 64))


def _default_compute(N, L, B1, sigmas_shard):
    from . import ecm_stage1_batch
    return ecm_stage1_batch(N, L, B1, sigmas_shard, want=("g",))


def compact_factors(st, g, lo: int, cap: int):
    """Fixed-shape, device-side compaction (no host sync): returns an int64 tensor of shape
    (cap + 1, 1 + L) — row 0 holds the number of factor-finding curves in this shard, rows 1..
    the first `cap` of them as (global index lo + i, g_i limbs); unused rows are -1."""
    import torch
    L = g.shape[1]
    dev = st.device
    flag = (st == FACTOR_STATUSES[0]) | (st == FACTOR_STATUSES[1])
    n = flag.to(torch.int64).sum()
    pos = torch.cumsum(flag.to(torch.int64), 0)  # 1-based row of each flagged curve
    keep = flag & (pos <= cap)
    row = torch.where(keep, pos, torch.zeros_like(pos))  # row 0 collects the rejects (overwritten below)
    val = torch.empty((st.shape[0], 1 + L), dtype=torch.int64, device=dev)
    val[:, 0] = torch.arange(lo, lo + st.shape[0], dtype=torch.int64, device=dev)
    val[:, 1:] = g.to(torch.int64) & 0xFFFFFFFF
    rec = torch.full((cap + 1, 1 + L), -1, dtype=torch.int64, device=dev)
    rec.index_copy_(0, row, val) if st.shape[0] else None
    rec[0] = 0
    rec[0, 0] = n
    return rec


def decode_records(recs, world: int, cap: int) -> list[tuple[int, int]]:
    """(curve index, g) pairs from gathered records (host numpy, shape (world*(cap+1), 1+L))."""
    out = []
    r = np.asarray(recs).reshape(world, cap + 1, -1)
    for w in range(world):
        n = int(r[w, 0, 0])
        for row in r[w, 1:1 + min(n, cap)]:
            out.append((int(row[0]), sum(int(x) << (32 * j) for j, x in enumerate(row[1:]))))
    return sorted(out)


def ecm_stage1_distributed(N: int, L: int, B1: int, sigmas, *, group=None, compute=None, device=None,
                           capacity: int | None = None, decode: str = "rank0", events: dict | None = None,
                           local: dict | None = None):
    """Run this rank's shard of `sigmas` (the FULL per-job seed array: host numpy, or a uint64 torch
    tensor — a CUDA tensor stays on the device, so a caller can stage the seeds before timing) and gather.

    Returns (status, factors): status is a uint8 tensor of all `count` curves in curve order
    (identical on every rank, on the gather device); factors is the sorted list of (curve_index,
    g) for the curves with status 1 or 4 on rank 0 (and on every rank with decode="all"), None on
    the other ranks.  decode="defer": no host decode; factors is None and `local` receives the raw
    gathered records ("recs", "world", "cap") for decode_records() outside a timed region.
    `compute(N, L, B1, sigma_tensor) -> {"status": u8[count_local], "g": u32[count_local, L]}`.
    `events`: optional dict; CUDA events "start", "computed", "gathered" are recorded into it on
    the current stream (kernel time = start..computed, gather time = computed..gathered).
    `local`: optional dict that receives this rank's own compute result and shard bounds.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    sig = sigmas if torch.is_tensor(sigmas) else np.asarray(sigmas, dtype=np.uint64)
    if torch.is_tensor(sig) and sig.dtype != torch.uint64:
        raise ValueError("sigmas tensor must be uint64")
    count = int(sig.numel()) if torch.is_tensor(sig) else sig.size
    lo, hi = shard_bounds(count, rank, world)
    # the shard is computed on this rank's GPU (or wherever `compute` wants it); the gather runs
    # on `device` (the NCCL device by default, CPU tensors under gloo)
    cuda = torch.cuda.is_available()
    compute_dev = "cuda" if (compute is None and cuda) else "cpu"
    device = device or ("cuda" if cuda else "cpu")
    shard = -(-count // world)
    cap = capacity if capacity is not None else default_capacity(shard)

    def mark(name):
        if events is not None and cuda:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            events[name] = ev

    shard_sig = (sig[lo:hi] if torch.is_tensor(sig) else torch.from_numpy(sig[lo:hi].copy())).to(compute_dev)
    mark("start")
    res = (compute or _default_compute)(N, L, B1, shard_sig)
    mark("computed")
    if local is not None:
        local.update(res, lo=lo, hi=hi)
    st = res["status"].to(device)
    g = res["g"].to(device)
    rec = compact_factors(st, g, lo, cap)
    if world == 1:
        mark("gathered")
        status, recs = st, rec
        n = int(rec[0, 0])
        if n > cap:
            cap = n
            recs = compact_factors(st, g, lo, cap)
    else:
        # 1) statuses, padded to the largest shard, one all_gather_into_tensor
        pad = torch.zeros(shard, dtype=torch.uint8, device=device)
        pad[: hi - lo] = st
        allst = torch.empty(world * shard, dtype=torch.uint8, device=device)
        dist.all_gather_into_tensor(allst, pad, group=group)
        # 2) fixed-capacity factor records, enqueued right behind it (no host sync in between)
        recs = torch.empty((world * (cap + 1), 1 + L), dtype=torch.int64, device=device)
        dist.all_gather_into_tensor(recs, rec, group=group)
        mark("gathered")
        if count % world == 0:
            status = allst
        else:
            keep = torch.cat([torch.arange(r * shard, r * shard + shard_bounds(count, r, world)[1]
                                           - shard_bounds(count, r, world)[0]) for r in range(world)])
            status = allst[keep.to(device)]
        # one host read after both collectives: exact second gather only on overflow
        counts = recs.view(world, cap + 1, 1 + L)[:, 0, 0].cpu()
        mx = int(counts.max())
        if mx > cap:
            cap = mx
            rec = compact_factors(st, g, lo, cap)
            recs = torch.empty((world * (cap + 1), 1 + L), dtype=torch.int64, device=device)
            dist.all_gather_into_tensor(recs, rec, group=group)
    if decode == "defer":
        if local is not None:
            local.update(recs=recs, world=world, cap=cap)
        return status, None
    if decode == "all" or (decode == "rank0" and rank == 0):
        return status, decode_records(recs.cpu().numpy(), world, cap)
    return status, None
