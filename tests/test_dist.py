"""World-size-2, -3 and -8 gloo tests of the multi-GPU shard + gather logic (paper_1310_3809_b200.dist)
on CPU, with the oracle standing in for the per-GPU kernel."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1310_3809_b200.dist import ecm_stage1_distributed, shard_bounds

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_compute(N, L, B1, sig_t):
    import oracle
    k, _ = oracle.stage1_k(B1)
    r = oracle.ecm_stage1(N, L, k, sig_t.numpy())
    return {"status": torch.from_numpy(r["status"]), "g": torch.from_numpy(r["g"].astype(np.int64))}


def _worker(rank, world, port, cfg, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        status, factors = ecm_stage1_distributed(cfg["N"], cfg["L"], cfg["B1"], cfg["sigmas"],
                                                 compute=_oracle_compute, device="cpu")
        out_q.put((rank, status.numpy().tobytes(), factors))
    finally:
        dist.destroy_process_group()


def test_shard_bounds_cover_exactly():
    for count in (1, 7, 256, 1 << 20):
        for w in (1, 2, 3, 8):
            b = [shard_bounds(count, r, w) for r in range(w)]
            assert b[0][0] == 0 and b[-1][1] == count
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))


@pytest.mark.parametrize("world", (2, 3, 8))
def test_gloo_gather_equals_single_process(orc, world):
    from workload import ecm_config
    cfg = ecm_config(L=6, nbits=190, pbits=32, B1=300, curves=75, seed=1)  # ragged: 75 curves
    cfg = {k: cfg[k] for k in ("N", "L", "B1", "sigmas")}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    k, _ = orc.stage1_k(cfg["B1"])
    want = orc.ecm_stage1(cfg["N"], 6, k, cfg["sigmas"])
    want_factors = sorted((int(i), orc.from_limbs(want["g"][i])) for i in np.nonzero(want["status"] == 1)[0])
    for rank, st_bytes, factors in results:
        st = np.frombuffer(st_bytes, np.uint8)
        assert np.array_equal(st, want["status"]), rank
        assert factors == want_factors, rank
    assert len(want_factors) > 0
