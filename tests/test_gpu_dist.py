"""The N > 1 ECM path with the real kernel: paper_1310_3809_b200.dist.ecm_stage1_distributed on 2
and 4 ranks sharing cuda:0 (collectives over gloo on CPU tensors; NCCL cannot put two ranks on one
GPU), each rank running ecm_stage1_batch (libecmgpu) on its contiguous curve shard.

Checked element by element: the gathered status vector and factor list against the oracle on a
C1-sized config (the planted 32-bit p is found on ~10 % of curves), and against one single-launch
GPU run of the same curves on C3's modulus and B1.  Curves are independent work items
(PAPER.md:310-312), so the sharded result must equal the single-launch one exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1310_3809_b200 import build
    build.build()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1310_3809_b200.dist import ecm_stage1_distributed
        loc = {}
        status, factors = ecm_stage1_distributed(cfg["N"], cfg["L"], cfg["B1"], cfg["sigmas"], device="cpu",
                                                 decode="all", local=loc)
        out_q.put((rank, status.numpy().tobytes(), factors, loc["lo"], loc["hi"],
                   loc["g"].cpu().numpy().tobytes()))
    except Exception as e:  # surface the worker's error in the parent's assertion
        out_q.put((rank, None, repr(e), 0, 0, b""))
        raise
    finally:
        dist.destroy_process_group()


def _run(world, cfg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0, res
    for r in res:
        assert r[1] is not None, r[2]
    return res


def _factors(status, g, lim):
    fl = np.nonzero((status == 1) | (status == 4))[0]
    return sorted((int(i), lim(g[i])) for i in fl)


@pytest.mark.parametrize("world", (2, 4))
def test_distributed_c1_equals_oracle(orc, world):
    from workload import ecm_config
    c = ecm_config("C1")  # 256 curves, B1 = 2000, 190-bit N with a planted 32-bit p
    cfg = {"N": c["N"], "L": 6, "B1": c["B1"], "sigmas": c["sigmas"]}
    k, _ = orc.stage1_k(cfg["B1"])
    want = orc.ecm_stage1(cfg["N"], 6, k, cfg["sigmas"])
    want_f = _factors(want["status"], want["g"], orc.from_limbs)
    assert len(want_f) >= 10
    res = _run(world, cfg)
    for rank, st, factors, lo, hi, gb in res:
        assert np.array_equal(np.frombuffer(st, np.uint8), want["status"]), rank
        assert factors == want_f, rank
        # each rank's own shard: g limb for limb
        g = np.frombuffer(gb, np.uint32).reshape(hi - lo, 6)
        assert np.array_equal(g, want["g"][lo:hi]), rank
        assert all(c["p"] == f or f % c["p"] == 0 for _, f in factors)
    assert [r[3] for r in res] == [r * 256 // world for r in range(world)]


@pytest.mark.parametrize("world", (2, 4))
def test_distributed_c3_equals_single_launch(world):
    import paper_1310_3809_b200 as eg
    from workload import ecm_config
    c = ecm_config("C3")  # C3's modulus and B1 = 50000; the first 6001 curves (ragged shards)
    cfg = {"N": c["N"], "L": 6, "B1": c["B1"], "sigmas": c["sigmas"][:6001]}
    one = eg.ecm_stage1_batch(cfg["N"], 6, cfg["B1"], torch.from_numpy(cfg["sigmas"].copy()).cuda(), want=("g",))
    st1 = one["status"].cpu().numpy()
    g1 = one["g"].cpu().numpy()
    want_f = _factors(st1, g1, eg.limbs_to_int)
    res = _run(world, cfg)
    for rank, st, factors, lo, hi, gb in res:
        assert np.array_equal(np.frombuffer(st, np.uint8), st1), rank
        assert factors == want_f, rank
        assert np.array_equal(np.frombuffer(gb, np.uint32).reshape(hi - lo, 6), g1[lo:hi]), rank
    for _, f in want_f:  # every flagged g divides N (planted 64-bit p)
        assert 1 < f < cfg["N"] and cfg["N"] % f == 0
