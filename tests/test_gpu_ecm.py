"""GPU parity: ecm_stage1_batch / ecm_ladder_batch (through the C ABI) vs the CPU oracle.

Bit-exact on every output (X, Z, g, status, xaff) for C1 (all 256 curves), for every width on
small configs with ragged curve counts, for degenerate seeds; [#E(F_p)]P = O on small primes
with brute-force group orders; C3 at full size (2^20 curves, B1 = 50000 — the launch bench.py
times for ECM) on a strided sample plus every flagged g checked by division.
"""
import numpy as np
import pytest

import paper_1310_3809_b200 as eg
from workload import ecm_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1310_3809_b200 import build
    build.build()
    return torch


def gpu_stage1(torch, N, L, B1, sig, **kw):
    s = torch.from_numpy(np.ascontiguousarray(sig, dtype=np.uint64)).cuda()
    r = eg.ecm_stage1_batch(N, L, B1, s, **kw)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in r.items()}


def assert_same(got, want, keys=("X", "Z", "g", "status", "xaff")):
    for k in keys:
        assert np.array_equal(got[k], want[k]), k


KERNELS = {"default": 0, "lanes1": eg.ECM_KERNEL_LANES1, "lanes4": eg.ECM_KERNEL_LANES4}


@pytest.mark.parametrize("kernel", list(KERNELS))
def test_c1_all_curves_bit_exact(orc, torch, kernel):
    """C1 (256 curves) through the default choice (the 4-lane latency kernel at this size) and
    both kernels forced: every output bit-exact."""
    cfg = ecm_config("C1")
    k, _ = orc.stage1_k(cfg["B1"])
    got = gpu_stage1(torch, cfg["N"], cfg["L"], cfg["B1"], cfg["sigmas"], flags=KERNELS[kernel])
    want = orc.ecm_stage1_mt(cfg["N"], cfg["L"], k, cfg["sigmas"])
    assert_same(got, want)
    found = got["status"] == 1
    assert 10 <= found.sum() <= 45
    for row in got["g"][found]:
        assert eg.limbs_to_int(row) == cfg["p"]


@pytest.mark.parametrize("kernel", ["lanes1", "lanes4"])
@pytest.mark.parametrize("L,nbits,pbits", [(4, 126, 30), (6, 190, 40), (8, 254, 40), (12, 382, 40), (16, 510, 40)])
def test_widths_ragged_counts(orc, torch, L, nbits, pbits, kernel):
    cfg = ecm_config(L=L, nbits=nbits, pbits=pbits, B1=400, curves=77, seed=20 + L)
    k, _ = orc.stage1_k(cfg["B1"])
    got = gpu_stage1(torch, cfg["N"], L, cfg["B1"], cfg["sigmas"], flags=KERNELS[kernel])
    want = orc.ecm_stage1_mt(cfg["N"], L, k, cfg["sigmas"])
    assert_same(got, want)


@pytest.mark.parametrize("kernel", ["lanes1", "lanes4"])
def test_ladder_explicit_scalars(orc, torch, kernel):
    cfg = ecm_config(L=6, nbits=190, pbits=32, B1=100, curves=40, seed=31)
    s = torch.from_numpy(cfg["sigmas"]).cuda()
    for k in (1, 2, 3, 4, 5, 7, 0x1F3, (1 << 200) + 12345, 2520):
        r = eg.ecm_ladder_batch(cfg["N"], 6, k, s, flags=KERNELS[kernel])
        got = {kk: v.cpu().numpy() for kk, v in r.items()}
        want = orc.ecm_stage1(cfg["N"], 6, k, cfg["sigmas"])
        assert_same(got, want)


def _curve_order(orc, p, sigma):
    st, x0, a24, _ = orc.suyama(p, 1, sigma)
    if st:
        return None
    A = (4 * a24 - 2) % p
    B = (x0 ** 3 + A * x0 * x0 + x0) % p
    if B == 0 or (A * A - 4) % p == 0:
        return None
    Binv = pow(B, -1, p)
    n = 1
    for x in range(p):
        r = (x * x * x + A * x * x + x) * Binv % p
        n += 1 if r == 0 else (2 if pow(r, (p - 1) // 2, p) == 1 else 0)
    return n


@pytest.mark.parametrize("p", [1009, 2003, 4093])
def test_group_order_kills_point(orc, torch, p):
    """[#E(F_p)]P = O: Z == 0, status ALL, g = p; with N = p in L = 4."""
    for sigma in range(6, 14):
        nE = _curve_order(orc, p, sigma)
        if nE is None:
            continue
        s = torch.tensor([sigma], dtype=torch.uint64).cuda()
        r = eg.ecm_ladder_batch(p, 4, nE, s)
        assert int(r["status"][0]) == 2
        assert eg.limbs_to_int(r["Z"][0].cpu().numpy()) == 0
        assert eg.limbs_to_int(r["g"][0].cpu().numpy()) == p


def test_degenerate_sigmas(orc, torch):
    # 15^2 - 5 = 220 = 20*11: u = 0 mod 11.  N = 11*13 -> setup factor 11; N = 11 -> status 3
    got = gpu_stage1(torch, 143, 4, 50, np.array([15, 6, 7], np.uint64))
    k, _ = orc.stage1_k(50)
    want = orc.ecm_stage1(143, 4, k, [15, 6, 7])
    assert_same(got, want)
    assert got["status"][0] == 4 and eg.limbs_to_int(got["g"][0]) == 11
    got = gpu_stage1(torch, 11, 4, 50, np.array([15], np.uint64))
    assert got["status"][0] == 3


def test_host_buffers_and_no_xaff(orc, torch):
    cfg = ecm_config(L=6, nbits=190, pbits=32, B1=300, curves=50, seed=41)
    k, _ = orc.stage1_k(cfg["B1"])
    r = eg.ecm_stage1_batch(cfg["N"], 6, cfg["B1"], cfg["sigmas"].copy(), flags=eg.ECM_HOST_BUFFERS)
    want = orc.ecm_stage1(cfg["N"], 6, k, cfg["sigmas"])
    assert_same(r, want)
    got = gpu_stage1(torch, cfg["N"], 6, cfg["B1"], cfg["sigmas"], want=("X", "Z", "g"))
    assert_same(got, want, keys=("X", "Z", "g", "status"))


def test_c3_full_size_sampled(orc, torch):
    """C3 (B1 = 50000, 2^20 curves, 190-bit N with a planted 64-bit p; the launch bench.py times):
    4096 strided curves bit-exact vs the oracle (about 20 s on the box's host cores); every flagged
    g divides N."""
    cfg = ecm_config("C3")
    N, L = cfg["N"], cfg["L"]
    got = gpu_stage1(torch, N, L, cfg["B1"], cfg["sigmas"], want=("X", "Z", "g"))
    idx = np.arange(0, cfg["curves"], cfg["curves"] // 4096) + 7
    k, _ = orc.stage1_k(cfg["B1"])
    want = orc.ecm_stage1_mt(N, L, k, cfg["sigmas"][idx])
    sub = {key: v[idx] for key, v in got.items()}
    assert_same(sub, want, keys=("X", "Z", "g", "status"))
    flagged = np.nonzero(got["status"] == 1)[0]
    assert len(flagged) > 1000  # Dickman estimate ~7k
    for i in flagged:
        g = eg.limbs_to_int(got["g"][i])
        assert 1 < g < N and N % g == 0


@pytest.mark.parametrize("L,nbits", [(6, 190), (8, 254)])
def test_ablation_variants_identical(orc, torch, L, nbits):
    """Every REDC form x eager/lazy reduction ECM kernel gives the same canonical outputs (the
    Lemma's lazy domain changes nothing observable)."""
    cfg = ecm_config(L=L, nbits=nbits, pbits=32, B1=300, curves=70, seed=50 + L)
    k, _ = orc.stage1_k(cfg["B1"])
    want = orc.ecm_stage1(cfg["N"], L, k, cfg["sigmas"])
    for var in (eg.ECM_REDC_WORD, eg.ECM_REDC_KNOWNLOW, eg.ECM_REDC_BLOCKTHM, eg.ECM_REDC_CLASSIC):
        for eager in (0, eg.ECM_EAGER):
            got = gpu_stage1(torch, cfg["N"], L, cfg["B1"], cfg["sigmas"], flags=var | eager)
            assert_same(got, want)


def test_ablation_flags_rejected_for_other_widths(torch):
    s = torch.tensor([6, 7], dtype=torch.uint64).cuda()
    with pytest.raises(eg.EcmError):
        eg.ecm_stage1_batch(2 ** 120 + 1, 4, 100, s, flags=eg.ECM_EAGER)


@pytest.mark.parametrize("L,nbits,flags", [
    (6, 190, 0),
    (8, 254, 0),
    (8, 254, eg.ECM_EAGER),
    (8, 254, eg.ECM_REDC_BLOCKTHM),
    (8, 254, eg.ECM_REDC_CLASSIC | eg.ECM_EAGER),
])
def test_prime_ladder_schedule(orc, torch, L, nbits, flags):
    """Paper-comparable prime-by-prime schedule (ECM_PRIME_LADDERS, §8(f) N2) vs the oracle's,
    bit for bit; and the same [k]P (status, affine x) as the full-k ladder."""
    cfg = ecm_config(L=L, nbits=nbits, pbits=32, B1=500, curves=45, seed=60 + L)
    got = gpu_stage1(torch, cfg["N"], L, cfg["B1"], cfg["sigmas"], flags=eg.ECM_PRIME_LADDERS | flags)
    want = orc.ecm_stage1_primes(cfg["N"], L, cfg["B1"], cfg["sigmas"])
    assert_same(got, want)
    full = gpu_stage1(torch, cfg["N"], L, cfg["B1"], cfg["sigmas"])
    assert np.array_equal(full["status"], got["status"]) and np.array_equal(full["xaff"], got["xaff"])


def test_c5_sampled_curves_full_b1(orc, torch):
    """C5's modulus and parameters (254-bit N = p*q with a planted 80-bit p, L = 8, B1 = 250000):
    48 curves strided over the 2^22 seeds, bit-exact vs the oracle at the full B1."""
    cfg = ecm_config("C5")
    idx = np.arange(0, cfg["curves"], cfg["curves"] // 48)[:48] + 3
    sig = cfg["sigmas"][idx]
    got = gpu_stage1(torch, cfg["N"], 8, cfg["B1"], sig)
    k, _ = orc.stage1_k(cfg["B1"])
    want = orc.ecm_stage1_mt(cfg["N"], 8, k, sig)
    assert_same(got, want)


# --------------------------------------------------------------------------------------
# small-parameter family (reading G16): a24 = s / 2^32, x0 = 2
# --------------------------------------------------------------------------------------
def small_seeds(sig):
    """Seeds in [1, 2^30) derived from the configs' Suyama sigmas."""
    return (np.asarray(sig, dtype=np.uint64) % np.uint64((1 << 30) - 1)) + np.uint64(1)


@pytest.mark.parametrize("kernel", list(KERNELS))
def test_small_family_c1_bit_exact(orc, torch, kernel):
    cfg = ecm_config("C1")
    k, _ = orc.stage1_k(cfg["B1"])
    seeds = np.concatenate([small_seeds(cfg["sigmas"]), np.array([0, 1 << 30, 1, (1 << 30) - 1], np.uint64)])
    got = gpu_stage1(torch, cfg["N"], 6, cfg["B1"], seeds, flags=eg.ECM_CURVE_SMALL | KERNELS[kernel])
    want = orc.ecm_stage1_mt(cfg["N"], 6, k, seeds, family="small")
    assert_same(got, want)
    assert list(got["status"][-4:-2]) == [3, 3]
    assert (got["status"] == 1).sum() >= 5


@pytest.mark.parametrize("kernel", ["lanes1", "lanes4"])
@pytest.mark.parametrize("L,nbits,pbits", [(4, 126, 30), (8, 254, 40), (12, 382, 40), (16, 510, 40)])
def test_small_family_widths(orc, torch, L, nbits, pbits, kernel):
    cfg = ecm_config(L=L, nbits=nbits, pbits=pbits, B1=400, curves=77, seed=50 + L)
    k, _ = orc.stage1_k(cfg["B1"])
    seeds = small_seeds(cfg["sigmas"])
    got = gpu_stage1(torch, cfg["N"], L, cfg["B1"], seeds, flags=eg.ECM_CURVE_SMALL | KERNELS[kernel])
    want = orc.ecm_stage1_mt(cfg["N"], L, k, seeds, family="small")
    assert_same(got, want)


def test_small_family_c3_sampled(orc, torch):
    """C3's modulus and B1 with 2^18 small-family curves (the one-lane kernel at scale): 128
    strided curves bit-exact, every flagged g divides N."""
    cfg = ecm_config("C3")
    seeds = small_seeds(cfg["sigmas"][: 1 << 18])
    got = gpu_stage1(torch, cfg["N"], 6, cfg["B1"], seeds, flags=eg.ECM_CURVE_SMALL)
    idx = np.linspace(0, seeds.size - 1, 128).astype(np.int64)
    k, _ = orc.stage1_k(cfg["B1"])
    want = orc.ecm_stage1_mt(cfg["N"], 6, k, seeds[idx], family="small")
    assert_same({kk: v[idx] for kk, v in got.items()}, want)
    flagged = np.nonzero(got["status"] == 1)[0]
    assert flagged.size > 0
    for i in flagged:
        gi = eg.limbs_to_int(got["g"][i])
        assert 1 < gi < cfg["N"] and cfg["N"] % gi == 0


def test_results_independent_of_sharding(torch):
    """1/2/4/8 contiguous shards (what each rank of an N-GPU run computes)
    concatenate to the single-launch result, with both kernel choices at the shard sizes."""
    cfg = ecm_config(L=6, nbits=190, pbits=40, B1=500, curves=3000, seed=61)
    full = gpu_stage1(torch, cfg["N"], 6, cfg["B1"], cfg["sigmas"])
    for w in (2, 4, 8):
        parts = [gpu_stage1(torch, cfg["N"], 6, cfg["B1"], cfg["sigmas"][r * 3000 // w:(r + 1) * 3000 // w])
                 for r in range(w)]
        for key in ("X", "Z", "g", "status", "xaff"):
            assert np.array_equal(np.concatenate([p[key] for p in parts]), full[key]), (w, key)


@pytest.mark.parametrize("kernel", ["lanes1", "lanes4"])
@pytest.mark.parametrize("L", (4, 6, 8, 12, 16))
def test_near_max_composite_every_width(orc, torch, L, kernel):
    """ECM on N = p q just below R/4 = 2^(32L-2) (the largest modulus the two spare bits allow,
    PAPER.md:189) at every width with both kernels: X, Z, g, status, xaff bit-exact vs the oracle."""
    from workload import near_max_composite, sigmas
    N, p, q = near_max_composite(L)
    assert N.bit_length() == 32 * L - 2
    sig = sigmas(62 + L, 45)
    k, _ = orc.stage1_k(400)
    want = orc.ecm_stage1_mt(N, L, k, sig)
    got = gpu_stage1(torch, N, L, 400, sig, flags=KERNELS[kernel])
    assert_same(got, want)
