"""GPU parity: ecm_mulmod_batch (through the C ABI) vs the CPU oracle, bit for bit.

Small sizes span several warp tiles and a ragged tail for every width, mode, layout and REDC
variant; C2 at full size (2^24 triples, the launch configuration bench.py times) is checked
element by element for K = 1 and 16 and on a strided sample for K = 256, plus the Lemma bound
out < 2N on every element.
"""
import numpy as np
import pytest

import paper_1310_3809_b200 as eg
from workload import mulmod_inputs

pytestmark = pytest.mark.gpu

VARIANTS = {"word": eg.ECM_REDC_WORD, "knownlow": eg.ECM_REDC_KNOWNLOW,
            "blockthm": eg.ECM_REDC_BLOCKTHM, "classic": eg.ECM_REDC_CLASSIC, "karatsuba": eg.ECM_REDC_KARATSUBA}


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1310_3809_b200 import build
    build.build()
    return torch


def dev(torch, x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def run_gpu(torch, a, b, n, L, iters, flags):
    if flags & eg.ECM_LAYOUT_SLICED:
        A, B, Nn = (dev(torch, x.T.copy()) for x in (a, b, n))
        out = eg.ecm_mulmod_batch(A, B, Nn, L=L, iters=iters, flags=flags)
        torch.cuda.synchronize()
        return out.cpu().numpy().T.copy()
    A, B, Nn = (dev(torch, x) for x in (a, b, n))
    out = eg.ecm_mulmod_batch(A, B, Nn, L=L, iters=iters, flags=flags)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def lt_2n(x, n):
    """Vectorised x < 2n for (count, L) limb arrays."""
    L = n.shape[1]
    n2 = np.zeros((n.shape[0], L + 1), np.uint64)
    c = np.zeros(n.shape[0], np.uint64)
    for j in range(L):
        t = (n[:, j].astype(np.uint64) << np.uint64(1)) + c
        n2[:, j] = t & np.uint64(0xFFFFFFFF)
        c = t >> np.uint64(32)
    n2[:, L] = c
    less = np.zeros(n.shape[0], bool)
    decided = np.zeros(n.shape[0], bool)
    for j in range(L, -1, -1):
        xj = x[:, j].astype(np.uint64) if j < L else np.zeros(n.shape[0], np.uint64)
        lt, gt = xj < n2[:, j], xj > n2[:, j]
        less |= ~decided & lt
        decided |= lt | gt
    return less


@pytest.mark.parametrize("L", (4, 6, 8, 12, 16))
@pytest.mark.parametrize("square", (False, True))
@pytest.mark.parametrize("layout", ("aos", "sliced"))
@pytest.mark.parametrize("kernel", ("stream", "warp"))
def test_parity_both_kernels(orc, torch, L, square, layout, kernel):
    # the CTA-tile streaming kernel (bulk-copy ring of 256-element tiles, ragged tail by direct
    # loads) and the warp-tile kernel, each forced at short and long chains; counts: several
    # full CTA tiles + a ragged tail (count % 4 == 0 keeps sliced rows on the bulk path), an
    # exact multiple of the tile, and a count below one tile (tail only)
    flags = ((eg.ECM_SQUARE if square else 0) | (eg.ECM_LAYOUT_SLICED if layout == "sliced" else 0) |
             (eg.ECM_KERNEL_STREAM if kernel == "stream" else eg.ECM_KERNEL_WARP))
    for count, iters in ((256 * 9 + 100, 1), (256 * 4, 3), (60, 2), (256 * 3 + 4, 16)):
        a, b, n = mulmod_inputs(count, L, seed=300 + L + count, lazy=True)
        got = run_gpu(torch, a, b, n, L, iters, flags)
        want = orc.mulmod_chain_mt(a, b, n, L, iters, square=square)
        assert np.array_equal(got, want), (L, square, layout, kernel, count, iters)


@pytest.mark.parametrize("L", (4, 6, 8, 12, 16))
@pytest.mark.parametrize("square", (False, True))
@pytest.mark.parametrize("layout", ("aos", "sliced"))
def test_parity_small_all_widths(orc, torch, L, square, layout):
    # several tiles and a ragged tail; 32*37+4 keeps sliced rows 16-byte aligned (vector path),
    # 32*37+5 does not (scalar path)
    count = 32 * 37 + (4 if L % 8 else 5)
    a, b, n = mulmod_inputs(count, L, seed=100 + L, lazy=True)
    flags = (eg.ECM_SQUARE if square else 0) | (eg.ECM_LAYOUT_SLICED if layout == "sliced" else 0)
    for iters in (1, 16):
        got = run_gpu(torch, a, b, n, L, iters, flags)
        want = orc.mulmod_chain_mt(a, b, n, L, iters, square=square)
        assert np.array_equal(got, want), (L, square, layout, iters)
        assert lt_2n(got, n).all()


@pytest.mark.parametrize("variant", list(VARIANTS))
@pytest.mark.parametrize("L", (4, 6, 8, 12, 16))
def test_parity_redc_variants_identical(orc, torch, variant, L):
    """Every REDC variant returns the same unique raw value."""
    count = 32 * 9 + 17
    a, b, n = mulmod_inputs(count, L, seed=200 + L, lazy=True)
    for square in (False, True):
        flags = VARIANTS[variant] | (eg.ECM_SQUARE if square else 0)
        got = run_gpu(torch, a, b, n, L, 7, flags)
        want = orc.mulmod_chain_mt(a, b, n, L, 7, square=square)
        assert np.array_equal(got, want), (variant, L, square)


def test_canonical_flag_and_edges(orc, torch):
    L = 6
    a, b, n = mulmod_inputs(1000, L, seed=7, lazy=True)
    # edge operands: 0, 1, 2n-1
    a[0] = 0
    b[1] = 0
    a[2] = 0; a[2, 0] = 1
    for i in (3, 4):  # 2n - 1
        c = 0
        for j in range(L):
            t = (int(n[i, j]) << 1) + c
            a[i, j] = t & 0xFFFFFFFF
            c = t >> 32
        a[i, 0] -= 1
    b[4] = a[4]
    for iters in (1, 3):
        got = run_gpu(torch, a, b, n, L, iters, eg.ECM_CANONICAL)
        want = orc.mulmod_chain_mt(a, b, n, L, iters, canonical=True)
        assert np.array_equal(got, want)
    assert not got[0].any() and not got[1].any()


def test_single_element_and_check_flag(orc, torch):
    L = 6
    a, b, n = mulmod_inputs(1, L, seed=8)
    got = run_gpu(torch, a, b, n, L, 5, 0)
    assert np.array_equal(got, orc.mulmod_chain(a, b, n, L, 5))
    A, B, Nn = (dev(torch, x) for x in (a, b, n))
    eg.ecm_mulmod_batch(A, B, Nn, L=L, iters=1, flags=eg.ECM_CHECK)
    bad = n.copy()
    bad[0, 0] &= ~np.uint32(1)  # even modulus
    with pytest.raises(eg.EcmError) as e:
        eg.ecm_mulmod_batch(A, B, dev(torch, bad), L=L, iters=1, flags=eg.ECM_CHECK)
    assert e.value.status == 2
    big = a.copy()
    big[0, L - 1] = 0xFFFFFFFF  # >= 2n
    with pytest.raises(eg.EcmError) as e:
        eg.ecm_mulmod_batch(dev(torch, big), B, Nn, L=L, iters=1, flags=eg.ECM_CHECK)
    assert e.value.status == 5


def test_host_buffers_path(orc, torch):
    L = 8
    a, b, n = mulmod_inputs(32 * 5 + 3, L, seed=9, lazy=True)
    out = eg.ecm_mulmod_batch(a, b, n, L=L, iters=4, flags=eg.ECM_HOST_BUFFERS)
    assert np.array_equal(out, orc.mulmod_chain(a, b, n, L, 4))


@pytest.mark.parametrize("iters", [1, 8])
@pytest.mark.parametrize("sliced", [False, True])
def test_host_buffers_with_check_odd_count(orc, torch, iters, sliced):
    """ECM_HOST_BUFFERS | ECM_CHECK stages a, b, n and out in one device scratch block; at L = 6 with an
    odd count the per-array strides must still be 16-byte aligned for the bulk copies and 128-bit
    accesses of both kernels (count >= 257: the streaming kernel at iters 1, the warp kernel at 8)."""
    L, count = 6, 32 * 9 + 1
    a, b, n = mulmod_inputs(count, L, seed=19, lazy=True)
    ref = orc.mulmod_chain(a, b, n, L, iters)
    fl = eg.ECM_HOST_BUFFERS | eg.ECM_CHECK
    if sliced:
        out = eg.ecm_mulmod_batch(a.T.copy(), b.T.copy(), n.T.copy(), L=L, iters=iters,
                                  flags=fl | eg.ECM_LAYOUT_SLICED)
        assert np.array_equal(out.T, ref)
    else:
        out = eg.ecm_mulmod_batch(a, b, n, L=L, iters=iters, flags=fl)
        assert np.array_equal(out, ref)
    bad = n.copy()
    bad[count - 1, 0] &= ~np.uint32(1)  # even modulus on the last element
    with pytest.raises(eg.EcmError) as e:
        eg.ecm_mulmod_batch(a, b, bad, L=L, iters=iters, flags=fl)
    assert e.value.status == 2


def test_c2_full_size(orc, torch):
    """C2: 2^24 triples, L = 6, the bench launch configuration; K = 1, 16 and 256 (the headline)
    element by element against the oracle (K = 256: 4.3e9 products, about 30 s on the box's host
    cores), out < 2N everywhere; AoS == sliced."""
    L, count = 6, 1 << 24
    a, b, n = mulmod_inputs(count, L, seed=2)
    A, B, Nn = (dev(torch, x) for x in (a, b, n))
    for iters in (1, 16):
        got = eg.ecm_mulmod_batch(A, B, Nn, L=L, iters=iters).cpu().numpy()
        want = orc.mulmod_chain_mt(a, b, n, L, iters)
        assert np.array_equal(got, want), iters
        assert lt_2n(got, n).all()
    got = eg.ecm_mulmod_batch(A, B, Nn, L=L, iters=256).cpu().numpy()
    assert lt_2n(got, n).all()
    want = orc.mulmod_chain_mt(a, b, n, L, 256)
    assert np.array_equal(got, want)
    # the same triples in the limb-sliced layout give the same outputs (K = 1: streaming kernel)
    S = [dev(torch, x.T.copy()) for x in (a, b, n)]
    g1 = eg.ecm_mulmod_batch(*S, L=L, iters=1, flags=eg.ECM_LAYOUT_SLICED).cpu().numpy().T
    assert np.array_equal(g1, orc.mulmod_chain_mt(a, b, n, L, 1))
    gs = eg.ecm_mulmod_batch(*S, L=L, iters=256, flags=eg.ECM_LAYOUT_SLICED).cpu().numpy().T
    assert np.array_equal(gs, got)


def test_host_buffers_pipelined_multichunk(orc, torch):
    """ECM_HOST_BUFFERS splits large batches into chunks over two internal streams."""
    L = 4
    count = (1 << 19) + 77
    a, b, n = mulmod_inputs(count, L, seed=10, lazy=True)
    ap, bp, np_ = (torch.from_numpy(x).pin_memory() for x in (a, b, n))
    out = torch.empty_like(ap).pin_memory()
    eg.ecm_mulmod_batch(ap, bp, np_, out, L=L, iters=3, flags=eg.ECM_HOST_BUFFERS)
    want = orc.mulmod_chain_mt(a, b, n, L, 3)
    assert np.array_equal(out.numpy(), want)
    sq = eg.ecm_mulmod_batch(a, b, n, L=L, iters=2, flags=eg.ECM_HOST_BUFFERS | eg.ECM_SQUARE)
    assert np.array_equal(sq, orc.mulmod_chain_mt(a, b, n, L, 2, square=True))


def test_host_buffers_pipelined_sliced(orc, torch):
    """ECM_HOST_BUFFERS | ECM_LAYOUT_SLICED: chunks move as 2-D copies of L rows; the ragged last
    chunk (count % 4 != 0) takes the warp-tile kernel."""
    L = 6
    count = (1 << 19) + 77
    a, b, n = mulmod_inputs(count, L, seed=11, lazy=True)
    sa, sb, sn = (torch.from_numpy(x.T.copy()).pin_memory() for x in (a, b, n))
    out = torch.empty_like(sa).pin_memory()
    for iters in (1, 5):
        eg.ecm_mulmod_batch(sa, sb, sn, out, L=L, iters=iters, flags=eg.ECM_HOST_BUFFERS | eg.ECM_LAYOUT_SLICED)
        want = orc.mulmod_chain_mt(a, b, n, L, iters)
        assert np.array_equal(out.numpy().T, want), iters


@pytest.mark.parametrize("sliced", [False, True])
def test_host_buffers_chunk_ramp(orc, torch, sliced):
    """A batch of ~20 waves through ECM_HOST_BUFFERS runs the whole chunk plan (abi.cu
    pipeline_chunks: 1, 1, 2, 3, 4, ... waves up to the cap, the last wave with the ragged rest) on
    both mulmod kernels (iters 1: streaming, 8: warp tiles); every element equals the oracle."""
    L, count = 6, 3_000_017
    a, b, n = mulmod_inputs(count, L, seed=21, lazy=True)
    for iters in (1, 8):
        if sliced:
            sa, sb, sn = (torch.from_numpy(x.T.copy()).pin_memory() for x in (a, b, n))
            out = torch.empty_like(sa).pin_memory()
            eg.ecm_mulmod_batch(sa, sb, sn, out, L=L, iters=iters, flags=eg.ECM_HOST_BUFFERS | eg.ECM_LAYOUT_SLICED)
            got = out.numpy().T
        else:
            got = eg.ecm_mulmod_batch(a, b, n, L=L, iters=iters, flags=eg.ECM_HOST_BUFFERS)
        assert np.array_equal(got, orc.mulmod_chain_mt(a, b, n, L, iters)), iters


def test_stream_kernel_in_place(orc, torch):
    """out may alias a (include/ecmgpu.h): the streaming kernel's prefetch never reads a tile
    after its output was stored."""
    L = 8
    count = 256 * 40 + 36
    a, b, n = mulmod_inputs(count, L, seed=12, lazy=True)
    want = orc.mulmod_chain_mt(a, b, n, L, 2)
    for fl, tr in ((0, False), (eg.ECM_LAYOUT_SLICED, True)):
        A, B, Nn = (dev(torch, x.T.copy() if tr else x) for x in (a, b, n))
        eg.ecm_mulmod_batch(A, B, Nn, A, L=L, iters=2, flags=fl | eg.ECM_KERNEL_STREAM)
        got = A.cpu().numpy()
        assert np.array_equal(got.T if tr else got, want), fl


def _random_triples_on_device(torch, count, L, sliced, seed):
    """Valid (a, b, n) limb arrays generated on the device (too large to build on the host):
    n odd with bitlen exactly 32L-2, a, b < n (top limb reduced below n's).  Returned as flat
    uint32-sized tensors in the requested layout, plus a (count, L) / (L, count) view helper."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    shape = (L, count) if sliced else (count, L)
    arrs = [torch.randint(0, 256, (count * L * 4,), dtype=torch.uint8, device="cuda", generator=g)
            .view(torch.int32).view(*shape) for _ in range(3)]
    a, b, n = arrs
    top = (lambda t: t[L - 1]) if sliced else (lambda t: t[:, L - 1])
    low = (lambda t: t[0]) if sliced else (lambda t: t[:, 0])
    low(n).bitwise_or_(1)
    nt = top(n)
    nt.bitwise_and_((1 << 29) - 1).bitwise_or_(1 << 29)  # bitlen(n) = 32L - 2
    for x in (a, b):
        xt = top(x)
        xt.copy_(torch.remainder(xt, nt))  # top limb < n's -> x < n
    # the arithmetic above needs int32 ops; the ABI takes uint32 limbs (same bits)
    return a.view(torch.uint32), b.view(torch.uint32), n.view(torch.uint32)


@pytest.mark.parametrize("layout", ("aos", "sliced"))
def test_max_size_64bit_offsets(orc, torch, layout):
    """Maximum sizes: count = 2^30 + 5 triples at L = 6 (24 GiB per array; word offsets up to
    6.4e9 > 2^32 in both layouts), the streaming kernel (K = 1) and the warp-tile kernel (K = 8),
    checked on a sample that includes the ragged tail and the last elements."""
    L, count = 6, (1 << 30) + 5
    free, _ = torch.cuda.mem_get_info()
    if free < 4 * count * L * 4 + (8 << 30):
        pytest.skip(f"needs ~{4 * count * L * 4 >> 30} GiB of free device memory")
    sliced = layout == "sliced"
    a, b, n = _random_triples_on_device(torch, count, L, sliced, seed=7)
    out = torch.empty_like(a)
    flags = eg.ECM_LAYOUT_SLICED if sliced else 0
    idx = np.unique(np.concatenate([np.linspace(0, count - 1, 3000).astype(np.int64),
                                    np.arange(count - 300, count), np.arange(0, 64),
                                    [(1 << 32) // L - 1, (1 << 32) // L, (1 << 32) // L + 1]]))
    it = torch.from_numpy(idx).cuda()

    def rows(t):  # (len(idx), L) host copies of the sampled elements (CUDA indexing needs int32)
        t = t.view(torch.int32)
        r = t[:, it].t() if sliced else t[it]
        return r.contiguous().cpu().numpy().view(np.uint32)

    ah, bh, nh = rows(a), rows(b), rows(n)
    for iters in (1, 8):
        eg.ecm_mulmod_batch(a, b, n, out, L=L, iters=iters, flags=flags)
        torch.cuda.synchronize()
        want = orc.mulmod_chain_mt(ah, bh, nh, L, iters)
        assert np.array_equal(rows(out), want), iters
    del a, b, n, out
    torch.cuda.empty_cache()


def test_fault_injection_is_detected(orc, torch):
    """SURVEY §5 fault injection: one element's modulus corrupted on the device only (a flipped bit,
    as a corrupted n'_0 would act) is caught by the element-wise parity comparison at exactly that
    element, and nowhere else — the parity harness has teeth."""
    L, count = 6, 32 * 9 + 3
    a, b, n = mulmod_inputs(count, L, seed=77)
    n_dev = n.copy()
    n_dev[17, 2] ^= np.uint32(1 << 5)  # stays odd and in range: a different, valid modulus
    A, B, Nn = (dev(torch, x) for x in (a, b, n_dev))
    got = eg.ecm_mulmod_batch(A, B, Nn, L=L, iters=8).cpu().numpy()
    want = orc.mulmod_chain_mt(a, b, n, L, 8)
    bad = np.nonzero((got != want).any(axis=1))[0]
    assert list(bad) == [17]


LAYOUT_KERNELS = {"aos_stream": eg.ECM_KERNEL_STREAM, "aos_warp": eg.ECM_KERNEL_WARP,
                  "sliced_stream": eg.ECM_LAYOUT_SLICED | eg.ECM_KERNEL_STREAM,
                  "sliced_warp": eg.ECM_LAYOUT_SLICED | eg.ECM_KERNEL_WARP}


@pytest.mark.parametrize("L", (4, 6, 8, 12, 16))
@pytest.mark.parametrize("variant", list(VARIANTS))
def test_width_limit_worst_cases(orc, torch, L, variant):
    """Moduli at and just below R/4 = 2^(32L-2) (top limb 0x3fffffff: the two spare bits of
    PAPER.md:189 and nothing more), the smallest full-width N and the tiny N = 3, 5, each with every
    ordered pair of operands from {0, 1, N-1, N, 2N-2, 2N-1}: the accumulator carry bounds of every
    REDC form are tightest here.  Every width x mul/sqr x AoS/sliced x
    streaming/warp-tile kernel x REDC variant, bit-exact against the oracle, raw outputs < 2N."""
    from workload import edge_mulmod_inputs
    a, b, n = edge_mulmod_inputs(L)  # 432 elements: one full 256-element tile + a ragged tail
    for square in (False, True):
        for iters in (1, 3):
            want = orc.mulmod_chain_mt(a, b, n, L, iters, square=square)
            assert lt_2n(want, n).all()
            for name, kf in LAYOUT_KERNELS.items():
                flags = VARIANTS[variant] | kf | (eg.ECM_SQUARE if square else 0)
                got = run_gpu(torch, a, b, n, L, iters, flags)
                assert np.array_equal(got, want), (name, square, iters)
