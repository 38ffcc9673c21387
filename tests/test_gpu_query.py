"""GPU parity of the query path against the CPU oracle (oracle/nasg_oracle.c).

Tolerances (north_star: fp32 path within 1e-3 relative for pdf and direction):
  * raw MLP outputs (fp32 FFMA vs fp32 oracle, different summation order):
    |d| <= 2e-5 * (1 + |raw|)
  * benign inputs: every query's direction |d dir| <= 1e-3 and pdf rel <= 1e-3
  * stress inputs (lambda, a log-uniform to the 3e3 clamps, near-degenerate
    pairs): >= 99.9 % of queries within 1e-3; lobe-selection flips (xi_select
    within rounding of a CDF boundary) are counted separately and must be
    <= 1e-4 of queries.
"""
import numpy as np
import pytest

import nasg_testutil as H

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2303_08064_b200 as nasg  # noqa: E402


def dev4(a3):
    """(n,3) or (n,4) numpy -> (n,4) float32 CUDA tensor."""
    a = np.zeros((len(a3), 4), np.float32)
    a[:, : min(4, a3.shape[1])] = a3[:, :4]
    return torch.from_numpy(a).cuda()


@pytest.fixture(scope="module")
def guide():
    g = nasg.Guide(nasg.TrainerConfig(seed=1234))
    yield g
    g.close()


def _split_q(q9):
    return dev4(q9[:, 0:3]), dev4(q9[:, 3:6]), dev4(q9[:, 6:9])


def _dir_pdf_check(gpu, ref, tol=1e-3):
    gpu = gpu.astype(np.float64)
    ddir = np.linalg.norm(gpu[:, :3] - ref[:, :3], axis=1)
    dpdf = np.abs(gpu[:, 3] - ref[:, 3]) / np.maximum(np.abs(ref[:, 3]), 1e-30)
    return ddir, dpdf


def test_init_weights_bit_exact(guide, orc):
    assert np.array_equal(guide.get_weights(), orc.init_network(1234))
    assert np.array_equal(guide.get_weights(published=True), orc.init_network(1234))


@pytest.mark.parametrize("n", [1, 127, 128, 4099])
def test_query_raw_matches_oracle(guide, orc, n):
    rng = np.random.default_rng(n)
    q9 = H.queries(rng, n, outside=0.1)
    raw = guide.query_raw(*_split_q(q9)).cpu().numpy()
    enc, _ = orc.encode(q9, H.BMIN, H.BMAX)
    ref = orc.forward(guide.get_weights(published=True), enc)
    assert raw.shape == ref.shape
    assert np.all(np.abs(raw - ref) <= 2e-5 * (1 + np.abs(ref))), np.abs(raw - ref).max()


def test_encode_clamp_counter(guide, orc):
    rng = np.random.default_rng(5)
    q9 = H.queries(rng, 1000, outside=0.5)
    guide.reset_encode_clamp_count()
    guide.query_raw(*_split_q(q9))
    torch.cuda.synchronize()
    _, clamped = orc.encode(q9, H.BMIN, H.BMAX)
    assert guide.encode_clamp_count == clamped > 0


@pytest.mark.parametrize("stress", [False, True])
def test_decode_sample_raw_matches_oracle(guide, orc, stress):
    rng = np.random.default_rng(11 + stress)
    n = 1 << 16
    raw, xi = H.raw_outputs(rng, n, stress=stress), H.xis(rng, n)
    out, c = guide.decode_sample_raw(torch.from_numpy(raw).cuda(), torch.from_numpy(xi).cuda())
    out, c = out.cpu().numpy(), c.cpu().numpy()
    ref, cref = orc.decode_sample(raw, xi, threads=8)
    assert np.allclose(c, cref, rtol=1e-6)
    ddir, dpdf = _dir_pdf_check(out, ref)
    bad = (ddir > 1e-3) | (dpdf > 1e-3)
    # a lobe-selection flip (xi_sel within rounding of a cumulative weight) sends
    # the sample to another lobe: a different direction altogether; every other
    # query outside 1e-3 is a genuine miss of the same lobe's sample
    flip = ddir > 0.05
    miss = bad & ~flip
    print(f"stress={stress}: outside 1e-3 {bad.mean():.2e} (lobe flips {flip.mean():.2e}, same-lobe misses "
          f"{miss.mean():.2e}; max same-lobe dir {ddir[~flip].max():.2e} pdf {dpdf[~flip].max():.2e})")
    if not stress:
        assert not bad.any(), (ddir.max(), dpdf.max())
    else:
        assert flip.mean() <= 1e-4 and miss.mean() <= 1e-3, (flip.mean(), miss.mean())


@pytest.mark.parametrize("stress", [False, True])
def test_decode_pdf_raw_matches_oracle(guide, orc, stress):
    rng = np.random.default_rng(21 + stress)
    n = 1 << 15
    raw = H.raw_outputs(rng, n, stress=stress)
    dirs = H.dirs(rng, n)
    if stress:  # half the directions sampled from the lobes themselves (high-density region)
        ref_s, _ = orc.decode_sample(raw, H.xis(rng, n), threads=8)
        dirs[: n // 2] = ref_s[: n // 2, :3].astype(np.float32)
    bsdf = rng.random(n).astype(np.float32)
    for b in (0.0, 0.6, 1.0):
        mix, guided = guide.decode_pdf_raw(torch.from_numpy(raw).cuda(), dev4(dirs), b, torch.from_numpy(bsdf).cuda())
        mix, guided = mix.cpu().numpy(), guided.cpu().numpy()
        mref, gref = orc.decode_pdf(raw, dirs, b, bsdf)
        rm = np.abs(mix - mref) / np.maximum(mref, 1e-30)
        rg = np.abs(guided - gref) / np.maximum(gref, 1e-30)
        big = mref > 1e-30
        if not stress:
            assert rm.max() <= 1e-3 and rg.max() <= 1e-3, (rm.max(), rg.max())
        else:
            assert (rm[big] > 1e-3).mean() <= 1e-3, (rm[big] > 1e-3).mean()
            assert (rg > 1e-3).mean() <= 1e-3
        if b == 0.0:
            assert np.array_equal(guided, bsdf)  # guided_pdf with b = 0


@pytest.mark.parametrize("n", [1, 333, 1 << 16])
def test_query_sample_fp32_matches_oracle(guide, orc, n):
    rng = np.random.default_rng(31 + n)
    q9, xi = H.queries(rng, n), H.xis(rng, n)
    c = torch.empty(n, dtype=torch.float32, device="cuda")
    out, _ = guide.query_sample(*_split_q(q9), torch.from_numpy(xi).cuda(), c=c)
    out, c = out.cpu().numpy(), c.cpu().numpy()
    ref, cref = orc.query_sample(guide.get_weights(published=True), q9, xi, threads=8)
    ddir, dpdf = _dir_pdf_check(out, ref.astype(np.float64))
    assert ddir.max() <= 1e-3 and dpdf.max() <= 1e-3, (ddir.max(), dpdf.max())
    assert np.allclose(c, cref, rtol=1e-5)


def test_query_pdf_fp32_matches_oracle(guide, orc):
    rng = np.random.default_rng(41)
    n = 20000
    q9, dirs = H.queries(rng, n), H.dirs(rng, n)
    bsdf = rng.random(n).astype(np.float32)
    mix, guided = guide.query_pdf(*_split_q(q9), dev4(dirs), 0.7, torch.from_numpy(bsdf).cuda())
    enc, _ = orc.encode(q9, H.BMIN, H.BMAX)
    raw = orc.forward(guide.get_weights(published=True), enc)
    mref, gref = orc.decode_pdf(raw, dirs, 0.7, bsdf)
    assert np.allclose(mix.cpu().numpy(), mref, rtol=1e-3, atol=0)
    assert np.allclose(guided.cpu().numpy(), gref, rtol=1e-3, atol=0)


def test_query_sample_host_matches_device(guide):
    n = (1 << 20) + 77  # more than one pipeline chunk, ragged
    x, wo, nrm, xi = nasg.synth_queries(7, n)
    c = np.empty(n, np.float32)
    out_h, _ = guide.query_sample_host(x, wo, nrm, xi, c=c)
    dev = [torch.from_numpy(a).cuda() for a in (x, wo, nrm, xi)]
    cd = torch.empty(n, dtype=torch.float32, device="cuda")
    out_d, _ = guide.query_sample(*dev, c=cd)
    assert np.array_equal(out_h, out_d.cpu().numpy())
    assert np.array_equal(c, cd.cpu().numpy())


def test_sampler_unbiased_full_size(guide):
    """Size-independent property at the benchmark size: E_q[1/q(w)] = 4 pi."""
    n = 1 << 22
    x, wo, nrm, xi = [torch.from_numpy(a).cuda() for a in nasg.synth_queries(99, n)]
    out, _ = guide.query_sample(x, wo, nrm, xi)
    out = out.double()
    assert torch.isfinite(out).all()
    assert torch.allclose(out[:, :3].norm(dim=1), torch.ones(n, dtype=torch.float64, device="cuda"), atol=1e-5)
    est = (1.0 / out[:, 3]).mean().item()
    se = (1.0 / out[:, 3]).std().item() / np.sqrt(n)
    assert abs(est - 4 * np.pi) < 5 * se + 1e-3, (est, se)


def test_empty_batch_is_noop(guide):
    e = torch.empty((0, 4), dtype=torch.float32, device="cuda")
    out, _ = guide.query_sample(e, e, e, e)
    assert out.shape == (0, 4)


def test_snapshot_isolation(orc):
    """Queries read the published snapshot; set_weights publishes (guiding.hpp:151-157)."""
    g = nasg.Guide(nasg.TrainerConfig(seed=3))
    rng = np.random.default_rng(3)
    q9 = H.queries(rng, 256)
    before = g.query_raw(*_split_q(q9)).cpu().numpy()
    w = orc.init_network(4)
    g.set_weights(w)
    after = g.query_raw(*_split_q(q9)).cpu().numpy()
    enc, _ = orc.encode(q9, H.BMIN, H.BMAX)
    assert np.allclose(after, orc.forward(w, enc), rtol=1e-4, atol=2e-5)
    assert not np.allclose(before, after)
    g.close()


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_publish_never_overwrites_a_snapshot_in_use(orc, prec):
    """A reader holds its snapshot (shared_ptr<const> NetworkSnapshot, net.hpp:161,
    guiding.hpp:139-141): a query queued on another stream behind a long kernel
    reads the weights that were published when it was issued, even when two
    publishes (the second one reusing its slot) are issued before it runs."""
    g = nasg.Guide(nasg.TrainerConfig(seed=3))
    g.precision = nasg.NASG_MLP_FP32 if prec == "fp32" else nasg.NASG_MLP_BF16
    rng = np.random.default_rng(4)
    q9 = H.queries(rng, 4096)
    xq = _split_q(q9)
    xi = dev4(H.xis(rng, 4096))
    ref, _ = g.query_sample(*xq, xi)
    ref = ref.cpu().numpy()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        torch.cuda._sleep(200_000_000)  # ~0.1 s: the query below waits behind it
        out, _ = g.query_sample(*xq, xi, stream=side)
    g.set_weights(orc.init_network(8))   # publish into the other slot
    g.set_weights(orc.init_network(9))   # reuses the slot the queued query reads: must wait for it
    side.synchronize()
    assert np.array_equal(out.cpu().numpy(), ref)
    new, _ = g.query_sample(*xq, xi)
    assert not np.allclose(new.cpu().numpy(), ref)
    g.close()


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_packed_rows_match_soa(guide, prec):
    """nasg_query_sample_packed / _host_packed (13-float rows) == the SoA entry points."""
    guide.precision = nasg.NASG_MLP_BF16 if prec == "bf16" else nasg.NASG_MLP_FP32
    try:
        n = 300_001
        x, wo, nrm, xi = nasg.synth_queries(11, n)
        q13 = np.ascontiguousarray(np.concatenate([x[:, :3], wo[:, :3], nrm[:, :3], xi], 1))
        dev = [torch.from_numpy(a).cuda() for a in (x, wo, nrm, xi)]
        c1 = torch.empty(n, dtype=torch.float32, device="cuda")
        ref, _ = guide.query_sample(*dev, c=c1)
        c2 = torch.empty(n, dtype=torch.float32, device="cuda")
        out, _ = guide.query_sample_packed(torch.from_numpy(q13).cuda(), c=c2)
        assert torch.equal(out, ref) and torch.equal(c1, c2)
        hc = np.empty(n, np.float32)
        hout, _ = guide.query_sample_host_packed(q13, c=hc)
        assert np.array_equal(hout, ref.cpu().numpy()) and np.array_equal(hc, c1.cpu().numpy())
    finally:
        guide.precision = nasg.NASG_MLP_FP32


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_packed_rows_unaligned_pointer(guide, prec):
    """A 13-float row array that is not 16-byte aligned (no TMA staging) gives the same results."""
    guide.precision = nasg.NASG_MLP_BF16 if prec == "bf16" else nasg.NASG_MLP_FP32
    try:
        n = 5_003
        x, wo, nrm, xi = nasg.synth_queries(12, n)
        q13 = np.concatenate([x[:, :3], wo[:, :3], nrm[:, :3], xi], 1).astype(np.float32)
        buf = torch.zeros(n * 13 + 1, dtype=torch.float32, device="cuda")
        buf[1:] = torch.from_numpy(q13.ravel()).cuda()
        un = buf[1:].view(n, 13)  # 4-byte offset from a 256-byte aligned allocation
        assert un.data_ptr() % 16 == 4
        out_u, _ = guide.query_sample_packed(un)
        out_a, _ = guide.query_sample_packed(torch.from_numpy(q13).cuda())
        assert torch.equal(out_u, out_a)
    finally:
        guide.precision = nasg.NASG_MLP_FP32
