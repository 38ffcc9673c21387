"""GPU parity of the tensor-core (tcgen05/TMEM) query path (NASG_MLP_BF16:
kind::f16 UMMAs with f16 operands, fp32 accumulation).

Stated contract, checked here:
  * the tensor-core MLP computes exactly f16(inputs) x f16(weights) with fp32
    accumulation and f16 re-quantisation after each ReLU: vs a numpy emulation
    of that arithmetic, >= 90 % of rows agree to 1e-4 (accumulation order) and
    max |d raw| <= 3e-3 (one-ulp f16 rounding flips of a hidden activation);
  * vs the fp32 oracle: raw |d| p99 <= 2e-3 (measured 7e-4 at random init;
    bf16 operands gave 1e-2);
  * K3 stage (fp32 epilogue) given identical raw outputs: direction and pdf
    within 1e-3 for all benign queries and >= 99.9 % of stress queries;
  * end to end vs the oracle: pdf relative p50 <= 1e-3 (measured 3.4e-4),
    lobe-selection mismatch (|d dir| > 0.05) <= 0.2 % (measured 0.03 %).
"""
import numpy as np
import pytest

import nasg_testutil as H

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2303_08064_b200 as nasg  # noqa: E402


def dev4(a3):
    a = np.zeros((len(a3), 4), np.float32)
    a[:, :3] = a3[:, :3]
    return torch.from_numpy(a).cuda()


def split_q(q9):
    return dev4(q9[:, 0:3]), dev4(q9[:, 3:6]), dev4(q9[:, 6:9])


def bf16(x):
    """Round-to-nearest-even to bfloat16, returned as float32."""
    x = np.ascontiguousarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def f16(x):
    """Round-to-nearest-even to IEEE half (saturating at +-65504), as float64."""
    return np.clip(np.asarray(x, np.float32), -65504.0, 65504.0).astype(np.float16).astype(np.float64)


def emulate_tc_mlp(w, enc):
    dims = [64, 128, 128, 128, 65]
    Ws, off = [], 0
    for l in range(4):
        n = dims[l] * dims[l + 1]
        Ws.append(f16(w[off:off + n].reshape(dims[l], dims[l + 1])))
        off += n
    h = f16(enc)
    for l in range(3):
        h = f16(np.maximum(h @ Ws[l], 0).astype(np.float32))
    return (h @ Ws[3]).astype(np.float32)


@pytest.fixture(scope="module")
def guide():
    g = nasg.Guide(nasg.TrainerConfig(seed=1234))
    g.precision = nasg.NASG_MLP_BF16
    yield g
    g.close()


@pytest.mark.parametrize("n", [1, 129, 385, 5000, (1 << 16) + 3])
def test_tc_raw_matches_f16_emulation(guide, orc, n):
    rng = np.random.default_rng(n)
    q9 = H.queries(rng, n, outside=0.1)
    raw = guide.query_raw(*split_q(q9)).cpu().numpy()
    enc, _ = orc.encode(q9, H.BMIN, H.BMAX)
    w = guide.get_weights(published=True)
    emu = emulate_tc_mlp(w, enc)
    err = np.abs(raw - emu)
    # fp32 accumulation order only, except where a hidden activation sits on an
    # f16 rounding boundary and flips by one f16 ulp (rare, bounded)
    rows_off = (err.max(axis=1) > 1e-4).mean()
    fp32 = orc.forward(w, enc)
    d = np.abs(raw - fp32)
    print(f"n={n} rows off emulation {rows_off:.4f} max {err.max():.2e} vs fp32 p99 {np.percentile(d, 99):.2e}")
    assert rows_off <= 0.1, rows_off  # measured 4-6 %
    assert err.max() <= 3e-3, err.max()  # measured <= 1.2e-3
    assert np.percentile(d, 99) <= 2e-3, np.percentile(d, 99)


def test_tc_clamp_counter(guide, orc):
    rng = np.random.default_rng(5)
    q9 = H.queries(rng, 3000, outside=0.5)
    guide.reset_encode_clamp_count()
    guide.query_raw(*split_q(q9))
    torch.cuda.synchronize()
    assert guide.encode_clamp_count == orc.encode(q9, H.BMIN, H.BMAX)[1]


@pytest.mark.parametrize("stress", [False, True])
def test_tc_epilogue_on_identical_raw(guide, orc, stress):
    """K3 in fp32 (the bf16 path's epilogue) vs the double oracle on the same raw."""
    rng = np.random.default_rng(50 + stress)
    n = 1 << 16
    raw, xi = H.raw_outputs(rng, n, stress=stress), H.xis(rng, n)
    out, c = guide.decode_sample_raw(torch.from_numpy(raw).cuda(), torch.from_numpy(xi).cuda())
    out = out.cpu().numpy().astype(np.float64)
    ref, cref = orc.decode_sample(raw, xi, threads=8)
    ddir = np.linalg.norm(out[:, :3] - ref[:, :3], axis=1)
    dpdf = np.abs(out[:, 3] - ref[:, 3]) / ref[:, 3]
    bad = (ddir > 1e-3) | (dpdf > 1e-3)
    assert np.allclose(c.cpu().numpy(), cref, rtol=1e-5)
    if not stress:
        assert not bad.any(), (ddir.max(), dpdf.max())
    else:
        assert bad.mean() <= 1e-3, (bad.mean(), np.median(dpdf))
    dirs = H.dirs(rng, n)
    mix, _ = guide.decode_pdf_raw(torch.from_numpy(raw).cuda(), dev4(dirs), 1.0)
    mref, _ = orc.decode_pdf(raw, dirs, 1.0)
    big = mref > 1e-20
    rel = np.abs(mix.cpu().numpy()[big] - mref[big]) / mref[big]
    assert (rel > 1e-3).mean() <= (1e-3 if stress else 0.0), (rel > 1e-3).mean()


def test_tc_query_sample_end_to_end(guide, orc):
    n = 1 << 16
    x, wo, nrm, xi = nasg.synth_queries(77, n)
    c = torch.empty(n, dtype=torch.float32, device="cuda")
    out, _ = guide.query_sample(*[torch.from_numpy(a).cuda() for a in (x, wo, nrm, xi)], c=c)
    out = out.cpu().numpy().astype(np.float64)
    q9 = np.concatenate([x[:, :3], wo[:, :3], nrm[:, :3]], 1)
    ref, cref = orc.query_sample(guide.get_weights(published=True), q9, xi, threads=8)
    ddir = np.linalg.norm(out[:, :3] - ref[:, :3], axis=1)
    same = ddir <= 0.05
    dpdf = np.abs(out[same, 3] - ref[same, 3]) / ref[same, 3]
    print(f"lobe mismatch {1 - same.mean():.2e} pdf p50 {np.median(dpdf):.2e} p99 {np.percentile(dpdf, 99):.2e} "
          f"c max {np.abs(c.cpu().numpy() - cref).max():.2e}")
    assert 1 - same.mean() <= 2e-3, 1 - same.mean()
    assert np.median(dpdf) <= 1e-3, np.median(dpdf)
    assert np.abs(c.cpu().numpy() - cref).max() <= 5e-3


def test_tc_query_pdf_consistent_with_sample(guide):
    """pdf mode at the sampled directions reproduces the sample mode's pdf."""
    n = 100000
    dev = [torch.from_numpy(a).cuda() for a in nasg.synth_queries(78, n)]
    out, _ = guide.query_sample(*dev)
    mix, guided = guide.query_pdf(dev[0], dev[1], dev[2], out.contiguous(), 0.0)
    rel = ((mix - out[:, 3]).abs() / out[:, 3]).cpu().numpy()
    assert np.percentile(rel, 99.9) <= 1e-3, np.percentile(rel, 99.9)
    assert torch.equal(guided, torch.zeros_like(guided))  # b = 0 and bsdf_pdf = 0


def test_tc_sampler_unbiased_full_size(guide):
    n = 1 << 22
    dev = [torch.from_numpy(a).cuda() for a in nasg.synth_queries(99, n)]
    out, _ = guide.query_sample(*dev)
    out = out.double()
    assert torch.isfinite(out).all()
    inv = 1.0 / out[:, 3]
    est, se = inv.mean().item(), inv.std().item() / np.sqrt(n)
    assert abs(est - 4 * np.pi) < 5 * se + 1e-3, (est, se)


def test_tc_matches_fp32_path_statistically(guide):
    """Same queries through both precisions: pdfs agree in distribution."""
    n = 1 << 18
    dev = [torch.from_numpy(a).cuda() for a in nasg.synth_queries(5, n)]
    a, _ = guide.query_sample(*dev)
    guide.precision = nasg.NASG_MLP_FP32
    b, _ = guide.query_sample(*dev)
    guide.precision = nasg.NASG_MLP_BF16
    same = (a[:, :3] - b[:, :3]).norm(dim=1) < 0.05
    rel = ((a[same, 3] - b[same, 3]).abs() / b[same, 3]).median().item()
    print(f"tc vs fp32 path: same lobe {same.float().mean().item():.5f} pdf p50 {rel:.2e}")
    assert same.float().mean().item() >= 0.998
    assert rel <= 1e-3
