"""nasg_query_shade: guided scattering for a wavefront tracer (SPEC.md tracer
trace_path; guided_pdf guiding.cpp:81-85; mixture_sample sphdist.cpp:183-198).

The shade epilogue must agree with the parity-tested sample / pdf entry points
on the same network snapshot (those are checked against the oracle in
test_gpu_query.py / test_gpu_tc.py):
  * xi_t = 0, b = 1  -> always the mixture technique: direction and q_mix equal
    nasg_query_sample's (same xi);  c' = c
  * xi_t = 1         -> never the mixture: direction = the BSDF sample exactly,
    q_mix(dir) and q_mix(nee) equal nasg_query_pdf at those directions
  * a device-side row count (n_dev) limits the rows written
Tolerance: 1e-5 relative (fp32 path, double epilogue both ways), 2e-4 for the
bf16 path's fp32 epilogue (different instruction order).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2303_08064_b200 as nasg  # noqa: E402


def unit(rng, n):
    v = rng.normal(size=(n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    out = np.zeros((n, 4), np.float32)
    out[:, :3] = v
    return out


@pytest.fixture(scope="module")
def guide():
    g = nasg.Guide(nasg.TrainerConfig(seed=77))
    yield g
    g.close()


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_shade_matches_sample_and_pdf(guide, prec):
    guide.precision = nasg.NASG_MLP_BF16 if prec == "bf16" else nasg.NASG_MLP_FP32
    tol = 1e-5 if prec == "fp32" else 2e-4
    try:
        n = 70_001
        rng = np.random.default_rng(3)
        x, wo, nrm, xi = [torch.from_numpy(a).cuda() for a in nasg.synth_queries(21, n)]
        db = unit(rng, n)
        dn = unit(rng, n)
        dn[:, 3] = 1.0
        dn[::7, 3] = 0.0  # some vertices without a light sample
        db_t, dn_t = torch.from_numpy(db).cuda(), torch.from_numpy(dn).cuda()
        # technique forced to the mixture
        db_t[:, 3] = 0.0
        out = guide.query_shade(x, wo, nrm, xi, db_t, dn_t, 1.0).cpu().numpy()
        c = torch.empty(n, dtype=torch.float32, device="cuda")
        ref, _ = guide.query_sample(x, wo, nrm, xi, c=c)
        ref, c = ref.cpu().numpy(), c.cpu().numpy()
        assert np.all(out[:, 1, 2] == 1.0)
        assert np.abs(out[:, 0, :3] - ref[:, :3]).max() <= 10 * tol
        assert np.allclose(out[:, 0, 3], ref[:, 3], rtol=tol, atol=0)
        assert np.allclose(out[:, 1, 1], c, rtol=1e-6) and np.allclose(out[:, 1, 3], c, rtol=1e-6)
        # q_mix at the NEE direction
        mix_n, _ = guide.query_pdf(x, wo, nrm, dn_t, 0.0)
        mix_n = mix_n.cpu().numpy()
        has = dn[:, 3] > 0
        assert np.allclose(out[has, 1, 0], mix_n[has], rtol=tol, atol=1e-30)
        assert np.all(out[~has, 1, 0] == 0.0)
        # technique forced to the BSDF sample
        db_t[:, 3] = 1.0
        out = guide.query_shade(x, wo, nrm, xi, db_t, dn_t, 0.5).cpu().numpy()
        assert np.all(out[:, 1, 2] == 0.0)
        assert np.array_equal(out[:, 0, :3], db[:, :3])
        mix_b, _ = guide.query_pdf(x, wo, nrm, db_t, 0.0)
        assert np.allclose(out[:, 0, 3], mix_b.cpu().numpy(), rtol=tol, atol=1e-30)
        assert np.allclose(out[:, 1, 1], 0.5 * c, rtol=1e-6)
    finally:
        guide.precision = nasg.NASG_MLP_FP32


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_shade_device_row_count(guide, prec):
    guide.precision = nasg.NASG_MLP_BF16 if prec == "bf16" else nasg.NASG_MLP_FP32
    try:
        n, live = 5000, 1234
        rng = np.random.default_rng(4)
        x, wo, nrm, xi = [torch.from_numpy(a).cuda() for a in nasg.synth_queries(22, n)]
        db, dn = torch.from_numpy(unit(rng, n)).cuda(), torch.from_numpy(unit(rng, n)).cuda()
        n_dev = torch.tensor([live], dtype=torch.int32, device="cuda")
        full = guide.query_shade(x, wo, nrm, xi, db, dn, 1.0)
        out = torch.full((n, 2, 4), -7.0, device="cuda")
        nasg._check(nasg.lib().nasg_query_shade(guide._h, n, nasg._ptr(n_dev), nasg._ptr(x), nasg._ptr(wo),
                                                nasg._ptr(nrm), nasg._ptr(xi), nasg._ptr(db), nasg._ptr(dn),
                                                1.0, nasg._ptr(out), nasg._stream(None)))
        assert torch.equal(out[:live], full[:live])
        assert bool((out[live:] == -7.0).all())
    finally:
        guide.precision = nasg.NASG_MLP_FP32
