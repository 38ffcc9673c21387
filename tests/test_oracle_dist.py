"""Pins the CPU restatement of the explicit-mixture density layer and the
vMF / SG baseline (oracle/nasg_oracle.c orc_dist_*, orc_vmf_fit_grad) to the
unmodified reference (sphdist.cpp:152-340 via oracle/_ref) and to the
committed golden fixture tests/golden/dist_ref.npz (make_golden_dist.py),
plus the SPEC.md examples for the vMF baseline and the
SG-reduction identity."""
import math
import os

import numpy as np
import pytest

import nasg_testutil as H

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "dist_ref.npz")


@pytest.fixture(params=["orc", "ref"])
def any_oracle(request):
    return request.getfixturevalue(request.param)


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("stress", [False, True])
def test_dist_restatement_matches_reference(orc, ref, kind, stress):
    rng = np.random.default_rng(11 + kind + 2 * stress)
    k = 8 if kind == 0 else 14
    comp, w = (H.nasg_records if kind == 0 else H.vmf_records)(rng, 300, k, stress=stress)
    d = np.zeros((300, 4), np.float32)
    d[:, :3] = H.dirs(rng, 300)
    xi = H.xis(rng, 300)
    for fn, arg in (("dist_pdf", d), ("dist_sample", xi), ("dist_grad", d)):
        a, b = getattr(orc, fn)(kind, comp, w, arg), getattr(ref, fn)(kind, comp, w, arg)
        assert np.allclose(a, b, rtol=1e-12, atol=1e-300, equal_nan=True), fn


def test_dist_restatement_matches_golden(orc):
    g = np.load(GOLDEN)
    for kind, name in ((0, "nasg"), (1, "vmf")):
        for tag in ("benign", "stress"):
            t = f"{name}_{tag}"
            comp, w = g[f"{t}_comp"], g[f"{t}_w"]
            assert np.allclose(orc.dist_pdf(kind, comp, w, g[f"{t}_dir"]), g[f"{t}_pdf"], rtol=1e-12, atol=1e-300)
            assert np.allclose(orc.dist_sample(kind, comp, w, g[f"{t}_xi"]), g[f"{t}_sample"], rtol=1e-12, atol=1e-14)
            assert np.allclose(orc.dist_grad(kind, comp, w, g[f"{t}_dir"]), g[f"{t}_grad"], rtol=1e-12, atol=1e-300)
    gr, ok = orc.vmf_fit_grad(g["fit_raw"], g["fit_samples"])
    assert np.array_equal(ok, g["fit_ok"])
    assert np.allclose(gr, g["fit_grad"], rtol=1e-12, atol=1e-300)


def test_vmf_fit_grad_matches_reference(orc, ref):
    rng = np.random.default_rng(5)
    for k in (1, 3, 14):
        raw = rng.normal(0.0, 1.0, 5 * k).astype(np.float32)
        raw[3 * k: 4 * k] = rng.uniform(-9.0, 9.0, k)  # both sharpness clamps
        s = np.zeros((500, 4), np.float32)
        s[:, :3] = H.dirs(rng, 500)
        s[:, 3] = rng.exponential(1.0, 500)
        a, oka = orc.vmf_fit_grad(raw, s)
        b, okb = ref.vmf_fit_grad(raw, s)
        assert np.array_equal(oka, okb)
        assert np.allclose(a, b, rtol=1e-12, atol=1e-300)


def test_vmf_fit_grad_finite_difference(orc):
    # d/d raw of -mean log q_mix(v) by central differences (double, via the pdf entry)
    rng = np.random.default_rng(8)
    k = 3
    raw = rng.normal(0.0, 1.0, 5 * k).astype(np.float32)
    s = np.zeros((64, 4), np.float32)
    s[:, :3] = H.dirs(rng, 64)
    s[:, 3] = 1.0
    g, ok = orc.vmf_fit_grad(raw, s)
    assert ok.all()

    def neg_log_q(r):
        nr = np.linalg.norm(r[: 3 * k].reshape(k, 3).astype(np.float64), axis=1)
        mu = r[: 3 * k].reshape(k, 3) / nr[:, None]
        lam = np.exp(r[3 * k: 4 * k].astype(np.float64))
        e = np.exp(r[4 * k:] - r[4 * k:].max())
        wts = e / e.sum()
        comp = np.concatenate([mu, lam[:, None]], 1)
        q = orc.dist_pdf(1, np.repeat(comp[None], 64, 0).astype(np.float32),
                         np.repeat(wts[None], 64, 0).astype(np.float32), s)
        return -np.log(q)

    # the pdf entry takes fp32 records, so difference at a step where fp32 rounding is negligible
    h = 1e-2
    for j in range(5 * k):
        rp, rm = raw.astype(np.float64).copy(), raw.astype(np.float64).copy()
        rp[j] += h
        rm[j] -= h
        fd = (neg_log_q(rp) - neg_log_q(rm)) / (2 * h)
        assert np.allclose(g[:, j], fd, rtol=2e-3, atol=2e-3), j


def test_vmf_sample_kat(any_oracle):
    # xi0 = 0 -> cos(theta) = 1, v = mu
    rng = np.random.default_rng(2)
    comp, w = H.vmf_records(rng, 64, 1)
    xi = H.xis(rng, 64)
    xi[:, 1] = 0.0
    out = any_oracle.dist_sample(1, comp, w, xi)
    mu = comp[:, 0, :3].astype(np.float64)
    mu /= np.linalg.norm(mu, axis=1, keepdims=True)
    assert np.allclose(out[:, :3], mu, atol=1e-12)


def test_vmf_pdf_integrates_to_one(any_oracle):
    # quadrature of the vMF pdf over the sphere = 1 +- 1e-6
    # (Gauss-Legendre in z x uniform phi; tilted axes so both directions matter)
    zg, wz = np.polynomial.legendre.leggauss(256)
    nphi = 512
    phi = (np.arange(nphi) + 0.5) * 2 * np.pi / nphi
    Z, P = np.meshgrid(zg, phi, indexing="ij")
    r = np.sqrt(1 - Z * Z)
    d = np.stack([r * np.cos(P), r * np.sin(P), Z, 0 * Z], -1).reshape(-1, 4).astype(np.float32)
    wq = (np.repeat(wz[:, None], nphi, 1) * (2 * np.pi / nphi)).reshape(-1)
    for lam, mu in ((0.5, (0.6, 0.0, 0.8)), (3.0, (0.0, 0.6, -0.8)), (20.0, (0.36, 0.48, 0.8))):
        comp = np.tile(np.array([*mu, lam], np.float32), (len(d), 1, 1))
        pdf = any_oracle.dist_pdf(1, comp, np.ones((len(d), 1), np.float32), d)
        assert (pdf * wq).sum() == pytest.approx(1.0, abs=1e-6)


def test_sg_reduction_identity(any_oracle):
    # SPEC.md:544 (acceptance 3): a = 0, eps = 0 -> NASG density = vMF density within 1e-9
    rng = np.random.default_rng(3)
    n = 400
    f = H.frames(rng, n)
    lam = np.exp(rng.uniform(np.log(1e-2), np.log(1e2), n))
    nasg = np.zeros((n, 1, 12), np.float32)
    nasg[:, 0, 0:3], nasg[:, 0, 3] = f[:, 0], lam
    nasg[:, 0, 4:7] = f[:, 1]
    nasg[:, 0, 8:11] = f[:, 2]
    vmf = np.zeros((n, 1, 4), np.float32)
    vmf[:, 0, 0:3], vmf[:, 0, 3] = f[:, 2], lam
    d = np.zeros((n, 4), np.float32)
    d[:, :3] = H.dirs(rng, n)
    w = np.ones((n, 1), np.float32)
    a, b = any_oracle.dist_pdf(0, nasg, w, d), any_oracle.dist_pdf(1, vmf, w, d)
    assert np.allclose(a, b, rtol=1e-9, atol=1e-300)


@pytest.mark.parametrize("kind", ["orc", "ref"])
def test_nasg_grad_logpdf_central_differences(kind, request):
    # SPEC.md:545 (acceptance 4a): the 7 decoded-scalar gradients of log(mixture
    # pdf) against central differences (step 1e-5, double precision) at 100 random
    # points, relative error < 1e-4.  Single-lobe mixtures: log pdf = log G - log K;
    # the finite differences go through frame_from_euler (pair renormalisation
    # included), nasg_log_eval and nasg_norm_const in double.
    o = request.getfixturevalue(kind)
    rng = np.random.default_rng(17)
    bad = 0
    for _ in range(100):
        ct = rng.uniform(-0.9, 0.9)
        ph, ta = rng.uniform(0, 2 * np.pi, 2)
        th = np.array([ct, np.sin(ph), np.cos(ph), np.sin(ta), np.cos(ta)])
        lam, a = np.exp(rng.uniform(np.log(0.1), np.log(20.0))), np.exp(rng.uniform(np.log(0.01), np.log(20.0)))

        def logp(t7):
            fr, _ = o.frame_from_euler(*t7[:5])
            c12 = np.concatenate([fr.reshape(9), [t7[5], t7[6], 0.0]])
            return o.nasg_log_eval(c12, v) - np.log(o.norm_const(t7[5], t7[6], 0.0))

        fr, _ = o.frame_from_euler(*th)
        # a direction near the lobe (where the gradient is large), away from the poles
        v = fr[2] + 0.6 * rng.normal(size=3)
        v /= np.linalg.norm(v)
        t7 = np.concatenate([th, [lam, a]])
        h = 1e-5
        fd = np.array([(logp(t7 + h * np.eye(7)[k]) - logp(t7 - h * np.eye(7)[k])) / (2 * h) for k in range(7)])
        rec = np.zeros((1, 1, 12), np.float32)
        rec[0, 0, 0:3], rec[0, 0, 3], rec[0, 0, 4:7], rec[0, 0, 7], rec[0, 0, 8:11] = fr[0], lam, fr[1], a, fr[2]
        d = np.zeros((1, 4), np.float32)
        d[0, :3] = v
        g = o.dist_grad(0, rec, np.ones((1, 1), np.float32), d)[0, 0, :7]
        err = np.abs(g - fd) / (np.abs(fd).max() + 1e-12)
        bad += err.max() > 1e-4
    assert bad == 0, bad


@pytest.mark.parametrize("kind", ["orc", "ref"])
def test_kl_loss_gradient_central_differences(kind, request):
    # SPEC.md:545 (acceptance 4c): kl_loss_gradient end to end through decode
    # (guiding.cpp:108-165) against central differences of loss_surrogate
    # (:167-176), relative error < 1e-4.  Raw outputs and the steps are multiples
    # of 2^-11, so raw +- h is exact in the float raw vector.
    o = request.getfixturevalue(kind)
    rng = np.random.default_rng(29)
    h = 2.0 ** -10

    def cd(raw, smp, b, step):  # central differences of loss_surrogate, all 65 coordinates
        pert = np.repeat(raw, 130, 0)
        for j in range(65):
            pert[2 * j, j] += step
            pert[2 * j + 1, j] -= step
        _, _, loss = o.kl_grad(pert.astype(np.float32), np.repeat(smp, 130, 0), b)
        return (loss[0::2] - loss[1::2]) / (2 * step)

    for b in (0.5, 1.0):
        raws = np.round(rng.normal(0.0, 0.7, (20, 65)) / (h / 2)) * (h / 2)
        s = H.samples(rng, 20, zero_p_frac=0.0)
        for r in range(20):
            g, ok, _ = o.kl_grad(raws[r:r + 1].astype(np.float32), s[r:r + 1], b)
            if not ok[0]:
                continue
            # Richardson extrapolation of the h and h/2 differences: O(h^4) truncation
            fd = (4.0 * cd(raws[r:r + 1], s[r:r + 1], b, h / 2) - cd(raws[r:r + 1], s[r:r + 1], b, h)) / 3.0
            scale = np.abs(fd).max()
            assert np.all(np.abs(g[0] - fd) <= 1e-4 * scale + 1e-12), (r, np.abs(g[0] - fd).max() / scale)
