"""Pins the CPU restatement (oracle/nasg_oracle.c) before it is trusted.

1. SPEC.md known-answer examples, run against BOTH the restatement and the
   unmodified reference (oracle/_ref).
2. Restatement vs reference on seeded random inputs (bit-exact where the
   same libm calls are made in the same order).
3. Restatement vs the committed golden fixtures (tests/golden/*.npz, made
   from oracle/_ref by tests/golden/make_golden.py) — this is what pins the
   oracle on hosts where /root/reference (hence oracle/_ref) is absent.
"""
import math
import os

import numpy as np
import pytest

import nasg_testutil as H

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(params=["orc", "ref"])
def any_oracle(request):
    return request.getfixturevalue(request.param)


# ---------------------------------------------------------------- KATs ----
def test_norm_const_kat(any_oracle):
    # SPEC.md:72 (K(lambda=1,a=0) ~ 5.43287; exact 2*pi*(1-e^-2))
    assert any_oracle.norm_const(1.0, 0.0) == pytest.approx(2 * math.pi * (1 - math.exp(-2)), rel=1e-14)
    # a=0 reduces to the SG integral, Eq. 6
    for lam in (1e-3, 0.5, 7.0, 3e3):
        assert any_oracle.norm_const(lam, 0.0) == pytest.approx(2 * math.pi * -math.expm1(-2 * lam) / lam, rel=1e-14)


def test_frame_from_euler_kat(any_oracle):
    f, ok = any_oracle.frame_from_euler(1, 0, 1, 0, 1)
    assert ok and np.allclose(f, np.eye(3))
    f, ok = any_oracle.frame_from_euler(0, 0, 1, 0, 1)
    assert np.allclose(f[2], [1, 0, 0]) and np.allclose(f[0], [0, 0, -1])
    f, ok = any_oracle.frame_from_euler(0.3, 0, 0, 0.5, 0.5)  # degenerate (sin,cos) pair
    assert not ok
    rng = np.random.default_rng(1)
    for _ in range(100):  # SPEC.md:56 orthonormality
        f, _ = any_oracle.frame_from_euler(*rng.uniform(-1, 1, 5))
        assert np.abs(f @ f.T - np.eye(3)).max() < 1e-6
        assert np.abs(np.cross(f[2], f[0]) - f[1]).max() < 1e-6


def _comp(lam, a, frame=np.eye(3)):
    return np.concatenate([frame[0], frame[1], frame[2], [lam, a, 0.0]])


def test_log_eval_kat(any_oracle):
    c = _comp(3.0, 2.0)
    assert any_oracle.nasg_log_eval(c, [0, 0, 1]) == 0.0
    assert any_oracle.nasg_log_eval(c, [0, 0, -1]) == -math.inf
    rng = np.random.default_rng(2)
    for v in H.dirs(rng, 50).astype(np.float64):  # SPEC.md:65 a=0 reduction
        v /= np.linalg.norm(v)
        if v[2] < -1 + 1e-6:
            continue
        assert any_oracle.nasg_log_eval(_comp(2.5, 0.0), v) == pytest.approx(2.5 * (v[2] - 1), rel=1e-9, abs=1e-12)


def test_sample_kat(any_oracle):
    rng = np.random.default_rng(3)
    f, _ = any_oracle.frame_from_euler(*rng.uniform(-1, 1, 5))
    c = _comp(4.0, 3.0, f)
    for x1, x2 in rng.random((10, 2)):
        assert np.allclose(any_oracle.nasg_sample(c, 1.0, x1, x2), f[2], atol=1e-12)
    c = _comp(1e3, 0.0, f)
    for x0, x1, x2 in rng.random((1000, 3)):
        assert any_oracle.nasg_sample(c, x0, x1, x2) @ f[2] > 0.99


def test_one_blob_kat(any_oracle):
    ob = any_oracle.one_blob(0.5)
    assert ob[9] == 1.0 and ob.argmax() == 9
    assert any_oracle.one_blob(0.0).argmax() == 0
    ref = np.exp(-((0.25 - (np.arange(19) + 0.5) / 19) ** 2) * 19 * 19 / 2).astype(np.float32)
    assert np.allclose(any_oracle.one_blob(0.25), ref, rtol=1e-6)


def test_encode_kat(any_oracle):
    q = np.array([[-1, -1, -1, 0.1, 0.2, 0.3, 0, 0, 1], [5, 0, 0, 0, 1, 0, 1, 0, 0]], np.float32)
    enc, clamped = any_oracle.encode(q, H.BMIN, H.BMAX)
    assert enc.shape == (2, 64) and (enc[:, 63] == 1).all()
    assert enc[0, 0] == enc[0, 19] == enc[0, 38] == enc[0, :57].max()  # p at box min -> t=0
    assert np.array_equal(enc[0, 57:63], q[0, 3:9])
    assert clamped == 1  # x=5 outside [-1,1]


def test_decode_zero_kat(any_oracle):
    d = any_oracle.decode(np.zeros(65, np.float32))[0]
    lobes = d[:104].reshape(8, 13)
    assert np.allclose(lobes[:, 9], 1) and np.allclose(lobes[:, 10], 1)
    assert np.allclose(lobes[:, 11], 1 / 8) and d[104] == 0.5
    assert np.allclose(lobes[:, 2], 0)  # cos(theta)=0 -> z on the equator, pairs -> (0,1)


def test_mixture_pdf_kat(any_oracle):
    # single effective component lambda=1, a=0 at v=z -> 1/K = 0.18406
    raw = np.zeros(65, np.float32)
    raw[40:56:2] = 0.0          # lambda = e^0 = 1
    raw[41:56:2] = -60.0        # a = e^-60 ~ 0
    raw[0:40:5] = 30.0          # cos(theta) -> 1 (sigmoid saturates)
    mix, guided = any_oracle.decode_pdf(raw, np.array([[0, 0, 1]], np.float32), b=0.0,
                                        bsdf_pdf=np.array([0.4], np.float32))
    assert mix[0] == pytest.approx(1 / (2 * math.pi * (1 - math.exp(-2))), rel=1e-6)
    assert guided[0] == pytest.approx(0.4, rel=1e-7)  # b=0 -> bsdf pdf
    _, guided = any_oracle.decode_pdf(raw, np.array([[0, 0, 1]], np.float32), b=1.0,
                                      bsdf_pdf=np.array([0.4], np.float32))
    assert guided[0] == pytest.approx(0.5 * mix[0] + 0.5 * np.float32(0.4), rel=1e-12)  # c=0.5


def test_schedules_kat(any_oracle):
    assert any_oracle.stride_update(4, 1 << 14, 1 << 16) == 2
    assert any_oracle.stride_update(4, 1 << 16, 1 << 16) == 4
    assert any_oracle.stride_update(4, 1 << 18, 1 << 16) == 8
    assert any_oracle.stride_update(4, 0, 1 << 16) == 1
    assert any_oracle.blend_coefficient(0) == 0
    assert any_oracle.blend_coefficient(4) == 1 / 64
    assert any_oracle.blend_coefficient(256) == 1.0


def test_adam_first_step_kat(any_oracle):
    w0 = any_oracle.init_network(7)
    w, m, v = w0.copy(), np.zeros_like(w0), np.zeros_like(w0)
    rng = np.random.default_rng(4)
    g = (rng.choice([-1, 1], w0.shape) * rng.uniform(1e-3, 1e-1, w0.shape)).astype(np.float32)
    ok, t = any_oracle.adam_step(w, m, v, g, 0)
    assert ok and t == 1
    assert np.allclose(w - w0, -0.002 * np.sign(g), atol=2e-6)
    g[5] = np.nan
    w1 = w.copy()
    ok, t = any_oracle.adam_step(w, m, v, g, 1)
    assert not ok and t == 1 and np.array_equal(w, w1)  # skip on non-finite, net.hpp:140-144


def test_mixture_integrates_to_one(any_oracle):
    """quadrature of mixture_pdf over the sphere = 1 +- 1e-3."""
    nt, nphi = 600, 1200
    ct = 1 - 2 * (np.arange(nt) + 0.5) / nt  # equal-area in cos(theta)
    ph = 2 * np.pi * (np.arange(nphi) + 0.5) / nphi
    st = np.sqrt(1 - ct**2)
    v = np.stack([np.outer(st, np.cos(ph)), np.outer(st, np.sin(ph)), np.outer(ct, np.ones(nphi))], -1)
    v = v.reshape(-1, 3).astype(np.float32)
    rng = np.random.default_rng(5)
    for _ in range(3):
        raw = H.raw_outputs(rng, 1)
        raw[0, 40:56] = rng.uniform(-1, 2.0, 16)  # moderate lambda, a for the grid
        mix, _ = any_oracle.decode_pdf(np.repeat(raw, len(v), 0), v)
        assert mix.sum() * 4 * np.pi / len(v) == pytest.approx(1.0, abs=1e-3)


def _np_forward64(w, x):
    W = _split(w)
    h = x.astype(np.float64)
    for l in range(3):
        h = np.maximum(h @ W[l], 0)
    return h @ W[3]


def _split(w, out_dim=65):
    dims = [64, 128, 128, 128, out_dim]
    out, off = [], 0
    for l in range(4):
        n = dims[l] * dims[l + 1]
        out.append(np.asarray(w[off:off + n], np.float64).reshape(dims[l], dims[l + 1]))
        off += n
    return out


def test_backward_finite_difference(orc):
    """backward matches central differences (float64) of <out, G>."""
    rng = np.random.default_rng(6)
    w = orc.init_network(3).astype(np.float64)
    x, _ = orc.encode(H.queries(rng, 4), H.BMIN, H.BMAX)
    G = rng.normal(0, 1, (4, 65))
    dw = orc.backward(w.astype(np.float32), x, G.astype(np.float32)).astype(np.float64)
    for i in rng.choice(len(w), 60, replace=False):
        h = 1e-6
        wp, wm = w.copy(), w.copy()
        wp[i] += h
        wm[i] -= h
        fd = ((_np_forward64(wp, x) - _np_forward64(wm, x)) * G).sum() / (2 * h)
        assert dw[i] == pytest.approx(fd, rel=1e-3, abs=1e-5)
    # linearity: backward(2G) == 2 backward(G)
    dw2 = orc.backward(w.astype(np.float32), x, (2 * G).astype(np.float32))
    assert np.allclose(dw2, 2 * dw.astype(np.float32), rtol=0, atol=1e-37)  # exact up to denormals


# ------------------------------------------------- restatement vs reference ----
def test_l0_and_init_match_reference(orc, ref):
    assert np.array_equal(orc.pcg32(42, 54, 100), ref.pcg32(42, 54, 100))
    for seed in (0, 1, 12345):
        assert np.array_equal(orc.init_network(seed), ref.init_network(seed))
    assert np.array_equal(orc.init_network(9, 33), ref.init_network(9, 33))


def test_encode_forward_backward_match_reference(orc, ref):
    rng = np.random.default_rng(7)
    q = H.queries(rng, 300, outside=0.2)
    e1, c1 = orc.encode(q, H.BMIN, H.BMAX)
    e2, c2 = ref.encode(q, H.BMIN, H.BMAX)
    assert np.array_equal(e1, e2) and c1 == c2 and c1 > 0
    w = orc.init_network(11)
    assert np.array_equal(orc.forward(w, e1), ref.forward(w, e1))
    G = rng.normal(0, 1, (300, 65)).astype(np.float32)
    assert np.array_equal(orc.backward(w, e1, G), ref.backward(w, e1, G))


@pytest.mark.parametrize("stress", [False, True])
def test_decode_sample_pdf_match_reference(orc, ref, stress):
    rng = np.random.default_rng(8 + stress)
    n = 2000
    raw, xi = H.raw_outputs(rng, n, stress=stress), H.xis(rng, n)
    assert np.allclose(orc.decode(raw), ref.decode(raw), rtol=1e-14, atol=1e-14)
    d1, c1 = orc.decode_sample(raw, xi)
    d2, c2 = ref.decode_sample(raw, xi)
    assert np.array_equal(c1, c2)
    assert np.allclose(d1, d2, rtol=1e-12, atol=1e-14)
    dirs = H.dirs(rng, n)
    bp = rng.random(n).astype(np.float32)
    m1, g1 = orc.decode_pdf(raw, dirs, 0.7, bp)
    m2, g2 = ref.decode_pdf(raw, dirs, 0.7, bp)
    assert np.allclose(m1, m2, rtol=1e-12, atol=0) and np.allclose(g1, g2, rtol=1e-12, atol=0)


@pytest.mark.parametrize("stress", [False, True])
def test_kl_grad_match_reference(orc, ref, stress):
    rng = np.random.default_rng(10 + stress)
    n = 2000
    raw, s = H.raw_outputs(rng, n, stress=stress), H.samples(rng, n)
    for b in (0.0, 0.5, 1.0):
        g1, ok1, l1 = orc.kl_grad(raw, s, b)
        g2, ok2, l2 = ref.kl_grad(raw, s, b)
        assert np.array_equal(ok1, ok2)
        assert np.allclose(g1, g2, rtol=1e-12, atol=1e-300)
        assert np.allclose(l1, l2, rtol=1e-12, equal_nan=True)


def test_query_sample_matches_reference(orc, ref):
    rng = np.random.default_rng(12)
    w = orc.init_network(5)
    q, xi = H.queries(rng, 1000), H.xis(rng, 1000)
    o1, c1 = orc.query_sample(w, q, xi)
    o2, c2 = ref.query_sample(w, q, xi)
    assert np.array_equal(o1, o2) and np.array_equal(c1, c2)


def test_trainer_matches_reference(orc, ref):
    rng = np.random.default_rng(13)
    s = H.samples(rng, 3000)
    cfg = dict(capacity=4096, batch=512, seed=21)  # 8 steps, reshuffle after 3000/512
    t1, t2 = orc.trainer(**cfg), ref.trainer(**cfg)
    for it, b in enumerate((0.0, 0.5, 1.0)):
        st1, st2 = t1.train(s, b), t2.train(s, b)
        assert st1["steps"] == st2["steps"] == 8
        assert st1["dropped"] == st2["dropped"] and st1["skipped"] == st2["skipped"]
        assert st1["mean_loss"] == pytest.approx(st2["mean_loss"], rel=1e-12)
        assert np.array_equal(t1.weights(), t2.weights())


def test_trainer_empty_buffer(any_oracle):
    t = any_oracle.trainer(seed=3)
    w0 = t.weights()
    st = t.train(np.zeros((0, 16), np.float32), 1.0)
    assert st["steps"] == 0 and np.array_equal(t.weights(), w0)


def test_checkpoint_roundtrip_cross(orc, ref, tmp_path):
    w = orc.init_network(17)
    p1, p2 = str(tmp_path / "a.nasg"), str(tmp_path / "b.nasg")
    assert orc.save_checkpoint(p1, w) == 0
    assert ref.save_checkpoint(p2, w) == 0
    assert open(p1, "rb").read() == open(p2, "rb").read()
    w2, n = ref.load_checkpoint(p1)
    assert n == 8 and np.array_equal(w2, w)
    with open(p1, "r+b") as f:
        f.write(b"XXXX")
    with pytest.raises(IOError):
        orc.load_checkpoint(p1)


def test_reference_loader_skips_the_optimizer_chunk(ref, tmp_path):
    """nasg_save_checkpoint_ex(NASG_CKPT_OPTIMIZER) appends the Adam state after
    the NASGNET1 weights ("NASGADM1", u64 t, u32 n, f32 m[n], f32 v[n]); the
    reference's load_checkpoint (net.cpp:54-82) reads the weights and ignores it."""
    import struct
    w = ref.init_network(23)
    p = str(tmp_path / "adam.nasg")
    assert ref.save_checkpoint(p, w) == 0
    rng = np.random.default_rng(1)
    m, v = rng.normal(size=w.size).astype(np.float32), rng.random(w.size).astype(np.float32)
    with open(p, "ab") as f:
        f.write(b"NASGADM1" + struct.pack("<QI", 1234, w.size) + m.tobytes() + v.tobytes())
    w2, n = ref.load_checkpoint(p)
    assert n == 8 and np.array_equal(w2, w)


# ------------------------------------------------------- golden fixtures ----
def _golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated")
    return np.load(path)


def test_restatement_matches_golden_query(orc):
    g = _golden("query_ref.npz")
    out, c = orc.query_sample(g["w"], g["q9"], g["xi"])
    assert np.array_equal(out, g["out"]) and np.array_equal(c, g["c"])
    raw = g["raw"]
    for stress in ("benign", "stress"):
        d, cc = orc.decode_sample(g[f"raw_{stress}"], g[f"xi_{stress}"])
        assert np.allclose(d, g[f"ds_{stress}"], rtol=1e-12, atol=1e-14)
    assert raw.shape[1] == 65


def test_restatement_matches_golden_train(orc):
    g = _golden("train_ref.npz")
    t = orc.trainer(capacity=int(g["capacity"]), batch=int(g["batch"]), seed=int(g["seed"]))
    for it in range(g["losses"].shape[0]):
        st = t.train(g["samples"], float(g["b"][it]))
        assert st["mean_loss"] == pytest.approx(g["losses"][it], rel=1e-12)
    assert np.array_equal(t.weights(), g["w_final"])


def test_restatement_matches_golden_kl(orc):
    g = _golden("kl_ref.npz")
    gr, ok, loss = orc.kl_grad(g["raw"], g["samples"], float(g["b"]))
    assert np.array_equal(ok, g["ok"])
    assert np.allclose(gr, g["grad"], rtol=1e-12, atol=1e-300)
    assert np.allclose(loss, g["loss"], rtol=1e-12, equal_nan=True)


def test_init_hidden_units_and_embedding(orc):
    """init_network with kHiddenUnits = H: H = 128 is the reference's init;
    embed/extract (the hidden-64 device layout) round-trip; the zero-embedded
    network's outputs equal a direct float64 hidden-64 forward."""
    from oracle.oracle import embed_hidden, extract_hidden
    assert np.array_equal(orc.init_network_hu(5, 128), orc.init_network(5))
    w = orc.init_network_hu(5, 64)
    assert w.shape == (16448,)
    we = embed_hidden(w, 64)
    assert we.shape == (49280,) and np.array_equal(extract_hidden(we, 64), w)
    enc, _ = orc.encode(H.queries(np.random.default_rng(3), 257), H.BMIN, H.BMAX)
    out = orc.forward(we, enc)
    mats, o = [], 0
    for r, c in [(64, 64), (64, 64), (64, 64), (64, 65)]:
        mats.append(w[o:o + r * c].reshape(r, c).astype(np.float64))
        o += r * c
    h = enc.astype(np.float64)
    for m in mats[:3]:
        h = np.maximum(h @ m, 0.0)
    ref = h @ mats[3]
    assert np.allclose(out, ref, rtol=1e-4, atol=1e-5)
