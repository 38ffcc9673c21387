"""Guided progressive render loop (nasg_render_*), checked against the SPEC.md
tracer module's examples and invariants (:378-478).  The reference specifies
the tracer but ships no code for it, so its oracle here is analytic:
  * white furnace: constant environment 1 over a lambertian plane of albedo
    0.5 -> every pixel's expectation is 0.5, with guiding on and any network
    state (SPEC trace_path example; the estimator must stay unbiased);
  * no emitters and zero environment -> exactly 0;
  * determinism: identical seed -> bitwise-identical film, guiding and online
    training included;
  * unbiasedness: guided and unguided renders of the box scene agree within
    3 combined standard errors; NEE + MIS agrees with the brute-force
    scattering-only estimator (SPEC's direct-light example); the ramp-free
    accumulation is the plain mean;
  * training records: collected samples are finite with q > 0, at most S kept.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2303_08064_b200 as nasg  # noqa: E402


def make(scene, prec="bf16", seed=5, **kw):
    lo, hi = nasg.scene_bounds(scene)
    g = nasg.Guide(nasg.TrainerConfig(seed=seed), bmin=lo, bmax=hi)
    p = nasg.NASG_MLP_BF16 if prec == "bf16" else nasg.NASG_MLP_FP32
    g.precision = p
    g.train_precision = p
    return g, nasg.Render(g, scene=scene, **kw)


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
def test_white_furnace_guided_is_unbiased(prec):
    # b = 1 from the second iteration (M = B = 1): guided scattering with whatever the
    # network has learnt so far; every frame must still average 0.5
    g, r = make(nasg.SCENE_FURNACE, prec, width=96, height=96, seed=11, schedule_m=1, schedule_b=1)
    try:
        vals = []
        for it in range(8):
            st = r.iteration()
            fr = r.image(1)[..., 0].ravel().astype(np.float64)
            if it >= 1:
                assert st["b"] == 1.0 and st["guided_vertices"] == st["vertices"] > 0
                vals.append(fr)
            assert st["nonfinite_paths"] == 0
        v = np.concatenate(vals)  # independent pixel estimates pooled over the guided frames
        se = v.std() / np.sqrt(v.size)
        assert se > 0  # guided frames do have variance (mixture sampling is live)
        assert abs(v.mean() - 0.5) <= 4 * se, (v.mean(), se)
    finally:
        r.close()
        g.close()


def test_dark_scene_is_black():
    g, r = make(nasg.SCENE_DARK, width=64, height=64, schedule_m=1, schedule_b=1)
    try:
        for _ in range(3):
            r.iteration()
        assert np.all(r.image() == 0.0)
    finally:
        r.close()
        g.close()


def test_render_is_deterministic():
    imgs = []
    for _ in range(2):
        g, r = make(nasg.SCENE_BOX, width=80, height=64, seed=7, schedule_m=1, schedule_b=4)
        try:
            for _ in range(6):
                r.iteration()
            imgs.append((r.image(), g.get_weights()))
        finally:
            r.close()
            g.close()
    assert np.array_equal(imgs[0][0], imgs[1][0])
    assert np.array_equal(imgs[0][1], imgs[1][1])


def test_lazy_train_stats_only_shifts_the_report():
    # lazy_train_stats = 1 queues the next iteration behind training instead of
    # waiting for it: same film, same weights; stats.train arrives one call later
    out = []
    for lazy in (False, True):
        g, r = make(nasg.SCENE_BOX, width=80, height=64, seed=7, schedule_m=1, schedule_b=4, lazy_train_stats=lazy)
        try:
            tr = [r.iteration()["train"] for _ in range(6)]
            out.append((r.image(), g.get_weights(), tr))
        finally:
            r.close()
            g.close()
    (ia, wa, ta), (ib, wb, tb) = out
    assert np.array_equal(ia, ib) and np.array_equal(wa, wb)
    assert tb[0].steps == 0
    assert [t.steps for t in tb[1:]] == [t.steps for t in ta[:-1]]
    assert [t.mean_loss for t in tb[1:]] == [t.mean_loss for t in ta[:-1]]


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
def test_pipelined_loop_is_unbiased_and_deterministic(prec):
    # pipelined = 1: tracing of i+1 overlaps training i (snapshot one iteration
    # staler).  The estimator stays unbiased (furnace expectation 0.5 with b = 1
    # and a network that changes under it), the run is bitwise deterministic, and
    # stats.train reports training i-2.
    runs = []
    for _ in range(2):
        g, r = make(nasg.SCENE_FURNACE, prec, width=96, height=96, seed=11, schedule_m=1, schedule_b=1,
                    pipelined=True)
        try:
            vals, trains = [], []
            for it in range(8):
                st = r.iteration()
                trains.append(st["train"].steps)
                fr = r.image(1)[..., 0].ravel().astype(np.float64)
                if it >= 1:
                    assert st["b"] == 1.0 and st["guided_vertices"] == st["vertices"] > 0
                    vals.append(fr)
            v = np.concatenate(vals)
            se = v.std() / np.sqrt(v.size)
            assert abs(v.mean() - 0.5) <= 4 * se, (v.mean(), se)
            assert trains[:2] == [0, 0] and all(t > 0 for t in trains[2:]), trains
            runs.append((r.image(), g.get_weights()))
        finally:
            r.close()
            g.close()
    assert np.array_equal(runs[0][0], runs[1][0]) and np.array_equal(runs[0][1], runs[1][1])


def test_pipelined_box_matches_serial_mean():
    # the box scene's pipelined render agrees with the serial SPEC loop's (both unbiased)
    means = []
    for pipelined in (False, True):
        g, r = make(nasg.SCENE_BOX, width=128, height=128, seed=5, schedule_m=1, schedule_b=4, pipelined=pipelined)
        try:
            for _ in range(48):
                r.iteration()
            img = r.image().astype(np.float64)
            means.append((img.mean(), img.std() / np.sqrt(img.size)))
        finally:
            r.close()
            g.close()
    (ma, sa), (mb, sb) = means
    assert abs(ma - mb) <= 4 * np.hypot(sa, sb) + 1e-3 * ma, means


def test_guided_matches_unguided_mean():
    """Guiding changes variance, never the mean (SPEC tracer invariants)."""
    res = {}
    for guiding in (False, True):
        g, r = make(nasg.SCENE_BOX, width=64, height=64, seed=3 + guiding, guiding=guiding,
                    ramp=False, schedule_m=1, schedule_b=2)
        try:
            fm = []
            for _ in range(40):
                r.iteration()
                fm.append(np.asarray(r.image(1)).mean(axis=(0, 1)) @ np.array([0.2126, 0.7152, 0.0722]))
            res[guiding] = np.array(fm[2:])  # guided frames from b = 1 on
        finally:
            r.close()
            g.close()
    a, b = res[False], res[True]
    se = np.sqrt(a.var(ddof=1) / a.size + b.var(ddof=1) / b.size)
    assert abs(a.mean() - b.mean()) <= 3 * se, (a.mean(), b.mean(), se)


def test_plain_mean_without_ramp_and_records():
    g, r = make(nasg.SCENE_CRACK, width=64, height=48, seed=9, ramp=False)
    try:
        frames = []
        for _ in range(4):
            st = r.iteration()
            frames.append(r.image(1))
            assert 0 < st["kept"] <= g.config.sample_capacity
            assert st["kept"] == min(st["collected"], g.config.sample_capacity)
            assert st["train"].steps > 0 and np.isfinite(st["train"].mean_loss)
            assert st["train"].dropped_samples == 0
        assert np.allclose(r.image(), np.mean(frames, axis=0), rtol=1e-5, atol=1e-6)
    finally:
        r.close()
        g.close()


def test_row_shards_tile_the_image():
    """Config 5's sharding: rows [0, h/2) and [h/2, h) rendered separately equal the full image."""
    full_g, full = make(nasg.SCENE_BOX, width=64, height=64, seed=13, collect=False, guiding=False)
    parts = []
    try:
        full.iteration()
        ref = full.image()
        for rb, re in ((0, 32), (32, 64)):
            g, r = make(nasg.SCENE_BOX, width=64, height=64, seed=13, collect=False, guiding=False,
                        row_begin=rb, row_end=re)
            r.iteration()
            parts.append(r.image())
            r.close()
            g.close()
    finally:
        full.close()
        full_g.close()
    assert np.array_equal(np.concatenate(parts, axis=0), ref)


def test_interleaved_row_bands_tile_the_image():
    """Config 5's load-balanced sharding: bands of 8 rows dealt round-robin over 3
    ranks (the last band partial) reassemble the full image exactly."""
    W, Hh, band, ns = 64, 60, 8, 3
    full_g, full = make(nasg.SCENE_BOX, width=W, height=Hh, seed=13, collect=False, guiding=False)
    try:
        full.iteration()
        ref = full.image()
    finally:
        full.close()
        full_g.close()
    out = np.full_like(ref, np.nan)
    for k in range(ns):
        g, r = make(nasg.SCENE_BOX, width=W, height=Hh, seed=13, collect=False, guiding=False,
                    row_band=band, shard=k, nshards=ns)
        r.iteration()
        img = r.image()
        rows = [y for b in range(k, -(-Hh // band), ns) for y in range(b * band, min(Hh, (b + 1) * band))]
        assert img.shape[0] == len(rows) == r.rows
        out[rows] = img
        r.close()
        g.close()
    assert np.array_equal(out, ref)


def test_interleaved_shards_collect_and_train():
    """With collection on, an interleaved shard collects over its compacted rows
    and trains (finite film, samples kept, Adam steps taken)."""
    g, r = make(nasg.SCENE_BOX, width=64, height=64, seed=3, row_band=8, shard=1, nshards=2,
                schedule_m=1, schedule_b=2)
    try:
        for _ in range(3):
            st = r.iteration()
        assert st["kept"] > 0 and st["train"].steps > 0
        assert np.isfinite(r.image()).all()
    finally:
        r.close()
        g.close()


def frame_means(scene, frames, skip=1, **kw):
    g, r = make(scene, **kw)
    try:
        fm = []
        for it in range(frames):
            r.iteration()
            if it >= skip:
                fm.append(np.asarray(r.image(1)).mean(axis=(0, 1)) @ np.array([0.2126, 0.7152, 0.0722]))
        return np.array(fm)
    finally:
        r.close()
        g.close()


@pytest.mark.parametrize("scene", [nasg.SCENE_BOX, nasg.SCENE_CRACK, nasg.SCENE_INDIRECT])
def test_nee_mis_matches_brute_force(scene):
    """NEE + balance-heuristic MIS against the scattering-only estimator, unguided and
    guided (b = 1 after the first frame): all three must share one mean.  A light
    occluding its own shadow rays, or mismatched MIS pdfs, shows up here."""
    common = dict(width=64, height=64, collect=False, ramp=False, schedule_m=1, schedule_b=1)
    bf = frame_means(scene, 161, seed=21, guiding=False, nee=False, **common)
    mis = frame_means(scene, 161, seed=22, guiding=False, nee=True, **common)
    gmis = frame_means(scene, 161, seed=23, guiding=True, nee=True, **common)
    for other in (mis, gmis):
        se = np.sqrt(bf.var(ddof=1) / bf.size + other.var(ddof=1) / other.size)
        assert abs(bf.mean() - other.mean()) <= 3.5 * se, (bf.mean(), other.mean(), se)


def test_guiding_lowers_mape_on_the_box():
    """Direction of effect on the directly lit Cornell box (PAPER Table 3 'Box' is lit
    directly too): at 512 spp the guided render's MAPE against a 16k-spp unguided reference
    is lower than the unguided render's (0.87x measured: NEE already handles most of this
    scene's light).  SPEC acceptance 7 itself is the indirect box below."""
    def render(guiding, spp, seed, collect):
        g, r = make(nasg.SCENE_BOX, width=128, height=128, seed=seed, guiding=guiding, collect=collect,
                    ramp=guiding)
        try:
            for _ in range(spp):
                r.iteration()
            return r.image()
        finally:
            r.close()
            g.close()
    ref = render(False, 16384, 99, False)
    u = nasg.mape(render(False, 512, 1, False), ref)
    gd = nasg.mape(render(True, 512, 1, True), ref)
    assert gd < 0.95 * u, (gd, u)


@pytest.mark.parametrize("seed", [1, 2])
def test_spec_acceptance_7_indirect_box(seed):
    """SPEC acceptance 7: on the shipped indirect-illumination box at 512 spp with a fixed
    seed, guided MAPE <= 0.8x unguided MAPE (reference: 16k-spp unguided render, distinct
    seed; SPEC defaults N = 8, S = 2^16, t = 2^12, e = 0.2, M = 4, B = 64, ramp on).
    Measured 0.715 (seed 1) and 0.730 (seed 2), profiles/r2_indirect_probe.txt."""
    def render(guiding, spp, s):
        g, r = make(nasg.SCENE_INDIRECT, width=128, height=128, seed=s, guiding=guiding, collect=guiding,
                    ramp=guiding)
        try:
            for _ in range(spp):
                r.iteration()
            return r.image()
        finally:
            r.close()
            g.close()
    ref = render(False, 16384, 99)
    u = nasg.mape(render(False, 512, seed), ref)
    gd = nasg.mape(render(True, 512, seed), ref)
    assert gd <= 0.8 * u, (gd, u, gd / u)


def test_spec_acceptance_9_determinism_on_the_indirect_box():
    """SPEC acceptance 9: two full guided renders of acceptance 7's scene at 32 spp with
    identical configs (SPEC defaults, online training on) give bitwise-identical films
    and network weights."""
    out = []
    for _ in range(2):
        g, r = make(nasg.SCENE_INDIRECT, width=128, height=128, seed=1)
        try:
            for _ in range(32):
                r.iteration()
            out.append((np.asarray(r.image()).copy(), g.get_weights()))
        finally:
            r.close()
            g.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
