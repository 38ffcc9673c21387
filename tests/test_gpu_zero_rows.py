"""Zero-gradient rows in the bf16 trainer (nasg_set_zero_row_skip).

Rows with p = 0 get a zero gradient from kl_loss_gradient (guiding.cpp:112)
and loss 0 from loss_surrogate (:170), counted (:267-270).  With skipping on
they are classified out of the network pass (train_classify_kernel); the step
must produce the same gradient (up to the tensor core's summation order), the
same TrainStats counts, the same loss, and the same encode clamp count, and
rows whose output could be non-finite (non-finite inputs; weights >= 1e7)
must still take the full path, where the reference drops them (:247-250).
The classification runs for steps with more 128-row tiles than SMs (148 on a
B200), so every case here is larger than 148 x 128 = 18,944 rows.
"""
import numpy as np
import pytest

import nasg_testutil as H

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2303_08064_b200 as nasg  # noqa: E402


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / nb if nb > 0 else np.linalg.norm(a)


def step(s, skip, n_comp=8, weights=None, outside=False, prec=nasg.NASG_MLP_BF16):
    n = len(s)
    g = nasg.Guide(nasg.TrainerConfig(seed=13, batch_size=n, sample_capacity=n, n_components=n_comp))
    g.train_precision = prec
    g.zero_row_skip = skip
    if weights is not None:
        g.set_weights(weights)
    g.reset_encode_clamp_count()
    g.train_step(torch.from_numpy(s).cuda(), None, n, n, 1.0)
    grad = g.last_grad()
    st = g.train_stats_take()
    clamps = g.encode_clamp_count
    w = g.get_weights()
    g.close()
    return grad, st, clamps, w


def stats_equal(a, b, n):
    assert a.steps == b.steps == 1
    assert a.dropped_samples == b.dropped_samples
    assert a.skipped_updates == b.skipped_updates
    # the per-row losses are the same arithmetic; a small step runs the KL of a
    # tile cooperatively over three warpgroups (float sums in another order)
    assert a.mean_loss == pytest.approx(b.mean_loss, rel=1e-6, abs=1e-12)


def outside_positions(s, rng, frac=0.2):
    m = rng.random(len(s)) < frac
    s[m, 0:3] *= 1.7  # some coordinates past the [-1, 1] bounds: clamped by the encode
    return s


@pytest.mark.parametrize("n_comp", [8, 4])
@pytest.mark.parametrize("n,zero_frac", [(20000, 0.5), (1 << 15, 0.5), (40000, 0.95), (25000, 0.0), (20480, 1.0)])
def test_skip_matches_full_pass(n_comp, n, zero_frac):
    rng = np.random.default_rng(n + int(zero_frac * 100))
    s = outside_positions(H.samples(rng, n, zero_p_frac=zero_frac), rng)
    g1, st1, c1, w1 = step(s, True, n_comp)
    g0, st0, c0, w0 = step(s, False, n_comp)
    stats_equal(st1, st0, n)
    assert c1 == c0 > 0
    if zero_frac < 1.0:
        assert rel_l2(g1, g0) <= 2e-4, rel_l2(g1, g0)  # fp32 summation order over other tiles
        # Adam's first step moves every weight by ~lr * sign(g): only entries
        # whose gradient is at rounding level may step the other way
        assert np.mean(np.abs(w1 - w0) > 1e-6) <= 1e-3
    else:  # every row zero: zero gradient, the Adam step is still taken
        assert not np.any(g1) and not np.any(g0)
        assert st1.mean_loss == 0.0 and st1.skipped_updates == 0


@pytest.mark.parametrize("n,zero_frac", [(20000, 0.5), (40000, 0.95), (12000, 1.0)])
def test_skip_matches_full_pass_fp32_trainer(n, zero_frac):
    """The fp32 (FFMA) trainer classifies too (steps with more 64-row tiles than SMs):
    the same gradient up to fp32 summation order, counts, loss and clamp counts."""
    rng = np.random.default_rng(n + 7)
    s = outside_positions(H.samples(rng, n, zero_p_frac=zero_frac), rng)
    g1, st1, c1, w1 = step(s, True, prec=nasg.NASG_MLP_FP32)
    g0, st0, c0, w0 = step(s, False, prec=nasg.NASG_MLP_FP32)
    stats_equal(st1, st0, n)
    assert c1 == c0 > 0
    if zero_frac < 1.0:
        assert rel_l2(g1, g0) <= 1e-5, rel_l2(g1, g0)
    else:
        assert not np.any(g1) and not np.any(g0)


def test_nonfinite_inputs_with_zero_p_are_dropped_like_the_reference():
    rng = np.random.default_rng(3)
    n = 1 << 15
    s = H.samples(rng, n, zero_p_frac=0.5)
    bad = np.arange(0, n, 997)
    s[bad, 3] = 0.0
    s[bad[::3], 4] = np.nan            # omega_o
    s[bad[1::3], 10] = np.inf          # normal
    s[bad[2::3], 0] = np.nan           # position
    g1, st1, _, _ = step(s, True)
    g0, st0, _, _ = step(s, False)
    stats_equal(st1, st0, n)
    assert st0.dropped_samples >= len(bad[::3]) + len(bad[1::3])
    # a non-finite input row poisons dW (h^T delta with NaN h), like the
    # reference's backward: the same non-finite entries, the step skipped
    assert np.array_equal(np.isfinite(g1), np.isfinite(g0)) and st1.skipped_updates == st0.skipped_updates
    f = np.isfinite(g0)
    assert rel_l2(g1[f], g0[f]) <= 1e-4  # the finite entries: small sums, summation order


def test_large_weights_disable_the_skip():
    """With a weight >= 1e7 the forward of a p = 0 row may overflow (the
    reference then drops it): every row takes the full path again."""
    rng = np.random.default_rng(4)
    n = 1 << 15
    s = H.samples(rng, n, zero_p_frac=0.5)
    w = nasg.Guide(nasg.TrainerConfig(seed=13)).get_weights().copy()
    w[:64 * 128] *= 3e3   # layer 1 x 3e3 and one weight past the bound
    w[5] = 2e7
    g1, st1, _, _ = step(s, True, weights=w)
    g0, st0, _, _ = step(s, False, weights=w)
    stats_equal(st1, st0, n)
    assert np.array_equal(g1, g0)  # the same full pass, bit for bit


def test_train_iteration_shuffled_steps():
    """S = 2^16, t = 2^15, nu = 2: four shuffled minibatch steps per iteration
    (the epoch permutation composed into the row list), half the rows zero:
    the same trajectory either way."""
    n = 1 << 16
    s = nasg.synth_samples(7, n)
    out = []
    for skip in (True, False):
        g = nasg.Guide(nasg.TrainerConfig(seed=5, batch_size=1 << 15, step_factor=2))
        g.train_precision = nasg.NASG_MLP_BF16
        g.zero_row_skip = skip
        ds = torch.from_numpy(s).cuda()
        sts = [g.train_iteration(ds, 0.5) for _ in range(2)]
        out.append((sts, g.get_weights()))
        g.close()
    (a, wa), (b, wb) = out
    for x, y in zip(a, b):
        assert x.steps == y.steps == 4 and x.dropped_samples == y.dropped_samples
        assert x.mean_loss == pytest.approx(y.mean_loss, rel=1e-4)
    assert rel_l2(wa, wb) <= 1e-3  # 8 Adam steps amplify summation-order noise
