"""GPU parity of the training path (K5 KL gradient, K6 backward, K8 Adam,
Trainer::train_iteration) against the CPU oracle.

Tolerances: the GPU computes the KL gradient in fp32 (the reference in
double, cast to float) and sums dW in a different order, so
  * per-step gradient: relative L2 error <= 1e-4 over all 49,280 entries;
  * Trainer iterations (fp32 Adam, bit-identical update formula):
    mean loss within 1e-4 relative and weights within 1e-3 relative L2
    after 3 iterations x 8 Adam steps from the same init.
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
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def _oracle_grad(orc, w, samples, b, e=0.2):
    """dW of one step on `samples` (in order), as guiding.cpp:242-273."""
    q9 = np.concatenate([samples[:, 0:3], samples[:, 4:7], samples[:, 8:11]], 1)
    enc, _ = orc.encode(q9, H.BMIN, H.BMAX)
    raw = orc.forward(w, enc)
    g, ok, loss = orc.kl_grad(raw, samples, b, e)
    og = (g * (1.0 / len(samples))).astype(np.float32)
    return orc.backward(w, enc, og), ok, loss


@pytest.mark.parametrize("b", [0.0, 1.0])
def test_single_step_gradient_matches_oracle(orc, b):
    g = nasg.Guide(nasg.TrainerConfig(seed=77, batch_size=3000, sample_capacity=3000))
    rng = np.random.default_rng(int(b * 10) + 1)
    s = H.samples(rng, 3000)
    w0 = g.get_weights()
    ds = torch.from_numpy(s).cuda()
    g.train_step(ds, None, len(s), len(s), b)
    grad = g.last_grad()
    ref, ok, loss = _oracle_grad(orc, w0, s, b)
    assert rel_l2(grad, ref) <= 1e-4, rel_l2(grad, ref)
    st = g.train_stats_take()
    assert st.steps == 1 and st.dropped_samples == int((~ok).sum())
    fin = ok & np.isfinite(loss)
    assert st.mean_loss == pytest.approx(loss[fin].mean(), rel=1e-4)
    g.close()


def test_train_iterations_track_oracle(orc):
    cfg = dict(capacity=4096, batch=512, seed=21)
    s = H.samples(np.random.default_rng(13), 3000)
    t_ref = orc.trainer(**cfg)
    g = nasg.Guide(nasg.TrainerConfig(seed=21, sample_capacity=4096, batch_size=512))
    ds = torch.from_numpy(s).cuda()
    for b in (0.0, 0.5, 1.0):
        st = g.train_iteration(ds, b)
        sr = t_ref.train(s, b)
        assert st.steps == sr["steps"] == 8
        assert st.dropped_samples == sr["dropped"] and st.skipped_updates == sr["skipped"] == 0
        assert st.mean_loss == pytest.approx(sr["mean_loss"], rel=1e-4)
        assert rel_l2(g.get_weights(), t_ref.weights()) <= 1e-3
    # publish happened: the snapshot equals the live weights
    assert np.array_equal(g.get_weights(published=True), g.get_weights())
    assert g.adam_t == 24
    g.close()


def test_adam_skip_on_nonfinite(orc):
    """Overflowing weights -> every row dropped, dW = inf*0 = NaN -> whole update skipped
    (net.hpp:140-144) — same counters as the reference."""
    w = orc.init_network(5)
    w[: 64 * 128] *= 1e37
    s = H.samples(np.random.default_rng(4), 600, zero_p_frac=0.0)
    t_ref = orc.trainer(capacity=1024, batch=256, seed=5)
    t_ref.set_weights(w)
    g = nasg.Guide(nasg.TrainerConfig(seed=5, sample_capacity=1024, batch_size=256))
    g.set_weights(w)
    st = g.train_iteration(torch.from_numpy(s).cuda(), 1.0)
    sr = t_ref.train(s, 1.0)
    assert (st.steps, st.skipped_updates, st.dropped_samples) == (sr["steps"], sr["skipped"], sr["dropped"])
    assert st.skipped_updates == 4
    assert np.array_equal(g.get_weights(), w)
    assert g.adam_t == 0
    g.close()


def test_empty_buffer_noop():
    g = nasg.Guide(nasg.TrainerConfig(seed=9))
    w0 = g.get_weights()
    st = g.train_iteration(None, 1.0)
    assert st.steps == 0 and np.array_equal(g.get_weights(), w0)
    g.close()


def test_data_parallel_shards_equal_full_batch(orc):
    """Fake multi-GPU: per-shard unnormalised gradients with the global 1/count
    scaling sum to the single-batch gradient (the NCCL allreduce contract)."""
    s = H.samples(np.random.default_rng(17), 4000)
    g = nasg.Guide(nasg.TrainerConfig(seed=31))
    w0 = g.get_weights()
    ds = torch.from_numpy(s).cuda()
    order = torch.arange(len(s), dtype=torch.int32, device="cuda")
    parts = []
    for lo, hi in ((0, 1500), (1500, 4000)):
        g.set_weights(w0)
        g.train_step(ds, order[lo:], hi - lo, len(s), 1.0)
        parts.append(g.last_grad().astype(np.float64))
    g.set_weights(w0)
    g.train_step(ds, order, len(s), len(s), 1.0)
    full = g.last_grad()
    assert rel_l2(parts[0] + parts[1], full) <= 1e-5
    g.close()


def test_checkpoint_roundtrip_with_oracle(orc, tmp_path):
    g = nasg.Guide(nasg.TrainerConfig(seed=44))
    p = str(tmp_path / "w.nasg")
    g.save_checkpoint(p)
    w, n = orc.load_checkpoint(p)
    assert n == 8 and np.array_equal(w, g.get_weights())
    w2 = orc.init_network(45)
    orc.save_checkpoint(p, w2)
    g.load_checkpoint(p)
    assert np.array_equal(g.get_weights(published=True), w2)
    with open(p, "r+b") as f:
        f.write(b"JUNK")
    with pytest.raises(nasg.NasgError):
        g.load_checkpoint(p)
    g.close()
