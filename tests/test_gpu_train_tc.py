"""bf16 tensor-core training path (k_train_tc.cu).

Stated bf16 training contract:
  * the step computes exactly the bf16 pipeline it claims: bf16 activations,
    double KL gradient of the fp32 raw outputs scaled by 1/count and rounded
    to bf16, bf16 deltas through W^T with the ReLU gates, dW in fp32 from
    bf16 operands — vs a numpy emulation of that pipeline, rel-L2 <= 2e-3
    (accumulation order; one-ulp bf16 flips);
  * vs the fp32 reference gradient: rel-L2 <= 0.35 (measured 0.13-0.22: bf16
    activations and deltas, 8-bit mantissas, summed over thousands of rows
    with cancellation);
  * the loss of a multi-iteration run tracks the fp32 reference within 6 %.
"""
import numpy as np
import pytest

import nasg_testutil as H

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2303_08064_b200 as nasg  # noqa: E402
from test_gpu_tc import bf16  # noqa: E402

DIMS = [64, 128, 128, 128, 65]


def split_w(w):
    out, off = [], 0
    for l in range(4):
        n = DIMS[l] * DIMS[l + 1]
        out.append(w[off:off + n].reshape(DIMS[l], DIMS[l + 1]).astype(np.float64))
        off += n
    return out


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def emulate_bf16_step(orc, w, samples, b, count):
    q9 = np.concatenate([samples[:, 0:3], samples[:, 4:7], samples[:, 8:11]], 1)
    enc, _ = orc.encode(q9, H.BMIN, H.BMAX)
    W = [bf16(x.astype(np.float32)).astype(np.float64) for x in split_w(w)]
    hs = [bf16(enc).astype(np.float64)]
    for l in range(3):
        hs.append(bf16(np.maximum(hs[-1] @ W[l], 0).astype(np.float32)).astype(np.float64))
    raw = (hs[3] @ W[3]).astype(np.float32)
    g, ok, _ = orc.kl_grad(raw, samples, b)
    d = bf16((g * (1.0 / count)).astype(np.float32)).astype(np.float64)
    dw = [None] * 4
    for l in (3, 2, 1, 0):
        dw[l] = hs[l].T @ d
        if l > 0:
            d = bf16(((d @ W[l].T) * (hs[l] > 0)).astype(np.float32)).astype(np.float64)
    return np.concatenate([x.ravel() for x in dw])


@pytest.mark.parametrize("n", [3000, 1 << 15])
def test_tc_gradient_matches_bf16_emulation(orc, n):
    s = H.samples(np.random.default_rng(n), n)
    g = nasg.Guide(nasg.TrainerConfig(seed=77, batch_size=n, sample_capacity=n))
    g.train_precision = nasg.NASG_MLP_BF16
    w0 = g.get_weights()
    g.train_step(torch.from_numpy(s).cuda(), None, n, n, 1.0)
    grad = g.last_grad()
    emu = emulate_bf16_step(orc, w0, s, 1.0, n)
    assert rel_l2(grad, emu) <= 2e-3, rel_l2(grad, emu)
    # vs the fp32 reference pipeline
    q9 = np.concatenate([s[:, 0:3], s[:, 4:7], s[:, 8:11]], 1)
    enc, _ = orc.encode(q9, H.BMIN, H.BMAX)
    gr, ok, loss = orc.kl_grad(orc.forward(w0, enc), s, 1.0)
    ref = orc.backward(w0, enc, (gr * (1.0 / n)).astype(np.float32))
    assert rel_l2(grad, ref) <= 0.35, rel_l2(grad, ref)
    st = g.train_stats_take()
    assert st.steps == 1 and abs(st.dropped_samples - int((~ok).sum())) <= max(2, n // 1000)
    g.close()


def test_tc_training_loss_tracks_reference(orc):
    n = 4096
    s = nasg.synth_samples(5, n)
    t_ref = orc.trainer(capacity=4096, batch=1024, seed=21)
    g = nasg.Guide(nasg.TrainerConfig(seed=21, sample_capacity=4096, batch_size=1024))
    g.train_precision = nasg.NASG_MLP_BF16
    ds = torch.from_numpy(s).cuda()
    for it in range(4):
        b = min(1.0, it / 2)
        st = g.train_iteration(ds, b)
        sr = t_ref.train(s, b)
        assert st.steps == sr["steps"] == 4 and st.skipped_updates == 0
        assert st.mean_loss == pytest.approx(sr["mean_loss"], rel=6e-2)
    g.close()


def test_tc_training_empty_and_ragged():
    g = nasg.Guide(nasg.TrainerConfig(seed=2, sample_capacity=1000, batch_size=333))
    g.train_precision = nasg.NASG_MLP_BF16
    s = torch.from_numpy(nasg.synth_samples(1, 999)).cuda()
    st = g.train_iteration(s, 1.0)
    assert st.steps == 4 and st.skipped_updates == 0 and np.isfinite(st.mean_loss)
    assert g.train_iteration(None, 1.0).steps == 0
    g.close()
