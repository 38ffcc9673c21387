"""BASELINE config 3 — online training, 2^18 radiance samples per Adam step:
the GPU loss curve and network outputs track the reference over 100 steps
from the same init (north_star: "mixture parameters and loss must track the
reference over 100 training steps").

Golden data (tests/golden/make_train_curve.py):
  train_curve_ref.npz — the unmodified reference (oracle/_ref), 100 steps,
                        fresh synthetic buffer per step, b = min(1, k/64);
  train_curve_rev.npz — the same with the dW reduction summed in reverse row
                        order: how far fp32 reassociation alone moves the
                        trajectory (the yardstick for the tolerance).
Metric: |loss_gpu - loss_ref| / mean|loss_ref| per step; network outputs on
the golden 1024-query probe set, relative L2, after steps 10/25/50/100.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2303_08064_b200 as nasg  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
N = 1 << 18


def _load(name):
    p = os.path.join(GOLDEN, name)
    if not os.path.exists(p):
        pytest.skip(f"{name} not generated")
    return np.load(p)


def run_curve(precision, steps, probe_q9):
    g = nasg.Guide(nasg.TrainerConfig(seed=3, sample_capacity=N, batch_size=N))
    g.train_precision = precision
    dev = [torch.from_numpy(np.ascontiguousarray(np.pad(probe_q9[:, k:k + 3], ((0, 0), (0, 1))))).cuda()
           for k in (0, 3, 6)]
    losses, probes = [], {}
    for k in range(steps):
        s = torch.from_numpy(nasg.synth_samples(1000 + k, N)).cuda()
        st = g.train_iteration(s, min(1.0, k / 64.0))
        assert st.steps == 1
        losses.append(st.mean_loss)
        if k + 1 in (10, 25, 50, 100):
            probes[k + 1] = g.query_raw(*dev).cpu().numpy()
    g.close()
    return np.array(losses), probes


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def test_fp32_training_tracks_reference_100_steps():
    ref, rev = _load("train_curve_ref.npz"), _load("train_curve_rev.npz")
    lr, lv = ref["losses"], rev["losses"]
    steps = len(lr)
    losses, probes = run_curve(nasg.NASG_MLP_FP32, steps, ref["probe_q9"])
    scale = np.abs(lr).mean()
    d_gpu = np.abs(losses - lr) / scale
    d_rev = np.abs(lv[:steps] - lr) / scale
    print("loss dev gpu max/mean", d_gpu.max(), d_gpu.mean(), "rev", d_rev.max(), d_rev.mean())
    # before chaotic amplification: same order as fp32 reassociation alone
    # (measured: gpu 1.1e-5, rev 5.5e-6 over the first 5 steps)
    assert d_gpu[:5].max() <= 5 * d_rev[:5].max() + 1e-6
    assert d_gpu.max() <= 5 * d_rev.max() + 1e-3
    for k in (10, 25, 50, 100):
        if f"probe_{k}" not in ref or k > steps:
            continue
        dg, dr = rel_l2(probes[k], ref[f"probe_{k}"]), rel_l2(rev[f"probe_{k}"], ref[f"probe_{k}"])
        print(f"probe after {k}: gpu {dg:.3e} rev {dr:.3e}")
        assert dg <= 5 * dr + 1e-3, (k, dg, dr)


def test_bf16_training_tracks_reference_100_steps():
    """The tensor-core trainer follows the reference's curve and, on the probe
    set, stays within 3x of the reference's own reassociation drift."""
    ref = _load("train_curve_ref.npz")
    lr = ref["losses"]
    losses, probes = run_curve(nasg.NASG_MLP_BF16, len(lr), ref["probe_q9"])
    scale = np.abs(lr).mean()
    d = np.abs(losses - lr) / scale
    # moving average over 10 steps: the curve, not the per-step noise
    ma = np.convolve(losses - lr, np.ones(10) / 10, mode="valid") / scale
    print("bf16 loss dev max", d.max(), "moving-average max", np.abs(ma).max())
    for k in (10, 25, 50, 100):
        print(f"bf16 probe after {k}: {rel_l2(probes[k], ref[f'probe_{k}']):.3e}")
    # f16 forward / scaled f16 backward (k_train_tc.cu): measured moving-average
    # deviation 2.9 %, probe rel-L2 0.060 / 0.089 / 0.099 / 0.133 after
    # 10 / 25 / 50 / 100 steps vs the reversed-sum reference's 0.031 / 0.090 /
    # 0.102 / 0.126 (the fp32 trainer: 0.040 / 0.098 / 0.107 / 0.131)
    assert np.abs(ma).max() <= 0.06
    rev = _load("train_curve_rev.npz")
    for k in (10, 25, 50, 100):
        dr = rel_l2(rev[f"probe_{k}"], ref[f"probe_{k}"])
        assert rel_l2(probes[k], ref[f"probe_{k}"]) <= 3 * dr + 1e-3, k
