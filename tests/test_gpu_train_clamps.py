"""Encode clamp counter across a multi-epoch train_iteration.

The reference encodes every buffer row once per train_iteration, before the
step loop (guiding.cpp:209-214), so encode_clamp_count (encoding.cpp:8,30)
grows by the buffer's clamped coordinates once per iteration, whatever the
number of epochs (step_factor) or minibatches."""
import numpy as np
import pytest

import nasg_testutil as H

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2303_08064_b200 as nasg  # noqa: E402


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("n,t,nu", [(4096, 1024, 3), (1 << 16, 1 << 14, 2), (3000, 3000, 4)])
def test_clamps_counted_once_per_iteration(precision, n, t, nu):
    rng = np.random.default_rng(n + nu)
    s = H.samples(rng, n, zero_p_frac=0.5)
    s[rng.random(n) < 0.3, 0:3] *= 1.6
    expect = int(np.sum((s[:, 0:3] < -1.0) | (s[:, 0:3] > 1.0)))
    assert expect > 0
    g = nasg.Guide(nasg.TrainerConfig(seed=1, sample_capacity=n, batch_size=t, step_factor=nu))
    g.train_precision = nasg.NASG_MLP_BF16 if precision == "bf16" else nasg.NASG_MLP_FP32
    g.reset_encode_clamp_count()
    ds = torch.from_numpy(s).cuda()
    st = g.train_iteration(ds, 1.0)
    assert st.steps == nu * ((n + t - 1) // t)
    assert g.encode_clamp_count == expect
    g.train_iteration(ds, 1.0)
    assert g.encode_clamp_count == 2 * expect
    g.close()
