"""The data-parallel exchange path of Trainer::train_iteration on a real NCCL
communicator: with a communicator attached, every Adam step
allreduces the unnormalised dW and the step statistics, re-checks the summed
gradient for non-finite entries and only then runs Adam (guiding.cpp:244-273,
net.hpp:137-158).

The pool has one GPU, so the communicator here has one rank: the exchange is
an identity, and the weights, Adam moments and statistics must be
bit-identical to a context without a communicator on the same samples — the
check that the NCCL code path itself (allreduce, allgather of buffer sizes,
finite re-check) is wired correctly.  The N > 1 rank/plan/shard logic is
covered with gloo in test_multi_rank.py, and on two GPUs (when present) by
tests/test_gpu_nccl_2rank.py.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2303_08064_b200 as nasg  # noqa: E402


def _train(prec, samples, comm, iters=2):
    g = nasg.Guide(nasg.TrainerConfig(seed=5, sample_capacity=len(samples), batch_size=2048))
    g.train_precision = prec
    if comm:
        g.comm_init(nasg.Guide.comm_unique_id(), 0, 1)
    l0, c0 = g.kernel_launches, g.counters()["collectives"]
    stats = [g.train_iteration(samples, 0.5) for _ in range(iters)]
    torch.cuda.synchronize()
    launches = g.kernel_launches - l0
    coll = g.counters()["collectives"] - c0
    w = g.get_weights()
    g.close()
    return w, stats, launches, coll


@pytest.mark.parametrize("prec", [nasg.NASG_MLP_FP32, nasg.NASG_MLP_BF16])
def test_one_rank_nccl_exchange_is_bit_identical(prec):
    s = torch.from_numpy(nasg.synth_samples(21, 8192)).cuda()
    w_ref, st_ref, l_ref, c_ref = _train(prec, s, comm=False)
    w_dp, st_dp, l_dp, c_dp = _train(prec, s, comm=True)
    steps = sum(x.steps for x in st_ref)
    assert steps == 8  # 2 iterations x ceil(8192 / 2048)
    # the exchange really ran: one grouped allreduce per Adam step plus one
    # buffer-size allgather per iteration, and no extra kernel of ours (the
    # finite re-check of the reduced gradient is inside the Adam launch)
    assert c_ref == 0 and c_dp == steps + 2
    assert l_dp == l_ref
    assert np.array_equal(w_ref.view(np.uint32), w_dp.view(np.uint32))
    for a, b in zip(st_ref, st_dp):
        assert (a.steps, a.dropped_samples, a.skipped_updates) == (b.steps, b.dropped_samples, b.skipped_updates)
        assert a.mean_loss == b.mean_loss


def test_one_rank_nccl_empty_buffer_is_noop():
    g = nasg.Guide(nasg.TrainerConfig(seed=5))
    g.comm_init(nasg.Guide.comm_unique_id(), 0, 1)
    w0 = g.get_weights()
    st = g.train_iteration(None, 1.0)
    assert st.steps == 0
    assert np.array_equal(w0, g.get_weights())
    g.close()


def test_one_rank_nccl_render_loop_is_bit_identical():
    # the guided render loop (configs 4-5) trains through the same exchange: with a
    # one-rank communicator the film and the weights must not change by a bit
    lo, hi = nasg.scene_bounds(nasg.SCENE_BOX)
    out = []
    for comm in (False, True):
        g = nasg.Guide(nasg.TrainerConfig(seed=7), bmin=lo, bmax=hi)
        g.precision = g.train_precision = nasg.NASG_MLP_BF16
        if comm:
            g.comm_init(nasg.Guide.comm_unique_id(), 0, 1)
        r = nasg.Render(g, scene=nasg.SCENE_BOX, width=80, height=64, schedule_m=1, schedule_b=4)
        try:
            for _ in range(4):
                r.iteration()
            out.append((r.image(), g.get_weights()))
        finally:
            r.close()
            g.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1].view(np.uint32), out[1][1].view(np.uint32))


@pytest.mark.parametrize("prec", [nasg.NASG_MLP_FP32, nasg.NASG_MLP_BF16])
def test_one_rank_nccl_skip_on_reduced_nonfinite(prec):
    """A NaN weight on the constant pad input makes every dW entry NaN; with a
    communicator the skip decision is re-taken on the allreduced gradient
    inside the (cooperative) Adam launch: every update skipped, weights and
    Adam t untouched (net.hpp:140-144)."""
    w = nasg.Guide(nasg.TrainerConfig(seed=5)).get_weights()
    w[63 * 128 + 0] = np.nan
    s = torch.from_numpy(nasg.synth_samples(4, 600)).cuda()
    g = nasg.Guide(nasg.TrainerConfig(seed=5, sample_capacity=1024, batch_size=256))
    g.train_precision = prec
    g.comm_init(nasg.Guide.comm_unique_id(), 0, 1)
    g.set_weights(w)
    st = g.train_iteration(s, 1.0)
    assert st.steps == 4 and st.skipped_updates == 4  # T = ceil(1024 / 256)
    assert np.array_equal(g.get_weights(), w, equal_nan=True)
    assert g.adam_t == 0
    # the flags were cleared: a clean network trains normally afterwards
    w2 = nasg.Guide(nasg.TrainerConfig(seed=6)).get_weights()
    g.set_weights(w2)
    st = g.train_iteration(s, 1.0)
    assert st.skipped_updates == 0 and g.adam_t == 4
    g.close()


def test_caller_device_is_restored():
    """Every C-ABI call makes the context's device current and restores the
    caller's afterwards (one process may drive several contexts)."""
    dev = torch.cuda.current_device()
    g = nasg.Guide(nasg.TrainerConfig(seed=1), device=dev)
    assert torch.cuda.current_device() == dev
    g.close()
