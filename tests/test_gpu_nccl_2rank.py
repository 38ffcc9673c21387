"""Two-rank data-parallel training over a real NCCL communicator on two GPUs
(SURVEY §8(e)): each rank trains on its own shard of the sample buffer, every
Adam step allreduces the unnormalised dW (one grouped NCCL launch with the step
statistics) and the global 1/count scaling (guiding.cpp:262) makes the update
the one of the union batch.  Skipped when fewer than two GPUs are visible.

With S = t (every step spans each rank's whole shard) the step's row set is
the union whatever the shuffle, so the 2-rank result must equal a 1-GPU
context trained on the union buffer up to fp32 summation order, and the two
ranks must hold bit-identical weights.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available() or torch.cuda.device_count() < 2:  # pragma: no cover
    pytest.skip("needs two CUDA devices", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

import paper_2303_08064_b200 as nasg  # noqa: E402

N0, N1 = 3000, 5192  # uneven shards; union 8192


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, prec, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    allsamp = nasg.synth_samples(31, N0 + N1)
    mine = allsamp[:N0] if rank == 0 else allsamp[N0:]
    g = nasg.Guide(nasg.TrainerConfig(seed=5, sample_capacity=N0 + N1, batch_size=N0 + N1), device=rank)
    g.train_precision = prec
    uid = [nasg.Guide.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    g.comm_init(uid[0], rank, 2)
    s = torch.from_numpy(mine).cuda()
    stats = [g.train_iteration(s, 0.5) for _ in range(3)]
    c = g.counters()
    q.put((rank, g.get_weights(), [(x.steps, x.mean_loss, x.dropped_samples, x.skipped_updates) for x in stats],
           c["collectives"], c["nranks"], torch.cuda.current_device()))
    g.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("prec", [nasg.NASG_MLP_FP32, nasg.NASG_MLP_BF16])
def test_two_rank_train_iteration_equals_union_batch(prec):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, port, prec, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    (_, w0, st0, coll0, nr0, dev0), (_, w1, st1, coll1, nr1, dev1) = res
    assert (nr0, nr1, dev0, dev1) == (2, 2, 0, 1)
    assert coll0 == coll1 == 3 + 3  # 3 iterations x (1 step exchange + 1 allgather)
    assert np.array_equal(w0.view(np.uint32), w1.view(np.uint32))  # identical replicas
    assert st0 == st1  # the step statistics are global
    # the union buffer on one GPU
    g = nasg.Guide(nasg.TrainerConfig(seed=5, sample_capacity=N0 + N1, batch_size=N0 + N1), device=0)
    g.train_precision = prec
    s = torch.from_numpy(nasg.synth_samples(31, N0 + N1)).cuda(0)
    w_init = g.get_weights()
    ref = [g.train_iteration(s, 0.5) for _ in range(3)]
    wr = g.get_weights()
    g.close()
    for (steps, loss, dropped, skipped), r in zip(st0, ref):
        assert (steps, dropped, skipped) == (r.steps, r.dropped_samples, r.skipped_updates)
        assert abs(loss - r.mean_loss) <= 1e-5 * abs(r.mean_loss)
    # Adam turns components that are pure rounding noise into +-lr steps, so the
    # bar is on the update: <= 5 % of its norm (a sign flip on <= 0.25 % of the
    # components), not on the weights' last bits
    err = np.linalg.norm(w0.astype(np.float64) - wr) / np.linalg.norm(wr.astype(np.float64) - w_init)
    assert err <= 0.05, err
