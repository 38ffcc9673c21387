"""Multi-rank (data-parallel training) host logic on CPU with gloo, world_size 2.

The GPU pool of this project has one GPU, so NCCL itself cannot run here; what
is tested is everything around it:
  * the data-parallel plan (nasg_dp_plan): identical global counts on all
    ranks, local counts summing to them, the single-rank plan equal to the
    reference's step loop (guiding.cpp:204-243);
  * the exchange contract the NCCL allreduce implements: rank-local gradients
    with the GLOBAL 1/count scaling (guiding.cpp:262), summed across ranks,
    equal the single-process gradient of the union batch; the skip decision on
    the reduced gradient and the Adam update are then identical on all ranks.
The per-rank gradients come from the CPU oracle; the collective is gloo.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import nasg_testutil as H
import paper_2303_08064_b200 as nasg


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_single_rank_plan_is_reference_loop():
    cfg = nasg.TrainerConfig(sample_capacity=4096, batch_size=512)
    loc, glo, res = nasg.dp_plan(cfg, [3000], 0)
    assert list(loc) == [512] * 5 + [440, 512, 512]  # count = min(t, n - cursor), reshuffle at epoch end
    assert list(glo) == list(loc)
    assert list(res) == [True, False, False, False, False, False, True, False]
    loc, glo, res = nasg.dp_plan(nasg.TrainerConfig(), [65536], 0)  # S=2^16, t=2^12 -> 16 steps
    assert len(loc) == 16 and (loc == 4096).all()
    loc, _, _ = nasg.dp_plan(nasg.TrainerConfig(), [0], 0)
    assert len(loc) == 0  # empty buffer: no-op


def test_uneven_plan_properties():
    cfg = nasg.TrainerConfig(sample_capacity=1 << 14, batch_size=1000, step_factor=2)
    n_all = [7, 0, 5000, 333]
    plans = [nasg.dp_plan(cfg, n_all, r) for r in range(len(n_all))]
    glo = plans[0][1]
    for p in plans:
        assert np.array_equal(p[1], glo)
    assert np.array_equal(sum(p[0] for p in plans), glo)
    assert (plans[1][0] == 0).all()  # an empty rank still participates with 0 rows
    assert abs(glo[0] - 1000) <= len(n_all)


def _worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle
    orc = Oracle("orc")
    cfg = nasg.TrainerConfig(sample_capacity=2048, batch_size=1024, seed=9)
    # this rank's tile of the sample buffer
    all_samples = H.samples(np.random.default_rng(123), 3000)
    lo, hi = (0, 1200) if rank == 0 else (1200, 3000)
    mine = all_samples[lo:hi]
    n_all = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(n_all, torch.tensor([len(mine)], dtype=torch.int64))
    n_all = [int(x.item()) for x in n_all]
    loc, glo, _ = nasg.dp_plan(cfg, n_all, rank)
    plans = [torch.zeros(len(glo), dtype=torch.int64) for _ in range(world)]
    dist.all_gather(plans, torch.from_numpy(glo.copy()))
    assert all(torch.equal(p, plans[0]) for p in plans)
    # step 0: local rows (identity order) with the global 1/count scaling
    w = orc.init_network(cfg.seed)
    rows = mine[: loc[0]]
    q9 = np.concatenate([rows[:, 0:3], rows[:, 4:7], rows[:, 8:11]], 1)
    enc, _ = orc.encode(q9, H.BMIN, H.BMAX)
    g, ok, _ = orc.kl_grad(orc.forward(w, enc), rows, 1.0)
    dw = orc.backward(w, enc, (g * (1.0 / glo[0])).astype(np.float32))
    t = torch.from_numpy(dw.astype(np.float64))
    dist.all_reduce(t)
    reduced = t.numpy().astype(np.float32)
    nonfinite = torch.tensor([0 if np.isfinite(reduced).all() else 1])
    dist.all_reduce(nonfinite, op=dist.ReduceOp.MAX)
    wn, m, v = w.copy(), np.zeros_like(w), np.zeros_like(w)
    ok_step, tt = orc.adam_step(wn, m, v, reduced, 0)
    digest = torch.tensor([float(np.frombuffer(wn.tobytes(), np.uint32).astype(np.uint64).sum() % (1 << 50))],
                          dtype=torch.float64)
    digests = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(digests, digest)
    if rank == 0:
        result_q.put((loc[0], glo[0], reduced, int(nonfinite.item()), ok_step,
                      [float(d.item()) for d in digests], (lo, hi)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gradient_exchange_matches_union_batch(orc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    loc0, glo0, reduced, nonfinite, ok_step, digests, _ = res
    assert glo0 == 1024 and nonfinite == 0 and ok_step
    assert digests[0] == digests[1]  # identical Adam update on both ranks
    # the union of both ranks' step-0 rows through one process
    all_samples = H.samples(np.random.default_rng(123), 3000)
    n0 = int(round(1024 * 1200 / 3000))  # the plan's proportional split
    assert loc0 == n0
    rows = np.concatenate([all_samples[:n0], all_samples[1200:1200 + 1024 - n0]])
    q9 = np.concatenate([rows[:, 0:3], rows[:, 4:7], rows[:, 8:11]], 1)
    enc, _ = orc.encode(q9, H.BMIN, H.BMAX)
    w = orc.init_network(9)
    g, ok, _ = orc.kl_grad(orc.forward(w, enc), rows, 1.0)
    full = orc.backward(w, enc, (g * (1.0 / 1024)).astype(np.float32))
    err = np.linalg.norm(reduced.astype(np.float64) - full) / np.linalg.norm(full)
    assert err <= 1e-6, err
