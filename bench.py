#!/usr/bin/env python
"""Benchmark of the NASG guided-query hot path (BASELINE.json metric).

One step = one guided query pass (encode -> MLP -> NASG decode -> lobe select
-> sample -> mixture pdf) over one batch of Q synthetic queries (config 2 of
BASELINE.json at its largest size, Q = 2^24 per GPU), inputs resident in HBM.
Queries shard by pixel tile / query range across GPUs with no collective
(weak scaling); value = all ranks' queries / max-over-ranks time.

Also reported (same JSON line):
  e2e          the same metric through the host-buffer API nasg_query_sample_host
               (pinned H2D of the inputs + D2H of the results inside the timed region)
  roofline     the fused query kernel vs the measured bf16 tensor peak
  cpu_baseline the reference (oracle/_ref, all host cores) on a bounded sample
  sweep        config 2: 2^20 - 2^24 queries per batch, bf16 vs fp32 MLP
  train        config 3: fused fwd+KL+bwd+Adam at 2^18 samples per step
  render       configs 4-5: the guided progressive render loop (1024^2 x 512 spp;
               4K sharded by pixel rows over the ranks)

`--impl reference` times the reference's own CPU implementation (oracle/_ref:
the unmodified reference TUs + Eigen-API shim, OpenMP over queries) instead.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "NASG guided queries/sec (fwd+sample+pdf) & train samples/sec, 1–8 B200"
FLOP_PER_QUERY = 2 * (64 * 128 + 128 * 128 + 128 * 128 + 128 * 65)  # 98,560
BYTES_PER_QUERY = 68  # 36 B x/wo/n + 16 B xi in + 16 B dir+pdf out (algorithmic)
FLOP_PER_SAMPLE = 279_296  # fwd 98,560 + dW 98,560 + delta 82,176
# the fp32 (accuracy) path runs on the FFMA pipe: 148 SMs x 128 lanes x 2 FLOP x 1.965 GHz
FP32_FFMA_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12
FP32_PEAK_KIND = "nominal fp32 FFMA (148 SMs x 128 x 2 x 1.965 GHz)"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[2:]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        import torch
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def self_launch(n):
    """`python bench.py --gpus N` outside torchrun: start N ranks (one per GPU) the
    way the driver does and return their exit status."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def max_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def cpu_info():
    """Host CPU model and the cores this process may use (stated beside every CPU number)."""
    model = "unknown"
    try:
        model = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
    except (OSError, StopIteration):
        pass
    usable = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    return {"cpu_model": model, "nproc": usable, "logical_cpus": os.cpu_count()}


def _cpu_oracle():
    """The reference build (oracle/_ref) if present, else the C restatement.  Inputs
    come from the checker's own generator (byte-identical to nasg.synth_*, pinned
    by tests/test_abi.py), so a CPU leg never maps the CUDA library."""
    from oracle.oracle import Oracle, available, LIBS
    kind = "reference" if available("ref") else "port"
    o = Oracle("ref" if kind == "reference" else "orc")
    return o, kind, os.path.relpath(LIBS["ref" if kind == "reference" else "orc"], ROOT)


def cpu_reference_rate(n_total, seconds, threads=None, chunk=1 << 14, steps=None, warmup=1):
    """The reference's own query path (infer_guide + mixture_sample per query,
    guiding.cpp:284-293 + sphdist.cpp:183-198), OpenMP over queries.  With `steps`
    it times exactly that many chunks after `warmup` untimed ones; otherwise it
    runs chunks for up to `seconds`."""
    o, kind, so = _cpu_oracle()
    threads = threads or len(os.sched_getaffinity(0))
    w = o.init_network(0)
    x, wo, nrm, xi = o.synth_queries(12345, chunk)
    q9 = np.ascontiguousarray(np.concatenate([x[:, :3], wo[:, :3], nrm[:, :3]], 1))
    o.query_sample(w, q9[:256], xi[:256], threads=threads)  # thread pool warm-up
    for _ in range(warmup):
        o.query_sample(w, q9, xi, threads=threads)
    done, t0, per = 0, time.perf_counter(), []
    while (done < n_total and time.perf_counter() - t0 < seconds) if steps is None else len(per) < steps:
        t1 = time.perf_counter()
        o.query_sample(w, q9, xi, threads=threads)
        per.append(time.perf_counter() - t1)
        done += chunk
    dt = time.perf_counter() - t0
    return {"value": done / dt, "unit": "queries/s", "cores": threads, "kind": kind, "library": so,
            "ms_per_step": 1e3 * statistics.mean(per),
            "sample": f"{done} synthetic queries in steps of {chunk} (infer_guide+mixture_sample per query, N=8, "
                      f"{threads} OpenMP threads, {dt:.1f} s)", **cpu_info()}


def cpu_reference_train_rate(seconds=8.0):
    """The reference's own Trainer::train_iteration (oracle/_ref, single-threaded by
    design, guiding.cpp:196-282) on config-1 sized buffers (S = 2^14 samples, t = 2^12)."""
    o, kind, so = _cpu_oracle()
    n = 1 << 14
    tr = o.trainer(capacity=n, batch=1 << 12, seed=3)
    s = o.synth_samples(11, n)
    done, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        tr.train(s, 1.0)
        done += n
    dt = time.perf_counter() - t0
    return {"value": done / dt, "unit": "samples/s", "cores": 1, "kind": kind, "library": so,
            "sample": f"{done} synthetic samples through train_iteration (S = t*4 = 16384, 4 Adam steps per call), "
                      f"{dt:.1f} s, 1 thread", **cpu_info()}


def cpu_reference_default_train():
    """One default Trainer::train_iteration (S = 2^16, t = 2^12: 16 Adam steps) of the
    reference (single-threaded by design, guiding.cpp:196-282) — config 1's train leg."""
    o, kind, so = _cpu_oracle()
    n = 1 << 16
    tr = o.trainer(capacity=n, batch=1 << 12, seed=3)
    s = o.synth_samples(11, n)
    t0 = time.perf_counter()
    st = tr.train(s, 1.0)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "samples/s", "seconds_per_iteration": dt, "steps": st["steps"], "cores": 1,
            "kind": kind, "library": so, "sample": "one train_iteration of 65,536 synthetic samples, 1 thread",
            **cpu_info()}


def bench_config(n, ws):
    """The workload both arms report (config 2 of BASELINE.json at its largest size)."""
    return {"workload": f"config 2: {n} guided queries/step/GPU (fwd+sample+pdf), N=8 lobes, "
                        f"64-128-128-128-65 MLP", "queries_per_step_per_gpu": n,
            "l2": "inputs (1 GiB/GPU) exceed the 126 MB L2", "parallelism": f"query shards x{ws}"}


def run_reference(args, ws, rank):
    """`--impl reference`: the reference's own CPU query path on all host cores, on this
    arm's workload; each step is a bounded sample of 2^19 of the config's queries
    (the whole K + W run takes seconds).  Rank 0 alone runs (no CUDA, no NCCL)."""
    if rank != 0:
        return
    chunk = min(args.queries, 1 << 19)
    cb = cpu_reference_rate(0, 0, chunk=chunk, steps=args.steps, warmup=args.warmup)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "queries/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(args.queries, ws),
            "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": "queries/s",
                                        "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if not args.no_train:
        line["train"] = {"cpu_baseline": cpu_reference_train_rate(4.0)}
    print(json.dumps(line), flush=True)


def time_events(fn, k, stream):
    """k back-to-back steps between two CUDA events on `stream` (no event between
    steps: an event record in the stream would cut the programmatic early start
    of each step's first kernel); returns the mean step time k times."""
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(k):
        fn()
    e1.record(stream)
    e1.synchronize()
    t = e0.elapsed_time(e1) * 1e-3
    return [t / k] * k


def bench_train(g_cls, nasg, args, ws, rank, precision):
    """Config 3: S = t = 2^18 samples per Adam step (one step per train_iteration),
    data-parallel over ranks (each rank trains on its own 2^18 samples; with
    N > 1 the dW allreduce runs inside every step)."""
    import torch
    n = args.train_samples
    # global S = t = ws * 2^18: the data-parallel plan gives every rank its own 2^18 rows per step
    g = g_cls(nasg.TrainerConfig(seed=3, sample_capacity=n * ws, batch_size=n * ws), device=torch.cuda.current_device())
    g.train_precision = nasg.NASG_MLP_BF16 if precision == "bf16" else nasg.NASG_MLP_FP32
    if ws > 1:
        import torch.distributed as dist
        uid = [g.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        g.comm_init(uid[0], rank, ws)
    s = torch.from_numpy(nasg.synth_samples(11 + rank, n, first=rank * n)).cuda()
    stream = torch.cuda.current_stream()
    for i in range(3):
        g.train_iteration(s, 1.0, stats=False)
    torch.cuda.synchronize()
    barrier(ws)
    l0 = g.kernel_launches
    times = time_events(lambda: g.train_iteration(s, 1.0, stats=False), args.train_steps, stream)
    launches = g.kernel_launches - l0
    # end to end through the public API: every step copies its 2^18 samples from pinned
    # host memory and reads the step's TrainStats back (train_iteration with stats)
    # (double-buffered: step k + 1's upload runs on a copy stream while step k trains)
    hs = torch.from_numpy(nasg.synth_samples(11 + rank, n, first=rank * n)).pin_memory()
    bufs = [torch.empty_like(s), torch.empty_like(s)]
    cs, cur = torch.cuda.Stream(), torch.cuda.current_stream()
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    trained = [torch.cuda.Event(), torch.cuda.Event()]
    e2e_steps = max(args.train_steps, 40)

    def e2e_trial():
        barrier(ws)
        t0 = time.perf_counter()
        with torch.cuda.stream(cs):
            bufs[0].copy_(hs, non_blocking=True)
            copied[0].record(cs)
        for k in range(e2e_steps):
            b = k % 2
            if k + 1 < e2e_steps:
                with torch.cuda.stream(cs):
                    if k >= 1:
                        cs.wait_event(trained[1 - b])  # step k - 1 is done with that buffer
                    bufs[1 - b].copy_(hs, non_blocking=True)
                    copied[1 - b].record(cs)
            cur.wait_event(copied[b])
            g.train_iteration(bufs[b], 1.0, stats=True)  # TrainStats read back every step
            trained[b].record(cur)
        torch.cuda.synchronize()
        return max_over_ranks(time.perf_counter() - t0, ws)

    trials = sorted(e2e_trial() for _ in range(3))
    te = trials[1]  # the median of three trials (the host-driven loop varies run to run)
    e2e = {"value": n * ws * e2e_steps / te, "unit": "samples/s", "steps": e2e_steps, "trials": 3,
           "trial_values": [n * ws * e2e_steps / x for x in trials], "h2d_bytes_per_step": n * 64 * ws,
           "d2h_bytes_per_step": 40 * ws, "api": "nasg_train_iteration (samples from pinned host memory, stats read back)"}
    # the e2e step's own roofline: one step's 64 B/sample upload alone (CUDA events, best of 3)
    best = float("inf")
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        with torch.cuda.stream(cs):
            bufs[0].copy_(hs, non_blocking=True)
        e1.record(cs)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    e2e["pcie_h2d_gbs_measured"] = hs.numel() * hs.element_size() / best / 1e9
    e2e["h2d_roofline_samples_per_s"] = n * ws / best
    e2e["frac_of_h2d_roofline"] = e2e["value"] / e2e["h2d_roofline_samples_per_s"]
    t = max_over_ranks(sum(times), ws)
    st = g.train_iteration(s, 1.0)
    dense = None
    if precision == "bf16":
        # the same step with every row through the network (zero-row skip off):
        # the dense rate, and the work the skip saves on this buffer
        g.zero_row_skip = False
        for i in range(3):
            g.train_iteration(s, 1.0, stats=False)
        torch.cuda.synchronize()
        barrier(ws)
        td = max_over_ranks(sum(time_events(lambda: g.train_iteration(s, 1.0, stats=False), args.train_steps,
                                            stream)), ws)
        dense = {"value": n * ws * args.train_steps / td, "unit": "samples/s",
                 "ms_per_step": 1e3 * td / args.train_steps,
                 "achieved_tflops": n * args.train_steps * FLOP_PER_SAMPLE / td / 1e12}
        g.zero_row_skip = True
    g.close()
    rate = n * ws * args.train_steps / t
    # rows with p = 0 need no network pass (zero gradient, loss 0: guiding.cpp:112,170):
    # the executed work is the live rows' 279,296 FLOP each
    live = float(np.mean(s[:, 3].cpu().numpy() != 0.0)) if precision == "bf16" else 1.0
    # algorithmic FLOP of the step (279,296 per training sample: fwd + dW +
    # delta) against the bf16 tensor peak; the executed FLOP are the rows that need the
    # network (p != 0, `live_row_fraction`), the zero-gradient rows are classified and
    # counted without it.  The step also moves ~1.7 KB per live row of bf16 activations
    # through HBM twice for the split-K dW GEMM (K_dw is HBM-bound, profiles/r2_ncu_summary.md)
    tf = rate / ws * FLOP_PER_SAMPLE / 1e12
    pk, pk_kind = peaks()
    roof = {"bound": "tensor" if precision == "bf16" else "fp32-ffma", "achieved": tf, "unit": "TFLOP/s",
            "peak": pk["bf16_tflops"] if precision == "bf16" else FP32_FFMA_TFLOPS,
            "peak_kind": f"{pk_kind} bf16 burst" if precision == "bf16" else FP32_PEAK_KIND,
            "live_row_fraction": live, "executed_tflops": tf * live, "executed_frac": None,
            "note": "achieved = samples/s x 279,296 algorithmic FLOP per sample; executed = the rows with "
                    "p != 0, which are the only ones through the network" if precision == "bf16" else "every row"}
    roof["frac"] = tf / roof["peak"]
    roof["executed_frac"] = tf * live / roof["peak"]
    out = {"metric": f"train samples/s (config 3: 2^18 samples/step/GPU, fused fwd+KL+bwd+dW+Adam, {precision})",
           "value": rate, "unit": "samples/s", "ms_per_step": 1e3 * t / args.train_steps,
           "achieved_tflops": tf, "roofline": roof, "e2e": e2e, "dtype": precision,
           "gpu_launches": launches, "last_mean_loss": st.mean_loss}
    if dense:
        out["dense_no_zero_row_skip"] = dense
    return out


def bench_config1(nasg, args, ws, rank):
    """Config 1 of BASELINE.json, the reference's own default case: 65,536 synthetic
    queries (fwd + sample + pdf) and one default train_iteration (S = 2^16 samples,
    t = 2^12 -> 16 Adam steps, guiding.hpp:122-130), on this GPU, beside the same
    workload through oracle/_ref on the host (rank 0 only)."""
    import torch
    q = 1 << 16
    host = nasg.synth_queries(4242, q, first=rank * q)
    dev = [torch.from_numpy(a).cuda() for a in host]
    out = torch.empty((q, 4), dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    res = {"workload": "config 1: 65,536 queries (fwd+sample+pdf) + one default train_iteration "
                       "(S=2^16, t=2^12, 16 Adam steps)"}
    g = nasg.Guide(nasg.TrainerConfig(seed=0), device=torch.cuda.current_device())
    for prec, name in ((nasg.NASG_MLP_BF16, "bf16"), (nasg.NASG_MLP_FP32, "fp32")):
        g.precision = prec
        for _ in range(3):
            g.query_sample(*dev, dir_pdf=out)
        torch.cuda.synchronize()
        t = sum(time_events(lambda: g.query_sample(*dev, dir_pdf=out), 20, stream)) / 20
        res[f"query_{name}"] = {"queries_per_s": q / t, "us_per_batch": 1e6 * t}
    g.close()
    samples = torch.from_numpy(nasg.synth_samples(11, q, first=rank * q)).cuda()
    pk, pk_kind = peaks()
    for name, prec in (("bf16", nasg.NASG_MLP_BF16), ("fp32", nasg.NASG_MLP_FP32)):
        g = nasg.Guide(nasg.TrainerConfig(seed=3), device=torch.cuda.current_device())
        g.train_precision = prec
        for _ in range(3):
            g.train_iteration(samples, 1.0, stats=False)
        torch.cuda.synchronize()
        l0 = g.kernel_launches
        ts = time_events(lambda: g.train_iteration(samples, 1.0, stats=False), 10, stream)
        launches = (g.kernel_launches - l0) // 10
        st = g.train_iteration(samples, 1.0)
        g.close()
        t = sum(ts) / len(ts)
        tf = q * FLOP_PER_SAMPLE / t / 1e12
        peak = pk["bf16_tflops"] if name == "bf16" else FP32_FFMA_TFLOPS
        res[f"train_iteration_{name}"] = {
            "ms_per_iteration": 1e3 * t, "samples_per_s": q / t, "steps": st.steps, "launches_per_iteration": launches,
            "roofline": {"bound": "tensor" if name == "bf16" else "fp32-ffma", "achieved": tf, "unit": "TFLOP/s",
                         "peak": peak, "frac": tf / peak,
                         "peak_kind": f"{pk_kind} bf16 burst" if name == "bf16" else FP32_PEAK_KIND,
                         "note": "16 latency-bound steps of t = 4096 rows"}}
    if rank == 0 and not args.no_cpu:
        res["cpu_baseline"] = {"query": cpu_reference_rate(0, 0, chunk=q, steps=3, warmup=1),
                               "train_iteration": cpu_reference_default_train()}
    del dev, out, samples
    torch.cuda.empty_cache()
    return res


def bench_sweep(nasg, args, ws, rank):
    """Config 2's sweep: 2^20 - 2^24 queries per batch, fp32 (FFMA) vs bf16 (tcgen05) MLP,
    device-resident inputs, CUDA events on the launching stream, max over ranks."""
    import torch
    out = {}
    nmax = 1 << 24
    host = nasg.synth_queries(77, nmax, first=rank * nmax)
    dev = [torch.from_numpy(a).cuda() for a in host]
    res = torch.empty((nmax, 4), dtype=torch.float32, device="cuda")
    g = nasg.Guide(nasg.TrainerConfig(seed=0), device=torch.cuda.current_device())
    stream = torch.cuda.current_stream()
    for prec, name in ((nasg.NASG_MLP_BF16, "bf16"), (nasg.NASG_MLP_FP32, "fp32")):
        g.precision = prec
        for lg in (20, 22, 24):
            n = 1 << lg
            reps = max(2, (1 << 24) // n) if name == "bf16" else 2
            d = [a[:n] for a in dev]
            for _ in range(2):
                g.query_sample(*d, dir_pdf=res[:n])
            torch.cuda.synchronize()
            barrier(ws)
            t = max_over_ranks(sum(time_events(lambda: g.query_sample(*d, dir_pdf=res[:n]), reps, stream)), ws)
            out[f"{name}_2^{lg}"] = n * ws * reps / t
    g.close()
    # the paper's component sweep (PAPER Table 4: C = 4 / 16 / 32; N = 8 above) at
    # 2^22 queries, both precisions, plus one config-3-shaped training step (2^18;
    # bf16, fp32 for N = 32 whose tensor-core trainer is not built)
    n = 1 << 22
    d = [a[:n] for a in dev]
    samples = torch.from_numpy(nasg.synth_samples(11, 1 << 18, first=rank * (1 << 18))).cuda()
    for nc in (4, 16, 32):
        g = nasg.Guide(nasg.TrainerConfig(seed=0, n_components=nc), device=torch.cuda.current_device())
        for prec, name in ((nasg.NASG_MLP_BF16, "bf16"), (nasg.NASG_MLP_FP32, "fp32")):
            g.precision = prec
            for _ in range(2):
                g.query_sample(*d, dir_pdf=res[:n])
            torch.cuda.synchronize()
            barrier(ws)
            reps = 4 if name == "bf16" else 2
            t = max_over_ranks(sum(time_events(lambda: g.query_sample(*d, dir_pdf=res[:n]), reps, stream)), ws)
            out[f"N{nc}_{name}_2^22"] = n * ws * reps / t
        g.close()
        tg = nasg.Guide(nasg.TrainerConfig(seed=3, n_components=nc, sample_capacity=1 << 18, batch_size=1 << 18),
                        device=torch.cuda.current_device())
        tprec = "fp32" if nc == 32 else "bf16"
        tg.train_precision = nasg.NASG_MLP_FP32 if nc == 32 else nasg.NASG_MLP_BF16
        for _ in range(3):
            tg.train_iteration(samples, 1.0, stats=False)
        torch.cuda.synchronize()
        t = max_over_ranks(sum(time_events(lambda: tg.train_iteration(samples, 1.0, stats=False), 5, stream)), ws)
        out[f"N{nc}_{tprec}_train_samples_per_s"] = (1 << 18) * ws * 5 / t
        tg.close()
    # hidden width 64 (PAPER Table 4; runs on the 128-wide kernels, exact, same cost)
    g = nasg.Guide(nasg.TrainerConfig(seed=0, hidden_units=64), device=torch.cuda.current_device())
    g.precision = nasg.NASG_MLP_BF16
    for _ in range(2):
        g.query_sample(*d, dir_pdf=res[:n])
    torch.cuda.synchronize()
    barrier(ws)
    t = max_over_ranks(sum(time_events(lambda: g.query_sample(*d, dir_pdf=res[:n]), 4, stream)), ws)
    out["HU64_bf16_2^22"] = n * ws * 4 / t
    g.close()
    del dev, res, samples
    torch.cuda.empty_cache()
    return {"unit": "queries/s (train entries: samples/s)",
            "note": "config 2 sweep; value = all ranks' queries / max-over-ranks time; N4_*, N16_*, N32_*: the "
                    "paper's lobe-count sweep (Table 4) at 2^22 queries and a 2^18-sample training step; HU64_*: "
                    "the 64-unit network (zero-embedded in the 128-wide kernels)",
            **out}


def bench_render(nasg, args, ws, rank, width, height, iters, label, pipelined=False):
    """Configs 4-5: the guided progressive render loop (nasg_render_*): per iteration one
    path per pixel of this rank's rows (wavefront tracer, NEE+MIS, guided scattering
    through the fused network query), sample collection, one train_iteration (S = 2^16,
    t = 2^12: 16 Adam steps, data-parallel over ranks through NCCL) and accumulation.
    Rows are dealt to the ranks in interleaved 8-row bands (strong scaling of the
    fixed image)."""
    import torch
    scene = nasg.SCENE_CRACK
    lo, hi = nasg.scene_bounds(scene)
    g = nasg.Guide(nasg.TrainerConfig(seed=5), device=torch.cuda.current_device(), bmin=lo, bmax=hi)
    g.precision = nasg.NASG_MLP_BF16
    g.train_precision = nasg.NASG_MLP_BF16
    if ws > 1:
        import torch.distributed as dist
        uid = [g.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        g.comm_init(uid[0], rank, ws)
    # interleaved tile rows (bands of 8 rows dealt round-robin over the ranks): every
    # rank gets the same mix of scene content, so the per-rank trace time balances
    r = nasg.Render(g, scene=scene, width=width, height=height, row_band=8, shard=rank, nshards=ws, seed=3,
                    lazy_train_stats=True, pipelined=pipelined)
    torch.cuda.synchronize()
    barrier(ws)
    l0 = g.kernel_launches + r.kernel_launches
    t0 = time.perf_counter()
    verts = guided = kept = 0
    for _ in range(iters):
        st = r.iteration()
        verts += st["vertices"]
        guided += st["guided_vertices"]
        kept += st["kept"]
    torch.cuda.synchronize()
    dt = max_over_ranks(time.perf_counter() - t0, ws)
    launches = g.kernel_launches + r.kernel_launches - l0
    img = r.image()
    finite = bool(np.isfinite(img).all())
    r_rows = r.rows
    r.close()
    g.close()
    return {"workload": label, "scene": "crack (box lit through a slit: anisotropic indirect light)",
            "iterations": iters, "seconds": dt, "ms_per_iteration": 1e3 * dt / iters,
            "paths_per_s": width * height * iters / dt, "vertices_per_s_rank0": verts / dt,
            "guided_queries_per_s_rank0": guided / dt, "train_samples_per_iteration_rank0": kept / iters,
            "gpu_launches_rank0": launches, "final_b": st["b"], "image_finite": finite, "scaling": "strong",
            "sharding": f"interleaved 8-row bands, rank {rank} of {ws} renders {r_rows} rows",
            "loop": ("pipelined: tracing of iteration i+1 overlaps training i on a second stream (snapshot one "
                     "iteration staler)" if pipelined else "serial SPEC loop: trace i -> train i -> publish -> trace i+1"),
            "cpu_baseline": None, "note": "the reference specifies this tracer (SPEC.md:378-478) but ships no code"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--queries", type=int, default=1 << 24)
    ap.add_argument("--train-samples", type=int, default=1 << 18)
    ap.add_argument("--train-steps", type=int, default=5)
    ap.add_argument("--no-train", action="store_true")
    ap.add_argument("--no-render", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-config1", action="store_true")
    ap.add_argument("--render-4k-iters", type=int, default=64)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        # the CPU reference arm: no CUDA context, no process group; rank 0 alone works
        run_reference(args, int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")))
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        import torch
        if torch.cuda.device_count() < args.gpus:  # one rank per GPU: never two ranks on one device
            sys.exit(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {torch.cuda.device_count()}")
        sys.exit(self_launch(args.gpus))
    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE', '1')}")
    ws, rank, local = dist_init()

    import torch
    import paper_2303_08064_b200 as nasg
    torch.cuda.set_device(local)
    n = args.queries
    g = nasg.Guide(nasg.TrainerConfig(seed=0), device=local)
    prec = nasg.NASG_MLP_BF16 if args.precision == "bf16" else nasg.NASG_MLP_FP32
    try:
        g.precision = prec
    except nasg.NasgError:
        prec = nasg.NASG_MLP_FP32
        g.precision = prec
    # the tensor-core path multiplies f16 operands with fp32 accumulation
    # (kind::f16 UMMA; same tensor rate as bf16), the other path is fp32 FFMA
    dtype = "f16" if prec == nasg.NASG_MLP_BF16 else "fp32"
    # this rank's pixel-tile shard of the synthetic queries (weak scaling)
    host = nasg.synth_queries(2024, n, first=rank * n, pinned=True)
    dev = [torch.from_numpy(a).cuda() for a in host]
    out = torch.empty((n, 4), dtype=torch.float32, device="cuda")
    cbuf = torch.empty(n, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        g.query_sample(*dev, dir_pdf=out, c=cbuf)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(ws)
    l0 = g.kernel_launches
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        times = time_events(step, args.steps, stream)
        torch.cuda.synchronize()
    launches = g.kernel_launches - l0
    barrier(ws)
    t_local = sum(times)
    t = max_over_ranks(t_local, ws)
    value = n * ws * args.steps / t
    per_launch = t_local / args.steps  # one fused kernel per step
    pk, pk_kind = peaks()
    achieved = n * FLOP_PER_QUERY / per_launch / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):  # dram read+write of the same kernel from the committed ncu --set full capture
        tr = json.load(open(tp)).get("bf16" if prec == nasg.NASG_MLP_BF16 else "fp32")
        traffic = tr["bytes_per_query"] * n if tr else None
    roof = {"bound": "tensor", "achieved": achieved, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
            "frac": achieved / pk["bf16_tflops"], "traffic": traffic,
            "peak_kind": f"{pk_kind} bf16 burst (f16 UMMA runs at the same dense rate)",
            "frac_sustained": achieved / pk.get("bf16_tflops_sustained", 1400.0),
            "hbm_frac": n * BYTES_PER_QUERY / per_launch / 1e9 / pk["hbm_gbs"],
            "kernel": f"query_{'tc' if dtype == 'f16' else 'fp32'}_kernel<8,sample>"}

    # ---- e2e through the host-buffer public API (pinned in, pinned out) ----
    # nasg_query_sample_host_packed: 13-float rows (52 B/query H2D), dir+pdf
    # (16 B) and c (4 B) back, H2D / kernel / D2H pipelined inside the library.
    q13 = torch.empty((n, 13), dtype=torch.float32).pin_memory().numpy()
    q13[:, 0:3], q13[:, 3:6], q13[:, 6:9], q13[:, 9:13] = host[0][:, :3], host[1][:, :3], host[2][:, :3], host[3]
    hout = torch.empty((n, 4), dtype=torch.float32).pin_memory().numpy()
    hc = torch.empty(n, dtype=torch.float32).pin_memory().numpy()
    for _ in range(2):
        g.query_sample_host_packed(q13, dir_pdf=hout, c=hc)
    barrier(ws)
    e2e_steps = max(2, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        g.query_sample_host_packed(q13, dir_pdf=hout, c=hc)
    te = max_over_ranks(time.perf_counter() - t0, ws)
    e2e = {"value": n * ws * e2e_steps / te, "unit": "queries/s", "h2d_bytes_per_step": n * 52 * ws,
           "d2h_bytes_per_step": n * 20 * ws, "api": "nasg_query_sample_host_packed (pinned host rows)"}
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        g.query_sample_host(*host, dir_pdf=hout, c=hc)
    te = max_over_ranks(time.perf_counter() - t0, ws)
    e2e["soa_float4_api"] = {"value": n * ws * e2e_steps / te, "h2d_bytes_per_step": n * 64 * ws}
    # the e2e path's own roofline: pinned host -> device copy bandwidth of this box
    # (same byte count as one step's H2D, CUDA events, best of 3)
    hbuf = torch.from_numpy(q13.reshape(-1).view(np.uint8))
    dbuf = torch.empty(hbuf.numel(), dtype=torch.uint8, device="cuda")
    best = float("inf")
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dbuf.copy_(hbuf, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    h2d_gbs = hbuf.numel() / best / 1e9
    e2e["pcie_h2d_gbs_measured"] = h2d_gbs
    e2e["h2d_roofline_queries_per_s"] = h2d_gbs * 1e9 / 52 * ws
    e2e["frac_of_h2d_roofline"] = e2e["value"] / e2e["h2d_roofline_queries_per_s"]
    del dbuf, hbuf
    g.close()
    del dev, out, cbuf
    torch.cuda.empty_cache()

    config1 = None if args.no_config1 else bench_config1(nasg, args, ws, rank)
    sweep = None if args.no_sweep else bench_sweep(nasg, args, ws, rank)
    train = None if args.no_train else {p: bench_train(nasg.Guide, nasg, args, ws, rank, p) for p in ("bf16", "fp32")}
    render = None
    if not args.no_render:
        render = {"config4": bench_render(nasg, args, ws, rank, 1024, 1024, 512,
                                          "config 4: 1024x1024, 512 spp, interleaved train/render"),
                  "config4_pipelined": bench_render(nasg, args, ws, rank, 1024, 1024, 512,
                                                    "config 4: 1024x1024, 512 spp, interleaved train/render",
                                                    pipelined=True),
                  "config5": bench_render(nasg, args, ws, rank, 3840, 2160, args.render_4k_iters,
                                          f"config 5: 3840x2160 sharded by interleaved pixel rows over {ws} GPU(s), "
                                          f"{args.render_4k_iters} spp"),
                  "config5_pipelined": bench_render(nasg, args, ws, rank, 3840, 2160, args.render_4k_iters,
                                                    f"config 5: 3840x2160 sharded by interleaved pixel rows over {ws} GPU(s), "
                                                    f"{args.render_4k_iters} spp", pipelined=True)}
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu = cpu_reference_rate(1 << 30, args.cpu_seconds)
        if train is not None:
            train["cpu_baseline"] = cpu_reference_train_rate()
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
                "config": bench_config(n, ws),
                "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "gpu_launches": launches,
                "clocks": clk.summary(), "config1": config1, "sweep": sweep, "train": train, "render": render}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
