"""Probe: where the end-to-end training step (config 3, 2^18 samples uploaded from pinned
host memory each step, TrainStats read back) loses time against max(upload, train).

Prints one JSON line: per-step ms of (a) the 16.7 MB upload alone, back to back,
(b) train_iteration with stats on a resident buffer, (c) the bench's double-buffered
loop, (d) the same loop with three buffers (two uploads in flight)."""
import json
import time

import torch

import paper_2303_08064_b200 as nasg

N, STEPS = 1 << 18, 40


def main():
    g = nasg.Guide(nasg.TrainerConfig(seed=3, sample_capacity=N, batch_size=N))
    g.train_precision = nasg.NASG_MLP_BF16
    hs = torch.from_numpy(nasg.synth_samples(11, N)).pin_memory()
    s = hs.cuda()
    for _ in range(3):
        g.train_iteration(s, 1.0)
    torch.cuda.synchronize()
    out = {}

    cs, cur = torch.cuda.Stream(), torch.cuda.current_stream()
    t0 = time.perf_counter()
    with torch.cuda.stream(cs):
        for _ in range(STEPS):
            s.copy_(hs, non_blocking=True)
    torch.cuda.synchronize()
    out["upload_ms"] = 1e3 * (time.perf_counter() - t0) / STEPS

    t0 = time.perf_counter()
    for _ in range(STEPS):
        g.train_iteration(s, 1.0, stats=True)
    torch.cuda.synchronize()
    out["train_stats_ms"] = 1e3 * (time.perf_counter() - t0) / STEPS

    t0 = time.perf_counter()
    for _ in range(STEPS):
        g.train_iteration(s, 1.0, stats=False)
    torch.cuda.synchronize()
    out["train_nostats_ms"] = 1e3 * (time.perf_counter() - t0) / STEPS

    for nb in (2, 3, 4):
        bufs = [torch.empty_like(s) for _ in range(nb)]
        copied = [torch.cuda.Event() for _ in range(nb)]
        trained = [torch.cuda.Event() for _ in range(nb)]
        vals = []
        for _trial in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            with torch.cuda.stream(cs):
                for j in range(min(nb - 1, STEPS)):
                    bufs[j].copy_(hs, non_blocking=True)
                    copied[j].record(cs)
            for k in range(STEPS):
                b = k % nb
                nxt = k + nb - 1
                if nxt < STEPS:
                    with torch.cuda.stream(cs):
                        if k >= 1:
                            cs.wait_event(trained[nxt % nb])
                        bufs[nxt % nb].copy_(hs, non_blocking=True)
                        copied[nxt % nb].record(cs)
                cur.wait_event(copied[b])
                g.train_iteration(bufs[b], 1.0, stats=True)
                trained[b].record(cur)
            torch.cuda.synchronize()
            vals.append(1e3 * (time.perf_counter() - t0) / STEPS)
        out[f"e2e_{nb}buf_ms"] = sorted(vals)
    g.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
