"""Where a config-4 render iteration's time goes (1 x B200): wall time of the
full loop (trace + guided queries + collection + train_iteration) vs the loop
without training (collect = 0) vs train_iteration alone on a 2^16-sample
buffer (wall and CUDA-event time), bf16 query and training paths.

    python profiles/render_phases.py [--iters 512] [--size 1024]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2303_08064_b200 as nasg  # noqa: E402


def loop(collect, iters, size, lazy=False, pipelined=False):
    lo, hi = nasg.scene_bounds(nasg.SCENE_CRACK)
    g = nasg.Guide(nasg.TrainerConfig(seed=5), bmin=lo, bmax=hi)
    g.precision = nasg.NASG_MLP_BF16
    g.train_precision = nasg.NASG_MLP_BF16
    r = nasg.Render(g, scene=nasg.SCENE_CRACK, width=size, height=size, seed=3, collect=collect,
                    lazy_train_stats=lazy, pipelined=pipelined)
    torch.cuda.synchronize()
    per = []
    t0 = time.perf_counter()
    for _ in range(iters):
        t = time.perf_counter()
        r.iteration()
        per.append(time.perf_counter() - t)
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
    r.close()
    g.close()
    per = np.array(per) * 1e3
    return {"ms_per_iteration": 1e3 * tot / iters, "ms_first_64": float(per[:64].mean()),
            "ms_last_128": float(per[-128:].mean())}


def train_alone(reps=20):
    g = nasg.Guide(nasg.TrainerConfig(seed=5))
    g.train_precision = nasg.NASG_MLP_BF16
    s = torch.from_numpy(nasg.synth_samples(2, 1 << 16)).cuda()
    for _ in range(3):
        g.train_iteration(s, 1.0)
    torch.cuda.synchronize()
    out = {}
    for stats in (True, False):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        ev0.record()
        for _ in range(reps):
            g.train_iteration(s, 1.0, stats=stats)
        ev1.record()
        torch.cuda.synchronize()
        out[f"stats={stats}"] = {"wall_ms": 1e3 * (time.perf_counter() - t0) / reps,
                                 "event_ms": ev0.elapsed_time(ev1) / reps}
    g.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=512)
    ap.add_argument("--size", type=int, default=1024)
    ap.add_argument("--only-full", action="store_true", help="just the full loop (for an ncu launch list)")
    a = ap.parse_args()
    if a.only_full:
        print(json.dumps(loop(True, a.iters, a.size, lazy=True)))
        return
    res = {"full": loop(True, a.iters, a.size), "full_lazy_stats": loop(True, a.iters, a.size, lazy=True),
           "full_pipelined": loop(True, a.iters, a.size, pipelined=True),
           "no_train": loop(False, a.iters, a.size), "train_alone": train_alone()}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
