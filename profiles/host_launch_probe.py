"""Is the small-batch training chain bound by the host's launch rate?  For
t = 4096 (S = 2^16: 16 Adam steps per train_iteration, and S = t: one step),
the wall time of the enqueueing call (no synchronisation inside, stats=False)
against the CUDA-event time of the same calls.  One JSON line per config."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08064_b200 as nasg  # noqa: E402

for S, t in ((1 << 16, 1 << 12), (1 << 12, 1 << 12)):
    g = nasg.Guide(nasg.TrainerConfig(seed=3, sample_capacity=S, batch_size=t))
    g.train_precision = nasg.NASG_MLP_BF16
    s = torch.from_numpy(nasg.synth_samples(11, S)).cuda()
    for _ in range(5):
        g.train_iteration(s, 1.0, stats=False)
    torch.cuda.synchronize()
    reps = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h0 = time.perf_counter()
    for _ in range(reps):
        g.train_iteration(s, 1.0, stats=False)
    h1 = time.perf_counter()
    e1.record()
    e1.synchronize()
    h2 = time.perf_counter()
    steps = S // t
    print(json.dumps({"S": S, "t": t, "steps_per_call": steps,
                      "host_enqueue_us_per_step": (h1 - h0) / reps / steps * 1e6,
                      "gpu_event_us_per_step": e0.elapsed_time(e1) / reps / steps * 1e3,
                      "wall_us_per_step": (h2 - h0) / reps / steps * 1e6,
                      "kernel_launches_total": g.kernel_launches}), flush=True)
    g.close()
