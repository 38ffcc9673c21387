"""A/B timing of the bf16 training step: python profiles/ab_train.py [label]
(the library is chosen by NASG_LIB).  Config 3 (S = t = 2^18, one Adam step per
train_iteration) and the render-sized step (t = 4096, AB_T env), CUDA events,
median of 5 x 20 steps; prints one JSON line per size."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08064_b200 as nasg  # noqa: E402

label = sys.argv[1] if len(sys.argv) > 1 else ""
for n in [int(v) for v in os.environ.get("AB_T", str(1 << 18)).split(",")]:
    g = nasg.Guide(nasg.TrainerConfig(seed=3, sample_capacity=n, batch_size=n))
    g.train_precision = nasg.NASG_MLP_BF16
    if "AB_SKIP" in os.environ:
        g.zero_row_skip = os.environ["AB_SKIP"] == "1"
    s = torch.from_numpy(nasg.synth_samples(11, n)).cuda()
    for _ in range(3):
        g.train_iteration(s, 1.0, stats=False)
    torch.cuda.synchronize()
    ms = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            g.train_iteration(s, 1.0, stats=False)
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1) / 20)
    m = statistics.median(ms)
    print(json.dumps({"label": label, "lib": nasg.LIB_PATH, "t": n, "skip": os.environ.get("AB_SKIP"), "ms_per_step": m, "samples_per_s": n / (m * 1e-3),
                      "ms": ms}), flush=True)
    g.close()
