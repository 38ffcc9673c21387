"""A/B timing of the bf16 query kernel: python profiles/ab_query.py [label]
(the library is chosen by NASG_LIB).  2^24 queries per launch, CUDA events,
median of 5 x 10 launches; prints one JSON line."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08064_b200 as nasg  # noqa: E402

n = 1 << 24
mode = os.environ.get("AB_MODE", "sample")
g = nasg.Guide(nasg.TrainerConfig(seed=0))
g.precision = nasg.NASG_MLP_BF16
x, wo, nrm, xi = [torch.from_numpy(a).cuda() for a in nasg.synth_queries(2024, n)]
out = torch.empty((n, 4), device="cuda")
c = torch.empty(n, device="cuda")
f = (lambda: g.query_sample(x, wo, nrm, xi, dir_pdf=out, c=c)) if mode == "sample" else \
    (lambda: g.query_pdf(x, wo, nrm, xi, 0.5))
for _ in range(3):
    f()
torch.cuda.synchronize()
rates = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    e1.synchronize()
    rates.append(10 * n / (e0.elapsed_time(e1) * 1e-3))
print(json.dumps({"label": sys.argv[1] if len(sys.argv) > 1 else "", "lib": nasg.LIB_PATH, "mode": mode,
                  "qps_median": statistics.median(rates), "qps": rates}))
