"""A/B timing of the tensor-core query kernel for a lobe count: AB_N (default 8),
2^22 queries per launch, median of 5 x 10 launches; one JSON line (NASG_LIB picks the build)."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08064_b200 as nasg  # noqa: E402

n = 1 << 22
nc = int(os.environ.get("AB_N", "8"))
g = nasg.Guide(nasg.TrainerConfig(seed=0, n_components=nc))
g.precision = nasg.NASG_MLP_BF16
x, wo, nrm, xi = [torch.from_numpy(a).cuda() for a in nasg.synth_queries(2024, n)]
out = torch.empty((n, 4), device="cuda")
for _ in range(3):
    g.query_sample(x, wo, nrm, xi, dir_pdf=out)
torch.cuda.synchronize()
rates = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        g.query_sample(x, wo, nrm, xi, dir_pdf=out)
    e1.record()
    e1.synchronize()
    rates.append(10 * n / (e0.elapsed_time(e1) * 1e-3))
print(json.dumps({"label": sys.argv[1] if len(sys.argv) > 1 else "", "N": nc, "qps_median": statistics.median(rates)}))
