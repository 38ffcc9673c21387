"""Large training batches (beyond config 3's 2^18): the tensor-core step at 2^20 and
2^22 samples per Adam step, skip on vs off (same gradient up to summation order,
same counts), and the step rate; plus a 2^26-query launch.  One JSON line per size."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08064_b200 as nasg  # noqa: E402

for lg in (20, 22):
    n = 1 << lg
    s = torch.from_numpy(nasg.synth_samples(5, n)).cuda()
    res = {"samples_per_step": n}
    grads = {}
    for skip in (True, False):
        g = nasg.Guide(nasg.TrainerConfig(seed=3, sample_capacity=n, batch_size=n))
        g.train_precision = nasg.NASG_MLP_BF16
        g.zero_row_skip = skip
        g.train_step(s, None, n, n, 1.0)
        grads[skip] = g.last_grad().astype(np.float64)
        st = g.train_stats_take()
        res[f"stats_skip{int(skip)}"] = [st.steps, st.mean_loss, st.dropped_samples]
        for _ in range(2):
            g.train_iteration(s, 1.0, stats=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g.train_iteration(s, 1.0, stats=False)
        e1.record()
        e1.synchronize()
        res[f"ms_per_step_skip{int(skip)}"] = e0.elapsed_time(e1) / 5
        res[f"samples_per_s_skip{int(skip)}"] = n / (e0.elapsed_time(e1) / 5 * 1e-3)
        g.close()
    res["grad_rel_l2_skip_vs_full"] = float(np.linalg.norm(grads[True] - grads[False]) / np.linalg.norm(grads[False]))
    print(json.dumps(res), flush=True)
    del s
    torch.cuda.empty_cache()

n = 1 << 26
g = nasg.Guide(nasg.TrainerConfig(seed=0))
g.precision = nasg.NASG_MLP_BF16
dev = [torch.from_numpy(a).cuda() for a in nasg.synth_queries(9, n)]
out = torch.empty((n, 4), device="cuda")
g.query_sample(*dev, dir_pdf=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    g.query_sample(*dev, dir_pdf=out)
e1.record()
e1.synchronize()
o = out.cpu().numpy()
print(json.dumps({"queries_per_launch": n, "queries_per_s": 3 * n / (e0.elapsed_time(e1) * 1e-3),
                  "all_finite": bool(np.isfinite(o).all()), "pdf_positive": bool((o[:, 3] > 0).all())}))
