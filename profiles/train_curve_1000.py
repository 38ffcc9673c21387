"""BASELINE config 3 as stated: online training with 2^18 radiance samples per
Adam step, a fresh seeded synthetic buffer every step (seed 1000 + k), blend
b = min(1, k/64), 1000 steps, for the bf16 (tcgen05) and the fp32 (FFMA)
trainers; the first 100 steps are compared with the reference's own curve
(tests/golden/train_curve_ref.npz, oracle/_ref run by
tests/golden/make_train_curve.py: the unmodified reference TUs).

    python profiles/train_curve_1000.py [out.json]

Writes the per-step losses, the step time (CUDA events around each
train_iteration, buffers uploaded beforehand outside the timed region) and the
tracking summary against the reference."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2303_08064_b200 as nasg  # noqa: E402

N = 1 << 18
STEPS = int(os.environ.get("CURVE_STEPS", "1000"))
ref = np.load(os.path.join(ROOT, "tests", "golden", "train_curve_ref.npz"))
lr = ref["losses"]
probe = ref["probe_q9"]
dev_probe = [torch.from_numpy(np.ascontiguousarray(np.pad(probe[:, k:k + 3], ((0, 0), (0, 1))))).cuda()
             for k in (0, 3, 6)]
out = {"workload": "config 3: 2^18 samples per Adam step, fresh seeded buffer per step, b = min(1, k/64)",
       "steps": STEPS, "reference_steps": int(len(lr)), "reference_losses": lr.tolist(), "runs": {}}
for name, prec in (("bf16", nasg.NASG_MLP_BF16), ("fp32", nasg.NASG_MLP_FP32)):
    g = nasg.Guide(nasg.TrainerConfig(seed=3, sample_capacity=N, batch_size=N))
    g.train_precision = prec
    bufs = [torch.empty((N, 16), dtype=torch.float32, device="cuda") for _ in range(2)]
    losses, ms, probes = [], [], {}
    nxt = torch.from_numpy(nasg.synth_samples(1000, N)).pin_memory()
    for k in range(STEPS):
        cur = bufs[k % 2]
        cur.copy_(nxt, non_blocking=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = g.train_iteration(cur, min(1.0, k / 64.0), stats=False)
        e1.record()
        if k + 1 < STEPS:
            nxt = torch.from_numpy(nasg.synth_samples(1000 + k + 1, N)).pin_memory()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
        st = g.train_stats_take()
        assert st.steps == 1
        losses.append(st.mean_loss)
        if k + 1 in (10, 25, 50, 100, 1000):
            probes[k + 1] = g.query_raw(*dev_probe).cpu().numpy()
    g.close()
    losses = np.array(losses)
    m = min(len(lr), STEPS)
    scale = np.abs(lr[:m]).mean()
    ma = np.convolve(losses[:m] - lr[:m], np.ones(10) / 10, mode="valid") / scale
    rel = {}
    for k in (10, 25, 50, 100):
        if k <= STEPS and f"probe_{k}" in ref:
            rel[k] = float(np.linalg.norm(probes[k] - ref[f"probe_{k}"]) / np.linalg.norm(ref[f"probe_{k}"]))
    out["runs"][name] = {
        "losses": losses.tolist(),
        "ms_per_step_median": float(np.median(ms)),
        "samples_per_s_median": N / (np.median(ms) * 1e-3),
        "vs_reference_first_100": {
            "max_abs_dev_over_mean_abs_loss": float(np.max(np.abs(losses[:m] - lr[:m])) / scale),
            "moving_avg10_max_dev": float(np.abs(ma).max()),
            "probe_rel_l2": rel,
        },
        "loss_mean_first_100": float(losses[:m].mean()),
        "loss_mean_last_100": float(losses[-100:].mean()),
        "finite": bool(np.all(np.isfinite(losses))),
    }
    print(name, json.dumps({k: v for k, v in out["runs"][name].items() if k != "losses"}), flush=True)
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "train_curve_1000.json")
with open(path, "w") as f:
    json.dump(out, f)
