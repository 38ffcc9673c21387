"""Probe: render-loop-sized training (S = 2^16, t = 2^12, 16 Adam steps per
train_iteration, bf16) per-iteration device time vs the minimum 128-row blocks
per dW split (NASG_DW_MIN_BPS, read once per process).  Prints one JSON line."""
import json, os, sys, torch
sys.path.insert(0, '.')
import paper_2303_08064_b200 as nasg
g = nasg.Guide(nasg.TrainerConfig(seed=3))
g.train_precision = nasg.NASG_MLP_BF16
s = torch.from_numpy(nasg.synth_samples(11, 1 << 16)).cuda()
for _ in range(5): g.train_iteration(s, 1.0, stats=False)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): g.train_iteration(s, 1.0, stats=False)
    e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1) / 10)
print(json.dumps({"min_bps": int(os.environ.get("NASG_DW_MIN_BPS", "1")), "ms_per_iteration": sorted(ts)}))
# Result (profiles/r1_dw_bps_probe.jsonl, with a temporary NASG_DW_MIN_BPS knob in
# train_tc_step, since removed): 1 block per split 0.495 ms, 2: 0.507, 4: 0.499,
# 8: 0.549 ms per iteration — fewer, longer splits do not pay at t = 4096; the
# knob was reverted and the one-block-per-split plan kept.
