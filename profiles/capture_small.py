"""Workload for the ncu capture of a render-loop-sized training step: bf16,
S = 2^16 samples, t = 2^12 per Adam step (16 steps per train_iteration)."""
import sys, torch
sys.path.insert(0, '.')
import paper_2303_08064_b200 as nasg
g = nasg.Guide(nasg.TrainerConfig(seed=3))
g.train_precision = nasg.NASG_MLP_BF16
import os
if "AB_SKIP" in os.environ:
    g.zero_row_skip = os.environ["AB_SKIP"] == "1"
s = torch.from_numpy(nasg.synth_samples(11, 1 << 16)).cuda()
for _ in range(2): g.train_iteration(s, 1.0, stats=False)
torch.cuda.synchronize()
print("ok")
