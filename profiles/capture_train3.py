"""Workload for ncu launch lists of the config-3 training step (tensor-core
trainer, S = t = 2^18 samples, one Adam step per train_iteration), 4 steps."""
import sys, torch
sys.path.insert(0, '.')
import paper_2303_08064_b200 as nasg
m = 1 << 18
t = nasg.Guide(nasg.TrainerConfig(seed=3, sample_capacity=m, batch_size=m))
t.train_precision = nasg.NASG_MLP_BF16
s = torch.from_numpy(nasg.synth_samples(11, m)).cuda()
for _ in range(4): t.train_iteration(s, 1.0, stats=False)
torch.cuda.synchronize()
print("ok")
