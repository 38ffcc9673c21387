"""Workload for the ncu captures of the fp32 (accuracy) path: two fp32 query
passes over 2^22 synthetic queries, then two fp32 training steps at 2^16 samples."""
import sys, torch
sys.path.insert(0, '.')
import paper_2303_08064_b200 as nasg
n = 1 << 22
g = nasg.Guide(nasg.TrainerConfig(seed=0))
g.precision = nasg.NASG_MLP_FP32
dev = [torch.from_numpy(a).cuda() for a in nasg.synth_queries(2024, n)]
out = torch.empty((n, 4), dtype=torch.float32, device="cuda")
c = torch.empty(n, dtype=torch.float32, device="cuda")
for _ in range(2): g.query_sample(*dev, dir_pdf=out, c=c)
g.close()
m = 1 << 16
t = nasg.Guide(nasg.TrainerConfig(seed=3, sample_capacity=m, batch_size=m))
t.train_precision = nasg.NASG_MLP_FP32
s = torch.from_numpy(nasg.synth_samples(11, m)).cuda()
for _ in range(2): t.train_iteration(s, 1.0, stats=False)
torch.cuda.synchronize()
print("ok")
