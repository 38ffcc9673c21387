"""Workload for an ncu launch list of config-4 render iterations (1024^2, crack
scene, bf16 query and training paths): 6 warm-up iterations, then 2 more.
    ncu --metrics gpu__time_duration.sum --clock-control none -s <skip> --csv ... python profiles/capture_render.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08064_b200 as nasg  # noqa: E402

lo, hi = nasg.scene_bounds(nasg.SCENE_CRACK)
g = nasg.Guide(nasg.TrainerConfig(seed=5), bmin=lo, bmax=hi)
g.precision = nasg.NASG_MLP_BF16
g.train_precision = nasg.NASG_MLP_BF16
r = nasg.Render(g, scene=nasg.SCENE_CRACK, width=1024, height=1024, seed=3)
for _ in range(8):
    r.iteration()
torch.cuda.synchronize()
r.close()
g.close()
print("ok")
