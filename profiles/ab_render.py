"""A/B timing of the config-4 render loop (1024^2, crack scene, bf16 paths):
ms per iteration over 96 iterations after 16 warm-up ones (NASG_LIB picks the build)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08064_b200 as nasg  # noqa: E402

label = sys.argv[1] if len(sys.argv) > 1 else ""
lo, hi = nasg.scene_bounds(nasg.SCENE_CRACK)
g = nasg.Guide(nasg.TrainerConfig(seed=5), bmin=lo, bmax=hi)
g.precision = nasg.NASG_MLP_BF16
g.train_precision = nasg.NASG_MLP_BF16
r = nasg.Render(g, scene=nasg.SCENE_CRACK, width=1024, height=1024, seed=3,
                collect=int(os.environ.get("AB_COLLECT", "1")))
for _ in range(16):
    r.iteration()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(96):
    r.iteration()
torch.cuda.synchronize()
ms = (time.perf_counter() - t0) / 96 * 1e3
print(json.dumps({"label": label, "collect": os.environ.get("AB_COLLECT", "1"), "ms_per_iteration": ms}), flush=True)
r.close()
g.close()
