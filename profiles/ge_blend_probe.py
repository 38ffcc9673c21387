import json, os, sys
import numpy as np
sys.path.insert(0, '/root/repo')
import paper_2303_08064_b200 as nasg
SC = {"box": nasg.SCENE_BOX, "attic": nasg.SCENE_ATTIC, "crack": nasg.SCENE_CRACK}
def render(scene, guiding, spp, seed, blend=0.2, size=128, nu=1, lr=0.002):
    lo, hi = nasg.scene_bounds(scene)
    g = nasg.Guide(nasg.TrainerConfig(seed=seed, loss_blend=blend, step_factor=nu, learning_rate=lr), bmin=lo, bmax=hi)
    g.precision = nasg.NASG_MLP_BF16; g.train_precision = nasg.NASG_MLP_BF16
    r = nasg.Render(g, scene=scene, width=size, height=size, seed=seed, guiding=guiding, collect=guiding, ramp=guiding)
    try:
        for _ in range(spp): st = r.iteration()
        return r.image(), st
    finally:
        r.close(); g.close()
for name in sys.argv[1].split(','):
    sc = SC[name]
    ref, _ = render(sc, False, 16384, 99)
    u = nasg.mape(render(sc, False, 512, 1)[0], ref)
    for blend in (0.2, 0.0, 0.5, 1.0):
        img, st = render(sc, True, 512, 1, blend=blend)
        print(name, "blend", blend, "ratio", round(nasg.mape(img, ref) / u, 4), {k: v for k, v in st.items() if k != 'train'}, flush=True)
