"""Guided vs unguided MAPE on the built-in scenes (SPEC acceptance 7 analogue):
128^2, 512 spp, M = 4, B = 64, against a 16k-spp unguided reference, for both
trainer precisions and both loop modes.

    python profiles/guiding_effect.py [--scene box|attic|crack] [--seeds 3]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2303_08064_b200 as nasg  # noqa: E402

SCENES = {"box": nasg.SCENE_BOX, "attic": nasg.SCENE_ATTIC, "crack": nasg.SCENE_CRACK}


def render(scene, guiding, spp, seed, prec=nasg.NASG_MLP_BF16, pipelined=False, size=128):
    lo, hi = nasg.scene_bounds(scene)
    g = nasg.Guide(nasg.TrainerConfig(seed=seed), bmin=lo, bmax=hi)
    g.precision = prec
    g.train_precision = prec
    r = nasg.Render(g, scene=scene, width=size, height=size, seed=seed, guiding=guiding, collect=guiding,
                    ramp=guiding, pipelined=pipelined)
    try:
        for _ in range(spp):
            r.iteration()
        return r.image()
    finally:
        r.close()
        g.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scene", default="box")
    ap.add_argument("--seeds", type=int, default=3)
    ap.add_argument("--spp", type=int, default=512)
    a = ap.parse_args()
    sc = SCENES[a.scene]
    ref = render(sc, False, 16384, 99)
    out = {}
    for seed in range(1, a.seeds + 1):
        u = nasg.mape(render(sc, False, a.spp, seed), ref)
        row = {"unguided": u}
        for name, kw in (("bf16", {}), ("fp32", {"prec": nasg.NASG_MLP_FP32}), ("bf16_pipelined", {"pipelined": True})):
            row[name] = nasg.mape(render(sc, True, a.spp, seed, **kw), ref) / u
        out[seed] = row
        print(a.scene, seed, json.dumps(row))
    print(a.scene, "median ratios", {k: float(np.median([r[k] for r in out.values()])) for k in ("bf16", "fp32", "bf16_pipelined")})


if __name__ == "__main__":
    main()
