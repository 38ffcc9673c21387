# guided / unguided MAPE (SPEC acceptance 7) on the render scenes
# usage: indirect_probe.py SCENES [REF_SPP] [fp32|bf16] [SEEDS]  (query + trainer precision; default tensor core)
import sys, time
sys.path.insert(0, '/root/repo')
import paper_2303_08064_b200 as nasg
PREC = nasg.NASG_MLP_FP32 if len(sys.argv) > 3 and sys.argv[3] == 'fp32' else nasg.NASG_MLP_BF16
def render(scene, guiding, spp, seed, size=128):
    lo, hi = nasg.scene_bounds(scene)
    g = nasg.Guide(nasg.TrainerConfig(seed=seed), bmin=lo, bmax=hi)
    g.precision = PREC; g.train_precision = PREC
    r = nasg.Render(g, scene=scene, width=size, height=size, seed=seed, guiding=guiding, collect=guiding, ramp=guiding)
    try:
        for _ in range(spp): r.iteration()
        return r.image()
    finally:
        r.close(); g.close()
for sc in [int(x) for x in sys.argv[1].split(',')]:
    t = time.time()
    ref = render(sc, False, int(sys.argv[2]) if len(sys.argv) > 2 else 16384, 99)
    u = nasg.mape(render(sc, False, 512, 1), ref)
    for seed in ([int(x) for x in sys.argv[4].split(',')] if len(sys.argv) > 4 else (1, 2)):
        gd = nasg.mape(render(sc, True, 512, seed), ref)
        u2 = u if seed == 1 else nasg.mape(render(sc, False, 512, seed), ref)
        print(f"scene {sc} seed {seed} unguided {u2:.4f} guided {gd:.4f} ratio {gd / u2:.4f} ({time.time() - t:.0f} s)", flush=True)
