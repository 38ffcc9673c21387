# guided / unguided MAPE (SPEC acceptance 7) on candidate indirect-illumination box scenes
import sys, time
sys.path.insert(0, '/root/repo')
import paper_2303_08064_b200 as nasg
def render(scene, guiding, spp, seed, size=128):
    lo, hi = nasg.scene_bounds(scene)
    g = nasg.Guide(nasg.TrainerConfig(seed=seed), bmin=lo, bmax=hi)
    g.precision = nasg.NASG_MLP_BF16; g.train_precision = nasg.NASG_MLP_BF16
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
    for seed in (1, 2):
        gd = nasg.mape(render(sc, True, 512, seed), ref)
        u2 = u if seed == 1 else nasg.mape(render(sc, False, 512, seed), ref)
        print(f"scene {sc} seed {seed} unguided {u2:.4f} guided {gd:.4f} ratio {gd / u2:.4f} ({time.time() - t:.0f} s)", flush=True)
