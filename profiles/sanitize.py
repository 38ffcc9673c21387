"""Small invocations of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python profiles/sanitize.py

query_tc_kernel (all modes), query_fp32_kernel, decode_raw_kernel, the bf16
and fp32 training chains (K_fb, K_dw, reduction, Adam; the cooperative Adam
launch of the communicator path), the render kernels, the explicit-mixture
kernels and the fit.  Sizes are tiny: the tools serialise and instrument
every access."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08064_b200 as nasg  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
torch.cuda.set_device(0)
n = 300  # 3 tiles, the last one ragged


def q(n, seed=1):
    return [torch.from_numpy(a).cuda() for a in nasg.synth_queries(seed, n)]


if what in ("all", "query"):
    g = nasg.Guide(nasg.TrainerConfig(seed=1))
    x, wo, nrm, xi = q(n)
    for prec in (nasg.NASG_MLP_BF16, nasg.NASG_MLP_FP32):
        g.precision = prec
        out, c = g.query_sample(x, wo, nrm, xi, c=torch.empty(n, device="cuda"))
        g.query_pdf(x, wo, nrm, xi, 0.5, bsdf_pdf=torch.rand(n, device="cuda"))
        raw = g.query_raw(x, wo, nrm)
        g.decode_sample_raw(raw, xi)
        g.decode_pdf_raw(raw, xi, 0.5)
        g.query_shade(x, wo, nrm, xi, xi, xi, 0.5)
    torch.cuda.synchronize()
    g.close()
    print("query ok")

if what in ("all", "train"):
    s = torch.from_numpy(nasg.synth_samples(3, 700)).cuda()
    for prec in (nasg.NASG_MLP_BF16, nasg.NASG_MLP_FP32):
        for comm in (False, True):
            g = nasg.Guide(nasg.TrainerConfig(seed=2, sample_capacity=1024, batch_size=256))
            g.train_precision = prec
            if comm:
                g.comm_init(nasg.Guide.comm_unique_id(), 0, 1)
            st = g.train_iteration(s, 0.5)
            torch.cuda.synchronize()
            g.close()
    # a step with more tiles than SMs: the zero-row classification (look-back
    # compaction) and the runtime-sized K_fb / K_dw / reduction
    big = 160 * 128 + 77
    s = torch.from_numpy(nasg.synth_samples(4, big)).cuda()
    g = nasg.Guide(nasg.TrainerConfig(seed=2, sample_capacity=big, batch_size=big))
    g.train_precision = nasg.NASG_MLP_BF16
    g.train_iteration(s, 0.5)
    torch.cuda.synchronize()
    g.close()
    print("train ok")

if what in ("all", "render"):
    lo, hi = nasg.scene_bounds(nasg.SCENE_BOX)
    g = nasg.Guide(nasg.TrainerConfig(seed=7, sample_capacity=1024, batch_size=512), bmin=lo, bmax=hi)
    g.precision = g.train_precision = nasg.NASG_MLP_BF16
    r = nasg.Render(g, scene=nasg.SCENE_BOX, width=32, height=24, schedule_m=1, schedule_b=1, max_depth=6)
    for _ in range(2):
        r.iteration()
    r.image()
    r.close()
    g.close()
    print("render ok")

if what in ("all", "dist"):
    rng = np.random.default_rng(0)
    k = 4
    comp = np.zeros((64, k, 12), np.float32)
    z = rng.normal(size=(64, k, 3))
    z /= np.linalg.norm(z, axis=-1, keepdims=True)
    xa = np.cross(z, [0.3, 0.5, 0.8])
    xa /= np.linalg.norm(xa, axis=-1, keepdims=True)
    ya = np.cross(z, xa)
    comp[..., 0:3], comp[..., 3], comp[..., 4:7], comp[..., 7], comp[..., 8:11] = xa, 5.0, ya, 2.0, z
    w = np.full((64, k), 1.0 / k, np.float32)
    dirs = np.zeros((64, 4), np.float32)
    dirs[:, :3] = z[:, 0]
    C, W, D = (torch.from_numpy(a).cuda() for a in (comp, w, dirs))
    nasg.dist_mixture_pdf(nasg.DIST_NASG, C, W, D)
    nasg.dist_mixture_sample(nasg.DIST_NASG, C, W, torch.rand(64, 4, device="cuda"))
    nasg.dist_grad_logpdf(nasg.DIST_NASG, C, W, D)
    cfg = nasg.FitConfig(steps=20, batch=128, checkpoints=2)
    nasg.fit(cfg, 2, nasg.DIST_NASG, comp[0], w[0], quad_nz=16)
    torch.cuda.synchronize()
    print("dist ok")
