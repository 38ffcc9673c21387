"""NASG vs vMF / SG expressiveness (PAPER Fig. 5, SPEC.md run_fit :500-508 and
acceptance 6 :547) on the GPU: fit 8-lobe NASG (64 scalars + c) and 14-lobe
vMF (70 scalars) guide distributions to analytic targets with the guider's KL
gradient and Adam, then report quadrature KL(target || model).

    python examples/fit_compare.py [--seeds 5] [--steps 2000] [--json out.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2303_08064_b200 as nasg  # noqa: E402


def _frame(z, hint):
    z = np.asarray(z, np.float64)
    z /= np.linalg.norm(z)
    x = np.cross(hint, z)
    x /= np.linalg.norm(x)
    return x, np.cross(z, x), z


def nasg_target(lobes):
    """lobes: [(z, hint, lambda, a, weight)] -> (k,12) records, (k,) weights."""
    rec, w = [], []
    for z, hint, lam, a, wt in lobes:
        x, y, zz = _frame(z, np.asarray(hint, np.float64))
        rec.append([*x, lam, *y, a, *zz, 0.0])
        w.append(wt)
    w = np.asarray(w, np.float64)
    return np.asarray(rec, np.float32), (w / w.sum()).astype(np.float32)


def vmf_target(lobes):
    rec = [[*(np.asarray(mu, np.float64) / np.linalg.norm(mu)), lam] for mu, lam, _ in lobes]
    w = np.asarray([wt for _, _, wt in lobes], np.float64)
    return np.asarray(rec, np.float32), (w / w.sum()).astype(np.float32)


def targets():
    t = {}
    # a thin curved band: three strongly anisotropic NASG lobes along an arc
    t["band"] = (nasg.DIST_NASG, *nasg_target([
        ((1.0, 0.0, 0.6), (0.0, 0.0, 1.0), 60.0, 200.0, 1.0),
        ((0.3, 0.9, 0.5), (0.0, 0.0, 1.0), 60.0, 200.0, 1.0),
        ((-0.7, 0.6, 0.4), (0.0, 0.0, 1.0), 60.0, 200.0, 1.0)]))
    # a curve of sharp isotropic lobes (a sine band on the sphere): in neither family
    phis = np.linspace(0.0, 1.5 * np.pi, 24)
    t["curve"] = (nasg.DIST_VMF, *vmf_target([((np.cos(p), np.sin(p), 0.35 * np.sin(3 * p)), 150.0, 1.0)
                                              for p in phis]))
    # isotropic: a single vMF (both families contain it)
    t["isotropic"] = (nasg.DIST_VMF, *vmf_target([((0.2, -0.4, 0.9), 25.0, 1.0)]))
    return t


MODELS = {"nasg8": (nasg.DIST_NASG, 8), "vmf14": (nasg.DIST_VMF, 14)}


def run(seeds=5, steps=2000, batch=1024, lr=0.02, checkpoints=10, quad_nz=512):
    out = {}
    for tname, (tk, tc, tw) in targets().items():
        row = {}
        for mname, (model, k) in MODELS.items():
            cfg = nasg.FitConfig(model=model, n_components=k, batch=batch, steps=steps, checkpoints=checkpoints,
                                 learning_rate=lr, seed=17)
            t0 = time.perf_counter()
            raw, kl = nasg.fit(cfg, seeds, tk, tc, tw, quad_nz=quad_nz)
            row[mname] = {"kl_final": kl[:, -1].tolist(), "kl_curve_mean": kl.mean(0).tolist(),
                          "seconds": time.perf_counter() - t0}
        out[tname] = row
    return out


def sweep(seeds=3, steps=2000, batch=1024, lr=0.02, quad_nz=512):
    """Lobe-count sweep (PAPER Table 4's N axis, position-free): NASG N in
    {2, 4, 8, 16} and vMF with the same number of scalars (8N / 5 lobes)."""
    out = {}
    for tname, (tk, tc, tw) in targets().items():
        row = {}
        for n in (2, 4, 8, 16):
            for model, k in ((nasg.DIST_NASG, n), (nasg.DIST_VMF, max(1, round(8 * n / 5)))):
                cfg = nasg.FitConfig(model=model, n_components=k, batch=batch, steps=steps, checkpoints=1,
                                     learning_rate=lr, seed=23)
                _, kl = nasg.fit(cfg, seeds, tk, tc, tw, quad_nz=quad_nz)
                row[f"{'nasg' if model == nasg.DIST_NASG else 'vmf'}{k}"] = float(np.median(kl[:, -1]))
        out[tname] = row
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=5)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--lr", type=float, default=0.02)
    ap.add_argument("--json", default=None)
    ap.add_argument("--sweep", action="store_true", help="lobe-count sweep instead of the 8-vs-14 comparison")
    a = ap.parse_args()
    if a.sweep:
        res = sweep(min(a.seeds, 3), a.steps, a.batch, a.lr)
        for t, row in res.items():
            print(f"{t:10s} " + "  ".join(f"{m}={v:.4f}" for m, v in row.items()))
        if a.json:
            json.dump(res, open(a.json, "w"), indent=1)
        return
    res = run(a.seeds, a.steps, a.batch, a.lr)
    for t, row in res.items():
        for m, r in row.items():
            print(f"{t:10s} {m:6s} KL final per seed {np.round(r['kl_final'], 4)}  ({r['seconds']:.2f} s)")
    if a.json:
        json.dump(res, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
