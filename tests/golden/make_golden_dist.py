"""Golden fixtures for the explicit-mixture density layer and the vMF / SG
baseline (sphdist.hpp:33-121, sphdist.cpp:152-340), from the UNMODIFIED
reference (oracle/_ref; run where /root/reference exists):

    python tests/golden/make_golden_dist.py

dist_ref.npz: for kind in (nasg, vmf) and (benign, stress) records, 256
queries x k lobes -> mixture pdf at random directions, mixture_sample
(dir, pdf), grad log pdf per lobe; plus the fit's vMF-model gradient
(vmf_grad_logpdf chain) for 1024 samples of a 14-lobe model.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import nasg_testutil as H  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402


def main():
    ref = Oracle("ref")
    rng = np.random.default_rng(20261018)
    fx = {}
    for kind, name in ((0, "nasg"), (1, "vmf")):
        for stress in (False, True):
            tag = f"{name}_{'stress' if stress else 'benign'}"
            k = 8 if kind == 0 else 14
            gen = H.nasg_records if kind == 0 else H.vmf_records
            comp, w = gen(rng, 256, k, stress=stress)
            d = np.zeros((256, 4), np.float32)
            d[:, :3] = H.dirs(rng, 256)
            xi = H.xis(rng, 256)
            fx[f"{tag}_comp"], fx[f"{tag}_w"], fx[f"{tag}_dir"], fx[f"{tag}_xi"] = comp, w, d, xi
            fx[f"{tag}_pdf"] = ref.dist_pdf(kind, comp, w, d)
            fx[f"{tag}_sample"] = ref.dist_sample(kind, comp, w, xi)
            fx[f"{tag}_grad"] = ref.dist_grad(kind, comp, w, d)
    raw = rng.normal(0.0, 1.0, 70).astype(np.float32)
    s = np.zeros((1024, 4), np.float32)
    s[:, :3] = H.dirs(rng, 1024)
    s[:, 3] = rng.exponential(1.0, 1024)
    s[::17, 3] = 0.0
    g, ok = ref.vmf_fit_grad(raw, s)
    fx.update(fit_raw=raw, fit_samples=s, fit_grad=g, fit_ok=ok)
    np.savez_compressed(os.path.join(HERE, "dist_ref.npz"), **fx)
    print("wrote dist_ref.npz")


if __name__ == "__main__":
    main()
