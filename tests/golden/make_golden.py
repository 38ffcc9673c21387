"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libnasg_ref.so, i.e. a host
where /root/reference exists):

    python tests/golden/make_golden.py

Fixtures (seeded, small):
  query_ref.npz : init_network(seed) weights, 512 queries -> infer_guide +
                  mixture_sample outputs; 2048 benign + 2048 stress raw
                  vectors -> decode + mixture_sample (double).
  kl_ref.npz    : 2048 stress raws + samples -> kl_loss_gradient, ok, loss.
  train_ref.npz : Trainer(S=2048, t=256, seed=5) over 3 iterations with
                  b = 0, 0.5, 1: mean losses + final weights.
The config-3 training curve (train_curve_ref.npz) is produced by
make_train_curve.py, which also needs the product library's synthetic
sample generator.
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
    rng = np.random.default_rng(20260318)

    w = ref.init_network(1234)
    q9, xi = H.queries(rng, 512, outside=0.1), H.xis(rng, 512)
    out, c = ref.query_sample(w, q9, xi)
    fx = dict(w=w, q9=q9, xi=xi, out=out, c=c, seed=np.int64(1234))
    fx["raw"] = ref.forward(w, ref.encode(q9, H.BMIN, H.BMAX)[0])
    for stress in (False, True):
        tag = "stress" if stress else "benign"
        raw, x = H.raw_outputs(rng, 2048, stress=stress), H.xis(rng, 2048)
        ds, cc = ref.decode_sample(raw, x)
        fx[f"raw_{tag}"], fx[f"xi_{tag}"], fx[f"ds_{tag}"], fx[f"c_{tag}"] = raw, x, ds, cc
    np.savez_compressed(os.path.join(HERE, "query_ref.npz"), **fx)

    raw, s = H.raw_outputs(rng, 2048, stress=True), H.samples(rng, 2048)
    g, ok, loss = ref.kl_grad(raw, s, 0.75)
    np.savez_compressed(os.path.join(HERE, "kl_ref.npz"), raw=raw, samples=s, b=np.float64(0.75),
                        grad=g, ok=ok, loss=loss)

    s = H.samples(rng, 2048)
    t = ref.trainer(capacity=2048, batch=256, seed=5)
    bs = np.array([0.0, 0.5, 1.0])
    losses = np.array([t.train(s, b)["mean_loss"] for b in bs])
    np.savez_compressed(os.path.join(HERE, "train_ref.npz"), samples=s, capacity=np.int64(2048),
                        batch=np.int64(256), seed=np.int64(5), b=bs, losses=losses,
                        w_final=t.weights())
    print("wrote golden fixtures; train losses", losses)


if __name__ == "__main__":
    main()
