"""Golden loss / network-output curve for BASELINE config 3 (online training:
2^18 radiance samples per Adam step), from the reference.

    python tests/golden/make_train_curve.py [steps] [--reverse]

Step k trains on a fresh synthetic buffer nasg_synth_samples(seed=1000+k,
2^18) (host-side generator of the product library, SURVEY §8d target field)
with TrainerConfig{S = t = 2^18, nu = 1, seed = 3} -> exactly one Adam step
per train_iteration, blend b = min(1, k/64).  Records the mean loss of every
step and the raw network outputs on a fixed 1024-query probe set after steps
10, 25, 50 and 100.

Default: the UNMODIFIED reference (oracle/_ref) -> train_curve_ref.npz.
--reverse: the C restatement with the dW reduction summed in reverse row
order -> train_curve_rev.npz, the reassociation yardstick the GPU tolerance
is derived from (tests/test_gpu_train_curve.py).
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import paper_2303_08064_b200 as nasg  # noqa: E402  (host-side synth generator only)
from oracle.oracle import Oracle  # noqa: E402

N_SAMPLES = 1 << 18
PROBE_AT = (10, 25, 50, 100)


def probe_queries():
    x, wo, nrm, _ = nasg.synth_queries(4242, 1024)
    return np.ascontiguousarray(np.concatenate([x[:, :3], wo[:, :3], nrm[:, :3]], 1))


def blend(k):
    return min(1.0, k / 64.0)


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else 100
    reverse = "--reverse" in sys.argv
    o = Oracle("orc" if reverse else "ref")
    if reverse:
        o.set_reverse_sum(True)
    t = o.trainer(capacity=N_SAMPLES, batch=N_SAMPLES, seed=3)
    q9 = probe_queries()
    enc, _ = o.encode(q9, (-1, -1, -1), (1, 1, 1))
    losses, probes = [], {}
    t0 = time.time()
    for k in range(steps):
        s = nasg.synth_samples(1000 + k, N_SAMPLES)
        st = t.train(s, blend(k))
        assert st["steps"] == 1
        losses.append(st["mean_loss"])
        if k + 1 in PROBE_AT:
            probes[f"probe_{k + 1}"] = o.forward(t.weights(), enc)
        print(f"step {k + 1}/{steps} loss {st['mean_loss']:.6f} ({time.time() - t0:.0f}s)", flush=True)
    name = "train_curve_rev.npz" if reverse else "train_curve_ref.npz"
    np.savez_compressed(os.path.join(HERE, name), losses=np.array(losses), probe_q9=q9, **probes)


if __name__ == "__main__":
    main()
