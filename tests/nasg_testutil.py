"""Seeded synthetic inputs shared by the tests (numpy; independent of the product)."""
import numpy as np

BMIN = np.array([-1.0, -1.0, -1.0], np.float32)
BMAX = np.array([1.0, 1.0, 1.0], np.float32)


def dirs(rng, n):
    z = 1.0 - 2.0 * rng.random(n)
    phi = 2.0 * np.pi * rng.random(n)
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    return np.stack([r * np.cos(phi), r * np.sin(phi), z], 1).astype(np.float32)


def queries(rng, n, outside=0.0):
    """(n,9) float32: position, omega_o, normal.  `outside` > 0 widens positions past the bounds."""
    pos = rng.uniform(-1.0 - outside, 1.0 + outside, (n, 3)).astype(np.float32)
    return np.concatenate([pos, dirs(rng, n), dirs(rng, n)], 1).astype(np.float32)


def xis(rng, n):
    return (rng.integers(0, 1 << 24, (n, 4)) * 2.0 ** -24).astype(np.float32)


def raw_outputs(rng, n, n_comp=8, stress=False):
    """Raw 8N+1 network outputs.  Benign: small logits like a random-init MLP.
    Stress: lambda, a log-uniform over [1e-4, 1e4] (beyond both clamps),
    large orientation logits (near-degenerate pairs, poles), wide softmax."""
    D = 8 * n_comp + 1
    if not stress:
        return rng.normal(0.0, 0.7, (n, D)).astype(np.float32)
    raw = np.empty((n, D), np.float32)
    raw[:, : 5 * n_comp] = rng.normal(0.0, 4.0, (n, 5 * n_comp))
    raw[:, 5 * n_comp : 7 * n_comp] = rng.uniform(np.log(1e-4), np.log(1e4), (n, 2 * n_comp))
    raw[:, 7 * n_comp : 8 * n_comp] = rng.normal(0.0, 3.0, (n, n_comp))
    raw[:, 8 * n_comp] = rng.normal(0.0, 6.0, n)
    return raw


def samples(rng, n, zero_p_frac=0.1):
    """(n,16) float32 training samples: pos,p, wo,q, n,pbsdf, wi,pad."""
    s = np.zeros((n, 16), np.float32)
    s[:, 0:3] = rng.uniform(-1, 1, (n, 3))
    s[:, 4:7] = dirs(rng, n)
    s[:, 8:11] = dirs(rng, n)
    s[:, 12:15] = dirs(rng, n)
    cos = np.maximum(0.0, np.sum(s[:, 8:11].astype(np.float64) * s[:, 12:15], 1))
    s[:, 11] = cos / np.pi
    s[:, 7] = rng.uniform(0.02, 1.0, n)
    p = rng.exponential(0.5, n) * cos
    p[rng.random(n) < zero_p_frac] = 0.0
    s[:, 3] = p
    return s


def frames(rng, n):
    """(n,3,3) random right-handed orthonormal frames (x, y, z rows)."""
    z = dirs(rng, n).astype(np.float64)
    h = dirs(rng, n).astype(np.float64)
    x = np.cross(h, z)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    y = np.cross(z, x)
    return np.stack([x, y, z], 1)


def nasg_records(rng, n, k, stress=False, eps_frac=0.25):
    """(n,k,12) float32 NASG records (x, lambda, y, a, z, eps) and (n,k) weights.
    Benign: lambda log-uniform [1e-2, 1e2], a log-uniform [1e-2, 1e2];
    stress: lambda to the 3e3 clamp, a in [0, 3e3]; eps > 0 on eps_frac of lobes."""
    f = frames(rng, n * k).reshape(n, k, 3, 3)
    hi = np.log(3e3) if stress else np.log(1e2)
    lam = np.exp(rng.uniform(np.log(1e-2), hi, (n, k)))
    a = np.exp(rng.uniform(np.log(1e-2), hi, (n, k)))
    a[rng.random((n, k)) < 0.1] = 0.0
    eps = np.where(rng.random((n, k)) < eps_frac, rng.uniform(0.0, 2.0, (n, k)), 0.0)
    rec = np.zeros((n, k, 12), np.float64)
    rec[..., 0:3], rec[..., 3] = f[:, :, 0], lam
    rec[..., 4:7], rec[..., 7] = f[:, :, 1], a
    rec[..., 8:11], rec[..., 11] = f[:, :, 2], eps
    w = rng.dirichlet(np.ones(k), n)
    return rec.astype(np.float32), w.astype(np.float32)


def vmf_records(rng, n, k, stress=False):
    """(n,k,4) float32 vMF records (mu, lambda) and (n,k) weights."""
    hi = np.log(3e3) if stress else np.log(1e2)
    rec = np.zeros((n, k, 4), np.float64)
    rec[..., 0:3] = dirs(rng, n * k).reshape(n, k, 3)
    rec[..., 3] = np.exp(rng.uniform(np.log(1e-2), hi, (n, k)))
    w = rng.dirichlet(np.ones(k), n)
    return rec.astype(np.float32), w.astype(np.float32)
