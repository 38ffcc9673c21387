"""TEST INFRASTRUCTURE ONLY — ctypes front-end for the two CPU checkers.

* ``Oracle("orc")`` loads ``oracle/build/libnasg_oracle.so`` — our plain-C
  restatement of the reference hot path (``oracle/nasg_oracle.c``).
* ``Oracle("ref")`` loads ``oracle/_ref/libnasg_ref.so`` — the UNMODIFIED
  reference TUs (``/root/reference/proj/src``) built against the Eigen-API
  shim (``oracle/eigen_shim``) plus the marshalling harness
  ``oracle/ref_capi.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The
product path (``paper_2303_08064_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
def _host_has_v3() -> bool:
    """x86-64-v3 (AVX2 + FMA + BMI2) on this host: the reference build in _ref/
    uses it; a host without it loads the generic build of the same code."""
    try:
        flags = next(l for l in open("/proc/cpuinfo") if l.startswith("flags")).split()
        return all(f in flags for f in ("avx2", "fma", "bmi2", "movbe"))
    except (OSError, StopIteration):
        return False


LIBS = {
    "orc": os.path.join(HERE, "build", "libnasg_oracle.so"),
    "ref": os.path.join(HERE, "_ref", "libnasg_ref.so" if _host_has_v3() else "libnasg_ref_generic.so"),
}

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i64, _u64, _int, _dbl, _flt, _vp = C.c_int64, C.c_uint64, C.c_int, C.c_double, C.c_float, C.c_void_p

_SIGS = {
    "pcg32": (None, [_u64, _u64, _int, _u32p]),
    "init_network": (None, [_u64, _int, _f32p]),
    "one_blob": (None, [_dbl, _int, _f32p]),
    "encode": (_u64, [_i64, _f32p, _f32p, _f32p, _f32p]),
    "forward": (None, [_f32p, _int, _i64, _f32p, _f32p]),
    "backward": (None, [_f32p, _int, _i64, _f32p, _f32p, _f32p]),
    "adam_step": (_int, [_int, _f32p, _f32p, _f32p, _f32p, _i64p, _flt]),
    "norm_const": (_dbl, [_dbl, _dbl, _dbl]),
    "frame_from_euler": (_int, [_dbl, _dbl, _dbl, _dbl, _dbl, _f64p]),
    "nasg_log_eval": (_dbl, [_f64p, _f64p]),
    "nasg_sample": (None, [_f64p, _dbl, _dbl, _dbl, _f64p]),
    "decode": (None, [_i64, _int, _f32p, _f64p]),
    "decode_sample": (None, [_i64, _int, _f32p, _f32p, _f64p, _vp, _int]),
    "decode_pdf": (None, [_i64, _int, _f32p, _f32p, _dbl, _vp, _vp, _vp]),
    "query_sample": (None, [_f32p, _int, _i64, _f32p, _f32p, _f32p, _f32p, _f32p, _vp, _int]),
    "kl_grad": (None, [_i64, _int, _f32p, _f32p, _dbl, _dbl, _f64p, _i32p, _f64p]),
    "dist_pdf": (None, [_int, _i64, _int, _f32p, _f32p, _f32p, _f64p]),
    "dist_sample": (None, [_int, _i64, _int, _f32p, _f32p, _f32p, _f64p]),
    "dist_grad": (None, [_int, _i64, _int, _f32p, _f32p, _f32p, _f64p]),
    "vmf_fit_grad": (None, [_int, _f32p, _i64, _f32p, _f64p, _i32p]),
    "stride_update": (_dbl, [_dbl, _u64, _u64]),
    "blend_coefficient": (_dbl, [_i64, _int, _int]),
    "trainer_create": (_vp, [_int, _int, _int, _int, _flt, _dbl, _u64, _f32p, _f32p]),
    "trainer_destroy": (None, [_vp]),
    "trainer_train": (None, [_vp, _i64, _f32p, _dbl, _f64p]),
    "trainer_get_weights": (None, [_vp, _f32p]),
    "trainer_set_weights": (None, [_vp, _f32p]),
    "save_checkpoint": (_int, [C.c_char_p, _f32p, _int, _int]),
    "load_checkpoint": (_int, [C.c_char_p, _f32p, _int, C.POINTER(C.c_int)]),
    "synth_queries": (None, [_u64, _i64, _i64, _f32p, _f32p, _f32p, _f32p, _f32p, _f32p]),
    "synth_samples": (None, [_u64, _i64, _i64, _f32p, _f32p, _f32p]),
}


def build(quiet: bool = True) -> None:
    """Build the checkers (``make -C oracle``); _ref only if /root/reference exists."""
    out = subprocess.run(["make", "-C", HERE, "all"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind])


def n_weights(out_dim: int, hidden: int = 128) -> int:
    return 64 * hidden + 2 * hidden * hidden + hidden * out_dim


def _layer_shapes(hidden, out_dim):
    return [(64, hidden), (hidden, hidden), (hidden, hidden), (hidden, out_dim)]


def embed_hidden(w, hidden, out_dim=65):
    """Canonical hidden-H weights -> the 128-wide layout with the extra units
    zero (the oracle then computes the hidden-H network exactly)."""
    out, src = [], 0
    for (r, c), (R, Cc) in zip(_layer_shapes(hidden, out_dim), _layer_shapes(128, out_dim)):
        blk = np.zeros((R, Cc), np.float32)
        blk[:r, :c] = np.asarray(w[src:src + r * c], np.float32).reshape(r, c)
        out.append(blk.ravel())
        src += r * c
    return np.concatenate(out)


def extract_hidden(w, hidden, out_dim=65):
    """Inverse of embed_hidden."""
    out, src = [], 0
    for (r, c), (R, Cc) in zip(_layer_shapes(hidden, out_dim), _layer_shapes(128, out_dim)):
        out.append(np.asarray(w[src:src + R * Cc]).reshape(R, Cc)[:r, :c].ravel())
        src += R * Cc
    return np.concatenate(out).astype(np.float32)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Oracle:
    """Uniform wrapper: ``Oracle('orc')`` (restatement) or ``Oracle('ref')`` (reference)."""

    def __init__(self, kind: str = "orc"):
        path = LIBS[kind]
        if not os.path.exists(path):
            if kind == "orc":
                build()
            else:
                raise FileNotFoundError(f"{path} missing (build on a host with /root/reference)")
        self.kind = kind
        self.lib = C.CDLL(path)
        pre = "orc_" if kind == "orc" else "ref_"
        for name, (res, args) in _SIGS.items():
            fn = getattr(self.lib, pre + name)
            fn.restype = res
            fn.argtypes = args
            setattr(self, "_" + name, fn)
        if kind == "orc":  # restatement-only extension (the reference fixes kHiddenUnits = 128)
            fn = self.lib.orc_init_network_hu
            fn.restype, fn.argtypes = None, [_u64, _int, _int, _f32p]
            self._init_network_hu = fn

    # ---- L0 / encoder / net ------------------------------------------------
    def pcg32(self, state, seq, n):
        out = np.empty(n, np.uint32)
        self._pcg32(state, seq, n, out)
        return out

    def init_network(self, seed, out_dim=65):
        w = np.empty(n_weights(out_dim), np.float32)
        self._init_network(seed, out_dim, w)
        return w

    def init_network_hu(self, seed, hidden, out_dim=65):
        """init_network with kHiddenUnits = hidden, canonical hidden-H layout."""
        w = np.empty(n_weights(out_dim, hidden), np.float32)
        self._init_network_hu(seed, hidden, out_dim, w)
        return w

    def one_blob(self, x, k=19):
        out = np.empty(k, np.float32)
        self._one_blob(float(x), k, out)
        return out

    def encode(self, q9, bmin, bmax):
        q9 = np.ascontiguousarray(q9, np.float32).reshape(-1, 9)
        out = np.empty((len(q9), 64), np.float32)
        clamped = self._encode(len(q9), q9, _f3(bmin), _f3(bmax), out)
        return out, int(clamped)

    def forward(self, w, x64, out_dim=65):
        x64 = np.ascontiguousarray(x64, np.float32).reshape(-1, 64)
        out = np.empty((len(x64), out_dim), np.float32)
        self._forward(np.ascontiguousarray(w, np.float32), out_dim, len(x64), x64, out)
        return out

    def backward(self, w, x64, out_grads, out_dim=65):
        x64 = np.ascontiguousarray(x64, np.float32).reshape(-1, 64)
        g = np.ascontiguousarray(out_grads, np.float32).reshape(-1, out_dim)
        dw = np.empty(n_weights(out_dim), np.float32)
        self._backward(np.ascontiguousarray(w, np.float32), out_dim, len(x64), x64, g, dw)
        return dw

    def adam_step(self, w, m, v, g, t, lr=0.002, out_dim=65):
        tt = np.array([t], np.int64)
        ok = self._adam_step(out_dim, w, m, v, np.ascontiguousarray(g, np.float32), tt, lr)
        return bool(ok), int(tt[0])

    # ---- sphdist ------------------------------------------------------------
    def norm_const(self, lam, a=0.0, eps=0.0):
        return self._norm_const(lam, a, eps)

    def frame_from_euler(self, ct, sp, cp, st, ctau):
        out = np.empty(9, np.float64)
        ok = self._frame_from_euler(ct, sp, cp, st, ctau, out)
        return out.reshape(3, 3), bool(ok)  # rows: x, y, z axes

    def nasg_log_eval(self, comp12, v):
        return self._nasg_log_eval(np.ascontiguousarray(comp12, np.float64), np.ascontiguousarray(v, np.float64))

    def nasg_sample(self, comp12, xi0, xi1, xi2):
        out = np.empty(3, np.float64)
        self._nasg_sample(np.ascontiguousarray(comp12, np.float64), xi0, xi1, xi2, out)
        return out

    # ---- guider -------------------------------------------------------------
    def decode(self, raw, n_comp=8):
        raw = np.ascontiguousarray(raw, np.float32).reshape(-1, 8 * n_comp + 1)
        out = np.empty((len(raw), 13 * n_comp + 1), np.float64)
        self._decode(len(raw), n_comp, raw, out)
        return out

    def decode_sample(self, raw, xi, n_comp=8, threads=0):
        raw = np.ascontiguousarray(raw, np.float32).reshape(-1, 8 * n_comp + 1)
        xi = np.ascontiguousarray(xi, np.float32).reshape(-1, 4)
        out = np.empty((len(raw), 4), np.float64)
        c = np.empty(len(raw), np.float64)
        self._decode_sample(len(raw), n_comp, raw, xi, out, _ptr(c), threads)
        return out, c

    def decode_pdf(self, raw, dirs, b=1.0, bsdf_pdf=None, n_comp=8):
        raw = np.ascontiguousarray(raw, np.float32).reshape(-1, 8 * n_comp + 1)
        dirs = np.ascontiguousarray(dirs, np.float32).reshape(-1, 3)
        mix = np.empty(len(raw), np.float64)
        guided = np.empty(len(raw), np.float64)
        bp = None if bsdf_pdf is None else np.ascontiguousarray(bsdf_pdf, np.float32)
        self._decode_pdf(len(raw), n_comp, raw, dirs, b, _ptr(bp), _ptr(mix), _ptr(guided))
        return mix, guided

    def query_sample(self, w, q9, xi, bmin=(-1, -1, -1), bmax=(1, 1, 1), out_dim=65, threads=0):
        q9 = np.ascontiguousarray(q9, np.float32).reshape(-1, 9)
        xi = np.ascontiguousarray(xi, np.float32).reshape(-1, 4)
        out = np.empty((len(q9), 4), np.float32)
        c = np.empty(len(q9), np.float32)
        self._query_sample(np.ascontiguousarray(w, np.float32), out_dim, len(q9), q9, xi,
                           _f3(bmin), _f3(bmax), out, _ptr(c), threads)
        return out, c

    def kl_grad(self, raw, samples, b=1.0, loss_blend=0.2, n_comp=8):
        D = 8 * n_comp + 1
        raw = np.ascontiguousarray(raw, np.float32).reshape(-1, D)
        s = np.ascontiguousarray(samples, np.float32).reshape(-1, 16)
        g = np.empty((len(raw), D), np.float64)
        ok = np.empty(len(raw), np.int32)
        loss = np.empty(len(raw), np.float64)
        self._kl_grad(len(raw), n_comp, raw, s, b, loss_blend, g, ok, loss)
        return g, ok.astype(bool), loss

    # ---- explicit mixtures (sphdist.hpp) and the fit's vMF model ------------------
    # kind 0 = NASG (12-float records), 1 = vMF (4-float records); comp is
    # (n, k, rec) float32, w (n, k), dirs / xi (n, 4)
    def _dist_args(self, kind, comp, w, v4):
        rec = 12 if kind == 0 else 4
        w = np.ascontiguousarray(w, np.float32)
        n, k = w.shape
        comp = np.ascontiguousarray(comp, np.float32).reshape(n, k, rec)
        v4 = np.ascontiguousarray(v4, np.float32).reshape(n, 4)
        return n, k, comp, w, v4

    def dist_pdf(self, kind, comp, w, dirs):
        n, k, comp, w, d = self._dist_args(kind, comp, w, dirs)
        out = np.empty(n, np.float64)
        self._dist_pdf(kind, n, k, comp, w, d, out)
        return out

    def dist_sample(self, kind, comp, w, xi):
        n, k, comp, w, x = self._dist_args(kind, comp, w, xi)
        out = np.empty((n, 4), np.float64)
        self._dist_sample(kind, n, k, comp, w, x, out)
        return out

    def dist_grad(self, kind, comp, w, dirs):
        n, k, comp, w, d = self._dist_args(kind, comp, w, dirs)
        out = np.empty((n, k, 8 if kind == 0 else 4), np.float64)
        self._dist_grad(kind, n, k, comp, w, d, out)
        return out

    def vmf_fit_grad(self, raw, samples4):
        raw = np.ascontiguousarray(raw, np.float32)
        k = len(raw) // 5
        s = np.ascontiguousarray(samples4, np.float32).reshape(-1, 4)
        g = np.empty((len(s), 5 * k), np.float64)
        ok = np.empty(len(s), np.int32)
        self._vmf_fit_grad(k, raw, len(s), s, g, ok)
        return g, ok.astype(bool)

    def stride_update(self, l, s, cap):
        return self._stride_update(l, s, cap)

    def blend_coefficient(self, i, m=4, bsteps=64):
        return self._blend_coefficient(i, m, bsteps)

    # ---- checkpoint -----------------------------------------------------------
    def save_checkpoint(self, path, w, out_dim=65, n_comp=8):
        return self._save_checkpoint(path.encode(), np.ascontiguousarray(w, np.float32), out_dim, n_comp)

    def load_checkpoint(self, path, max_floats=1 << 20):
        w = np.empty(max_floats, np.float32)
        n = C.c_int(0)
        total = self._load_checkpoint(path.encode(), w, max_floats, C.byref(n))
        if total < 0:
            raise IOError(f"checkpoint load failed ({total}): {path}")
        return w[:total].copy(), n.value

    # ---- synthetic workloads (byte-identical to nasg.synth_*) -------------------
    def synth_queries(self, seed, n, first=0, bmin=(-1, -1, -1), bmax=(1, 1, 1)):
        """(n,4) float32 x4: x, wo, nrm, xi — SURVEY §8d synthetic queries."""
        arrs = [np.empty((n, 4), np.float32) for _ in range(4)]
        self._synth_queries(seed, first, n, _f3(bmin), _f3(bmax), *arrs)
        return tuple(arrs)

    def synth_samples(self, seed, n, first=0, bmin=(-1, -1, -1), bmax=(1, 1, 1)):
        """(n,16) float32 training samples (nasg_train_sample layout)."""
        out = np.empty((n, 16), np.float32)
        self._synth_samples(seed, first, n, _f3(bmin), _f3(bmax), out)
        return out

    # ---- trainer --------------------------------------------------------------
    def set_reverse_sum(self, on: bool):
        """Restatement only: sum dW over batch rows in reverse (reassociation yardstick)."""
        fn = self.lib.orc_set_reverse_sum
        fn.argtypes, fn.restype = [C.c_int], None
        fn(int(on))

    def trainer(self, **kw):
        return _Trainer(self, **kw)


class _Trainer:
    def __init__(self, o: Oracle, n_comp=8, capacity=1 << 16, batch=1 << 12, step_factor=1,
                 lr=0.002, loss_blend=0.2, seed=0, bmin=(-1, -1, -1), bmax=(1, 1, 1)):
        self.o, self.n_comp = o, n_comp
        self.h = o._trainer_create(n_comp, capacity, batch, step_factor, lr, loss_blend, seed,
                                   _f3(bmin), _f3(bmax))

    def __del__(self):
        if getattr(self, "h", None):
            self.o._trainer_destroy(self.h)
            self.h = None

    def train(self, samples, b):
        s = np.ascontiguousarray(samples, np.float32).reshape(-1, 16)
        st = np.zeros(4, np.float64)
        self.o._trainer_train(self.h, len(s), s, b, st)
        return {"steps": int(st[0]), "mean_loss": float(st[1]), "dropped": int(st[2]), "skipped": int(st[3])}

    def weights(self):
        w = np.empty(n_weights(8 * self.n_comp + 1), np.float32)
        self.o._trainer_get_weights(self.h, w)
        return w

    def set_weights(self, w):
        self.o._trainer_set_weights(self.h, np.ascontiguousarray(w, np.float32))


def _f3(v):
    return np.ascontiguousarray(np.asarray(v, np.float32).reshape(3))
