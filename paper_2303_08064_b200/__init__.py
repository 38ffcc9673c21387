"""B200-native NASG online path-guiding hot path (arXiv 2303.08064).

Thin ctypes binding of the C ABI in ``include/nasg/nasg.h`` (implemented in
``csrc/`` and built to ``lib/libnasg_b200.so`` for sm_100a).  It mirrors the
reference's C++ guiding API nouns (guiding.hpp): ``TrainerConfig``,
``TrainStats``, ``Trainer.train_iteration``, ``publish``/``snapshot``,
``infer_guide`` + ``mixture_sample`` (batched as ``query_sample``),
``guided_pdf`` (``query_pdf``), ``decode`` (``decode_sample_raw``).

Device buffers are passed as torch CUDA tensors (PyTorch is used only for
device memory and streams); host buffers as numpy arrays.  There is no CPU
fallback: every call runs the CUDA library or raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# NASG_LIB selects another build of the same library (A/B experiments only)
LIB_PATH = os.environ.get("NASG_LIB") or os.path.join(_HERE, "lib", "libnasg_b200.so")

NASG_MLP_FP32 = 0
NASG_MLP_BF16 = 1


class NasgError(RuntimeError):
    pass


class _Config(C.Structure):
    _fields_ = [("n_components", C.c_int), ("sample_capacity", C.c_int), ("batch_size", C.c_int),
                ("step_factor", C.c_int), ("learning_rate", C.c_float), ("loss_blend", C.c_double),
                ("seed", C.c_uint64), ("hidden_units", C.c_int)]


class _Stats(C.Structure):
    _fields_ = [("steps", C.c_int), ("mean_loss", C.c_double), ("dropped_samples", C.c_uint64),
                ("skipped_updates", C.c_uint64)]


class _Counters(C.Structure):
    _fields_ = [("encode_clamps", C.c_uint64), ("kernel_launches", C.c_uint64), ("adam_steps", C.c_int64),
                ("iterations", C.c_int64), ("rank", C.c_int), ("nranks", C.c_int), ("collectives", C.c_uint64)]


class _RenderConfig(C.Structure):
    _fields_ = [("scene", C.c_int), ("width", C.c_int), ("height", C.c_int), ("row_begin", C.c_int),
                ("row_end", C.c_int), ("seed", C.c_uint64), ("max_depth", C.c_int), ("rr_depth", C.c_int),
                ("guiding", C.c_int), ("collect", C.c_int), ("ramp", C.c_int), ("schedule_m", C.c_int),
                ("schedule_b", C.c_int), ("nee", C.c_int), ("lazy_train_stats", C.c_int),
                ("pipelined", C.c_int), ("row_band", C.c_int), ("shard", C.c_int), ("nshards", C.c_int)]


class _RenderStats(C.Structure):
    _fields_ = [("iteration", C.c_int64), ("b", C.c_double), ("stride", C.c_double), ("paths", C.c_int64),
                ("vertices", C.c_int64), ("guided_vertices", C.c_int64), ("collected", C.c_int64),
                ("kept", C.c_int64), ("nonfinite_paths", C.c_int64), ("train", _Stats)]


SCENE_FURNACE, SCENE_BOX, SCENE_CRACK, SCENE_DARK, SCENE_ATTIC, SCENE_INDIRECT = 0, 1, 2, 3, 4, 5


@dataclass
class TrainerConfig:
    """TrainerConfig (guiding.hpp:122-130)."""
    n_components: int = 8
    sample_capacity: int = 1 << 16
    batch_size: int = 1 << 12
    step_factor: int = 1
    learning_rate: float = 0.002
    loss_blend: float = 0.2
    seed: int = 0
    hidden_units: int = 128  # kHiddenUnits (net.hpp); 64 = the paper's smaller network (nasg.h)


@dataclass
class TrainStats:
    """TrainStats (guiding.hpp:132-137)."""
    steps: int
    mean_loss: float
    dropped_samples: int
    skipped_updates: int


_lib = None


def lib():
    """Load libnasg_b200.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NasgError(f"CUDA library missing: {LIB_PATH} (run `python -c 'import __graft_entry__ as g; g.build()'`)")
    L = C.CDLL(LIB_PATH)
    vp, i64, u64, i32, f32, f64, sz = C.c_void_p, C.c_int64, C.c_uint64, C.c_int, C.c_float, C.c_double, C.c_size_t
    sigs = {
        "nasg_config_default": (None, [vp]),
        "nasg_create": (i32, [vp, i32, vp, vp, C.POINTER(vp)]),
        "nasg_destroy": (i32, [vp]),
        "nasg_status_string": (C.c_char_p, [i32]),
        "nasg_last_error": (C.c_char_p, []),
        "nasg_n_weights": (i32, [i32]),
        "nasg_n_weights_hu": (i32, [i32, i32]),
        "nasg_set_weights": (i32, [vp, vp, sz]),
        "nasg_get_weights": (i32, [vp, vp, sz, i32]),
        "nasg_publish": (i32, [vp]),
        "nasg_set_precision": (i32, [vp, i32]),
        "nasg_get_precision": (i32, [vp]),
        "nasg_set_train_precision": (i32, [vp, i32]),
        "nasg_get_train_precision": (i32, [vp]),
        "nasg_set_zero_row_skip": (i32, [vp, i32]),
        "nasg_get_zero_row_skip": (i32, [vp]),
        "nasg_save_checkpoint": (i32, [vp, C.c_char_p]),
        "nasg_save_checkpoint_ex": (i32, [vp, C.c_char_p, i32]),
        "nasg_load_checkpoint": (i32, [vp, C.c_char_p]),
        "nasg_query_sample": (i32, [vp, i64, vp, vp, vp, vp, vp, vp, vp]),
        "nasg_query_pdf": (i32, [vp, i64, vp, vp, vp, vp, f32, vp, vp, vp, vp]),
        "nasg_query_raw": (i32, [vp, i64, vp, vp, vp, vp, vp]),
        "nasg_query_shade": (i32, [vp, i64, vp, vp, vp, vp, vp, vp, vp, f32, vp, vp]),
        "nasg_decode_sample_raw": (i32, [vp, i64, vp, vp, vp, vp, vp]),
        "nasg_decode_pdf_raw": (i32, [vp, i64, vp, vp, f32, vp, vp, vp, vp]),
        "nasg_query_sample_host": (i32, [vp, i64, vp, vp, vp, vp, vp, vp]),
        "nasg_query_sample_packed": (i32, [vp, i64, vp, vp, vp, vp]),
        "nasg_query_sample_host_packed": (i32, [vp, i64, vp, vp, vp]),
        "nasg_train_iteration": (i32, [vp, i64, vp, f64, vp, vp]),
        "nasg_train_step": (i32, [vp, vp, vp, i64, i64, f64, vp]),
        "nasg_train_stats_take": (i32, [vp, vp]),
        "nasg_get_last_grad": (i32, [vp, vp, sz]),
        "nasg_adam_t": (i64, [vp]),
        "nasg_comm_unique_id": (i32, [vp]),
        "nasg_comm_init": (i32, [vp, vp, i32, i32]),
        "nasg_attach_nccl": (i32, [vp, vp, i32, i32]),
        "nasg_get_counters": (i32, [vp, vp]),
        "nasg_encode_clamp_count": (u64, [vp]),
        "nasg_reset_encode_clamp_count": (None, [vp]),
        "nasg_kernel_launches": (u64, [vp]),
        "nasg_blend_coefficient": (f64, [i64, i32, i32]),
        "nasg_stride_update": (f64, [f64, u64, u64]),
        "nasg_synth_queries": (None, [u64, i64, i64, vp, vp, vp, vp, vp, vp]),
        "nasg_synth_samples": (None, [u64, i64, i64, vp, vp, vp]),
        "nasg_dp_plan": (i32, [vp, vp, i32, i32, i32, vp, vp, vp]),
        "nasg_render_config_default": (None, [vp]),
        "nasg_render_scene_bounds": (i32, [i32, vp, vp]),
        "nasg_render_create": (i32, [vp, vp, C.POINTER(vp)]),
        "nasg_render_destroy": (i32, [vp]),
        "nasg_render_iteration": (i32, [vp, vp]),
        "nasg_render_image": (i32, [vp, vp, i32]),
        "nasg_render_kernel_launches": (u64, [vp]),
        "nasg_mape": (f64, [vp, vp, i64]),
        "nasg_dist_mixture_pdf": (i32, [i32, i64, i32, vp, vp, vp, vp, vp]),
        "nasg_dist_mixture_sample": (i32, [i32, i64, i32, vp, vp, vp, vp, vp]),
        "nasg_dist_grad_logpdf": (i32, [i32, i64, i32, vp, vp, vp, vp, vp]),
        "nasg_fit_raw_dim": (i32, [i32, i32]),
        "nasg_fit": (i32, [vp, i32, i32, i32, vp, vp, vp, vp, vp, i32]),
        "nasg_fit_gradient": (i32, [i32, i32, vp, i64, vp, vp]),
        "nasg_fit_kl": (i32, [i32, i32, vp, vp, i32, i32, i32, vp, i32, vp]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    _lib = L
    return L


def exported_symbols():
    """Names of every function declared in include/nasg/nasg.h."""
    import re
    hdr = os.path.join(os.path.dirname(_HERE), "include", "nasg", "nasg.h")
    txt = re.sub(r"/\*.*?\*/", "", open(hdr).read(), flags=re.S)
    return sorted(set(re.findall(r"\b(nasg_[a-z0-9_]+)\s*\(", txt)))


def _check(rc):
    if rc != 0:
        L = lib()
        raise NasgError(f"{L.nasg_status_string(rc).decode()}: {L.nasg_last_error().decode()}")


def _f3(v):
    return np.ascontiguousarray(np.asarray(v, np.float32).reshape(3))


def _ptr(t):
    """Device pointer of a torch tensor (or None), host pointer of a numpy array."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    if hasattr(t, "data_ptr"):
        if not t.is_contiguous():
            raise NasgError("tensor must be contiguous")
        return t.data_ptr()
    return int(t)


_CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: torch's default stream has handle 0


def _stream(stream):
    """Stream handle for the C ABI; defaults to torch's current stream so that
    results are ordered with the caller's torch work (NULL would mean the
    context's private stream)."""
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    h = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    return h if h else _CUDA_STREAM_LEGACY


def n_weights(n_components: int = 8, hidden_units: int = 128) -> int:
    return lib().nasg_n_weights_hu(n_components, hidden_units)


def blend_coefficient(iteration: int, m: int = 4, b_steps: int = 64) -> float:
    """BlendSchedule::coefficient (guiding.hpp:83-86)."""
    return lib().nasg_blend_coefficient(iteration, m, b_steps)


def stride_update(l: float, collected: int, capacity: int) -> float:
    """stride_update (guiding.cpp:178-182)."""
    return lib().nasg_stride_update(l, collected, capacity)


def synth_queries(seed: int, n: int, first: int = 0, bmin=(-1, -1, -1), bmax=(1, 1, 1), pinned: bool = False):
    """Synthetic queries of SURVEY.md §8d as host float32 arrays (n,4) x 4: x, wo, nrm, xi."""
    arrs = []
    for _ in range(4):
        if pinned:
            import torch
            arrs.append(torch.empty((n, 4), dtype=torch.float32).pin_memory().numpy())
        else:
            arrs.append(np.empty((n, 4), np.float32))
    lo, hi = _f3(bmin), _f3(bmax)  # keep alive across the call
    lib().nasg_synth_queries(seed, first, n, lo.ctypes.data, hi.ctypes.data,
                             *[a.ctypes.data for a in arrs])
    return tuple(arrs)


def synth_samples(seed: int, n: int, first: int = 0, bmin=(-1, -1, -1), bmax=(1, 1, 1)):
    """Synthetic training samples (n,16) float32 (nasg_train_sample layout)."""
    out = np.empty((n, 16), np.float32)
    lo, hi = _f3(bmin), _f3(bmax)
    lib().nasg_synth_samples(seed, first, n, lo.ctypes.data, hi.ctypes.data, out.ctypes.data)
    return out


def dp_plan(config: TrainerConfig, n_per_rank, rank: int):
    """Data-parallel minibatch plan of one train_iteration (host-only, see nasg.h):
    returns (local_count, global_count, reshuffle_before) arrays, one entry per step."""
    cfg = _Config(config.n_components, config.sample_capacity, config.batch_size, config.step_factor,
                  config.learning_rate, config.loss_blend, config.seed, config.hidden_units)
    n_all = np.ascontiguousarray(n_per_rank, np.int64)
    max_steps = config.step_factor * -(-config.sample_capacity // config.batch_size)
    loc = np.zeros(max_steps, np.int64)
    glo = np.zeros(max_steps, np.int64)
    res = np.zeros(max_steps, np.int32)
    steps = lib().nasg_dp_plan(C.byref(cfg), n_all.ctypes.data, len(n_all), rank, max_steps, loc.ctypes.data,
                               glo.ctypes.data, res.ctypes.data)
    if steps < 0:
        raise NasgError("bad data-parallel plan arguments")
    return loc[:steps], glo[:steps], res[:steps].astype(bool)


class Guide:
    """One GPU's guiding context: live Trainer state + published snapshot.

    Mirrors ``nasg::Trainer`` (guiding.hpp:142-166) and the per-point query
    functions, batched over device tensors.
    """

    def __init__(self, config: TrainerConfig | None = None, device: int | None = None, bmin=(-1, -1, -1),
                 bmax=(1, 1, 1)):
        """device: CUDA ordinal (default: torch's current device, else 0)."""
        self.config = config or TrainerConfig()
        if device is None:
            try:
                import torch
                device = torch.cuda.current_device() if torch.cuda.is_available() else 0
            except ImportError:
                device = 0
        cfg = _Config(self.config.n_components, self.config.sample_capacity, self.config.batch_size,
                      self.config.step_factor, self.config.learning_rate, self.config.loss_blend, self.config.seed,
                      self.config.hidden_units)
        h = C.c_void_p()
        lo, hi = _f3(bmin), _f3(bmax)
        _check(lib().nasg_create(C.byref(cfg), device, lo.ctypes.data, hi.ctypes.data, C.byref(h)))
        self._h = h
        self.device = device
        self.n_components = self.config.n_components
        self.out_dim = 8 * self.n_components + 1
        self.nw = n_weights(self.n_components, self.config.hidden_units)

    def close(self):
        if getattr(self, "_h", None):
            lib().nasg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- parameters ------------------------------------------------------------
    def set_weights(self, w):
        w = np.ascontiguousarray(w, np.float32)
        _check(lib().nasg_set_weights(self._h, w.ctypes.data, w.size))

    def get_weights(self, published: bool = False):
        w = np.empty(self.nw, np.float32)
        _check(lib().nasg_get_weights(self._h, w.ctypes.data, w.size, int(published)))
        return w

    def publish(self):
        _check(lib().nasg_publish(self._h))

    @property
    def precision(self) -> int:
        return lib().nasg_get_precision(self._h)

    @precision.setter
    def precision(self, p: int):
        _check(lib().nasg_set_precision(self._h, int(p)))

    @property
    def train_precision(self) -> int:
        """MLP arithmetic of training (NASG_MLP_FP32 default, NASG_MLP_BF16 tensor cores)."""
        return lib().nasg_get_train_precision(self._h)

    @train_precision.setter
    def train_precision(self, p: int):
        _check(lib().nasg_set_train_precision(self._h, int(p)))

    @property
    def zero_row_skip(self) -> bool:
        """bf16 trainer: p = 0 rows counted without the network pass (nasg_set_zero_row_skip)."""
        return lib().nasg_get_zero_row_skip(self._h) == 1

    @zero_row_skip.setter
    def zero_row_skip(self, on: bool):
        _check(lib().nasg_set_zero_row_skip(self._h, 1 if on else 0))

    def save_checkpoint(self, path: str, optimizer: bool = False):
        """NASGNET1 weights; optimizer=True appends the Adam state (nasg_save_checkpoint_ex)."""
        if optimizer:
            _check(lib().nasg_save_checkpoint_ex(self._h, path.encode(), 1))
        else:
            _check(lib().nasg_save_checkpoint(self._h, path.encode()))

    def load_checkpoint(self, path: str):
        _check(lib().nasg_load_checkpoint(self._h, path.encode()))

    @property
    def kernel_launches(self) -> int:
        return lib().nasg_kernel_launches(self._h)

    def counters(self) -> dict:
        """nasg_get_counters: clamps, launches, Adam t, iterations, rank / nranks."""
        c = _Counters()
        _check(lib().nasg_get_counters(self._h, C.byref(c)))
        return {k: getattr(c, k) for k, _ in _Counters._fields_}

    def attach_nccl(self, comm_handle: int, rank: int, nranks: int):
        """nasg_attach_nccl with an existing ncclComm_t (an integer handle)."""
        _check(lib().nasg_attach_nccl(self._h, comm_handle, rank, nranks))

    @property
    def encode_clamp_count(self) -> int:
        return lib().nasg_encode_clamp_count(self._h)

    def reset_encode_clamp_count(self):
        lib().nasg_reset_encode_clamp_count(self._h)

    # ---- queries (torch CUDA tensors, (n,4) float32) --------------------------------
    def query_sample(self, x, wo, nrm, xi, dir_pdf=None, c=None, stream=None):
        import torch
        n = x.shape[0]
        if dir_pdf is None:
            dir_pdf = torch.empty((n, 4), dtype=torch.float32, device=x.device)
        _check(lib().nasg_query_sample(self._h, n, _ptr(x), _ptr(wo), _ptr(nrm), _ptr(xi), _ptr(dir_pdf), _ptr(c),
                                       _stream(stream)))
        return dir_pdf, c

    def query_pdf(self, x, wo, nrm, dirs, b, bsdf_pdf=None, stream=None):
        import torch
        n = x.shape[0]
        mix = torch.empty(n, dtype=torch.float32, device=x.device)
        guided = torch.empty(n, dtype=torch.float32, device=x.device)
        _check(lib().nasg_query_pdf(self._h, n, _ptr(x), _ptr(wo), _ptr(nrm), _ptr(dirs), float(b), _ptr(bsdf_pdf),
                                    _ptr(mix), _ptr(guided), _stream(stream)))
        return mix, guided

    def query_shade(self, x, wo, nrm, xi, d_bsdf, d_nee, b, n_dev=None, stream=None):
        """Guided scattering at path vertices (nasg_query_shade): returns (n, 2, 4)
        [(dir xyz, q_mix(dir)), (q_mix(nee), c', guided, c)]."""
        import torch
        n = x.shape[0]
        out = torch.empty((n, 2, 4), dtype=torch.float32, device=x.device)
        _check(lib().nasg_query_shade(self._h, n, _ptr(n_dev), _ptr(x), _ptr(wo), _ptr(nrm), _ptr(xi), _ptr(d_bsdf),
                                      _ptr(d_nee), float(b), _ptr(out), _stream(stream)))
        return out

    def query_raw(self, x, wo, nrm, stream=None):
        import torch
        n = x.shape[0]
        raw = torch.empty((n, self.out_dim), dtype=torch.float32, device=x.device)
        _check(lib().nasg_query_raw(self._h, n, _ptr(x), _ptr(wo), _ptr(nrm), _ptr(raw), _stream(stream)))
        return raw

    def decode_sample_raw(self, raw, xi, stream=None):
        import torch
        n = raw.shape[0]
        out = torch.empty((n, 4), dtype=torch.float32, device=raw.device)
        c = torch.empty(n, dtype=torch.float32, device=raw.device)
        _check(lib().nasg_decode_sample_raw(self._h, n, _ptr(raw), _ptr(xi), _ptr(out), _ptr(c), _stream(stream)))
        return out, c

    def decode_pdf_raw(self, raw, dirs, b, bsdf_pdf=None, stream=None):
        import torch
        n = raw.shape[0]
        mix = torch.empty(n, dtype=torch.float32, device=raw.device)
        guided = torch.empty(n, dtype=torch.float32, device=raw.device)
        _check(lib().nasg_decode_pdf_raw(self._h, n, _ptr(raw), _ptr(dirs), float(b), _ptr(bsdf_pdf), _ptr(mix),
                                         _ptr(guided), _stream(stream)))
        return mix, guided

    def query_sample_host(self, x, wo, nrm, xi, dir_pdf=None, c=None):
        """Host numpy in/out; H2D, kernel and D2H are pipelined inside the library."""
        n = x.shape[0]
        if dir_pdf is None:
            dir_pdf = np.empty((n, 4), np.float32)
        _check(lib().nasg_query_sample_host(self._h, n, _ptr(x), _ptr(wo), _ptr(nrm), _ptr(xi), _ptr(dir_pdf),
                                            _ptr(c)))
        return dir_pdf, c

    def query_sample_packed(self, q13, dir_pdf=None, c=None, stream=None):
        """Device (n,13) float32 rows: position, omega_o, normal, xi."""
        import torch
        n = q13.shape[0]
        if dir_pdf is None:
            dir_pdf = torch.empty((n, 4), dtype=torch.float32, device=q13.device)
        _check(lib().nasg_query_sample_packed(self._h, n, _ptr(q13), _ptr(dir_pdf), _ptr(c), _stream(stream)))
        return dir_pdf, c

    def query_sample_host_packed(self, q13, dir_pdf=None, c=None):
        """Host (n,13) float32 rows; 52 B/query over PCIe."""
        n = q13.shape[0]
        if dir_pdf is None:
            dir_pdf = np.empty((n, 4), np.float32)
        _check(lib().nasg_query_sample_host_packed(self._h, n, _ptr(q13), _ptr(dir_pdf), _ptr(c)))
        return dir_pdf, c

    # ---- training ----------------------------------------------------------------------
    def train_iteration(self, samples, blend_b: float, stream=None, stats: bool = True) -> TrainStats | None:
        """Trainer::train_iteration (guiding.cpp:196-282) on a device (n,16) float32 tensor."""
        n = 0 if samples is None else samples.shape[0]
        st = _Stats()
        _check(lib().nasg_train_iteration(self._h, n, _ptr(samples) if n else None, float(blend_b),
                                          C.byref(st) if stats else None, _stream(stream)))
        if not stats:
            return None
        return TrainStats(st.steps, st.mean_loss, st.dropped_samples, st.skipped_updates)

    def train_step(self, samples, order, count: int, global_count: int, blend_b: float, stream=None):
        _check(lib().nasg_train_step(self._h, _ptr(samples), _ptr(order), count, global_count, float(blend_b),
                                     _stream(stream)))

    def train_stats_take(self) -> TrainStats:
        st = _Stats()
        _check(lib().nasg_train_stats_take(self._h, C.byref(st)))
        return TrainStats(st.steps, st.mean_loss, st.dropped_samples, st.skipped_updates)

    def last_grad(self):
        g = np.empty(self.nw, np.float32)
        _check(lib().nasg_get_last_grad(self._h, g.ctypes.data, g.size))
        return g

    @property
    def adam_t(self) -> int:
        return lib().nasg_adam_t(self._h)

    # ---- multi-GPU ------------------------------------------------------------------------
    @staticmethod
    def comm_unique_id() -> bytes:
        buf = (C.c_char * 128)()
        _check(lib().nasg_comm_unique_id(buf))
        return bytes(buf)

    def comm_init(self, unique_id: bytes, rank: int, nranks: int):
        buf = (C.c_char * 128).from_buffer_copy(unique_id)
        _check(lib().nasg_comm_init(self._h, buf, rank, nranks))


# ---- guided progressive render loop (SPEC.md tracer module; nasg_render_*) -----------
def scene_bounds(scene: int):
    lo, hi = np.zeros(3, np.float32), np.zeros(3, np.float32)
    _check(lib().nasg_render_scene_bounds(scene, lo.ctypes.data, hi.ctypes.data))
    return lo, hi


def mape(img, ref) -> float:
    """SPEC.md tracer mape (PAPER §7): relative error with eps 0.01, worst 0.1 % dropped."""
    a = np.ascontiguousarray(img, np.float32).reshape(-1, 3)
    b = np.ascontiguousarray(ref, np.float32).reshape(-1, 3)
    if a.shape != b.shape:
        raise NasgError("mape: dimension mismatch")
    return lib().nasg_mape(a.ctypes.data, b.ctypes.data, a.shape[0])


class Render:
    """nasg_render: wavefront guided path tracer + online training on one GPU's pixel rows."""

    def __init__(self, guide: Guide, scene: int = SCENE_BOX, width: int = 256, height: int = 256,
                 row_begin: int = 0, row_end: int = 0, seed: int = 1, guiding: bool = True,
                 collect: bool = True, ramp: bool = True, max_depth: int = 16, rr_depth: int = 5,
                 schedule_m: int = 4, schedule_b: int = 64, nee: bool = True, lazy_train_stats: bool = False,
                 pipelined: bool = False, row_band: int = 0, shard: int = 0, nshards: int = 1):
        cfg = _RenderConfig()
        lib().nasg_render_config_default(C.byref(cfg))
        cfg.scene, cfg.width, cfg.height = scene, width, height
        cfg.row_begin, cfg.row_end, cfg.seed = row_begin, row_end, seed
        cfg.max_depth, cfg.rr_depth = max_depth, rr_depth
        cfg.guiding, cfg.collect, cfg.ramp = int(guiding), int(collect), int(ramp)
        cfg.schedule_m, cfg.schedule_b = schedule_m, schedule_b
        cfg.nee = int(nee)
        cfg.lazy_train_stats = int(lazy_train_stats)
        cfg.pipelined = int(pipelined)
        cfg.row_band, cfg.shard, cfg.nshards = row_band, shard, nshards
        h = C.c_void_p()
        _check(lib().nasg_render_create(guide._h, C.byref(cfg), C.byref(h)))
        self._h, self.guide = h, guide
        self.width = width
        if row_band > 0:
            self.rows = sum(min(height, (k + 1) * row_band) - k * row_band
                            for k in range(shard, -(-height // row_band), nshards))
        else:
            self.rows = (row_end if row_end > 0 else height) - row_begin

    def iteration(self) -> dict:
        st = _RenderStats()
        _check(lib().nasg_render_iteration(self._h, C.byref(st)))
        out = {k: getattr(st, k) for k, _ in _RenderStats._fields_ if k != "train"}
        out["train"] = TrainStats(st.train.steps, st.train.mean_loss, st.train.dropped_samples,
                                  st.train.skipped_updates)
        return out

    def image(self, which: int = 0) -> np.ndarray:
        img = np.empty((self.rows, self.width, 3), np.float32)
        _check(lib().nasg_render_image(self._h, img.ctypes.data, which))
        return img

    @property
    def kernel_launches(self) -> int:
        return lib().nasg_render_kernel_launches(self._h)

    def close(self):
        if getattr(self, "_h", None):
            lib().nasg_render_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- explicit-parameter mixtures: NASG and the vMF / SG baseline (sphdist.hpp) --
DIST_NASG, DIST_VMF = 0, 1
_REC = {DIST_NASG: 12, DIST_VMF: 4}


def _dist(fn, kind, comp, weights, v4, out, stream):
    n, k = weights.shape
    if comp.numel() != n * k * _REC[kind] or v4.numel() != 4 * n:
        raise NasgError("shape mismatch")
    _check(fn(kind, n, k, _ptr(comp), _ptr(weights), _ptr(v4), _ptr(out), _stream(stream)))
    return out


def dist_mixture_pdf(kind, comp, weights, dirs, stream=None):
    """mixture_pdf (sphdist.hpp:84) / vmf_mixture_pdf (:117) over per-query explicit
    mixtures.  comp (n, k, 12|4) float32 records, weights (n, k), dirs (n, 4) CUDA tensors."""
    import torch
    out = torch.empty(weights.shape[0], dtype=torch.float32, device=weights.device)
    return _dist(lib().nasg_dist_mixture_pdf, kind, comp, weights, dirs, out, stream)


def dist_mixture_sample(kind, comp, weights, xi, stream=None):
    """mixture_sample (sphdist.hpp:97-98) / vmf_mixture_sample (:119-120): (n, 4) dir + pdf."""
    import torch
    out = torch.empty((weights.shape[0], 4), dtype=torch.float32, device=weights.device)
    return _dist(lib().nasg_dist_mixture_sample, kind, comp, weights, xi, out, stream)


def dist_grad_logpdf(kind, comp, weights, dirs, stream=None):
    """nasg_grad_logpdf (sphdist.hpp:68-71, 8 floats per component) /
    vmf_grad_logpdf (:121, 4 floats) for every component: (n, k, 8|4)."""
    import torch
    n, k = weights.shape
    out = torch.empty((n, k, 8 if kind == DIST_NASG else 4), dtype=torch.float32, device=weights.device)
    return _dist(lib().nasg_dist_grad_logpdf, kind, comp, weights, dirs, out, stream)


class _FitConfig(C.Structure):
    _fields_ = [("model", C.c_int), ("n_components", C.c_int), ("batch", C.c_int), ("steps", C.c_int),
                ("checkpoints", C.c_int), ("learning_rate", C.c_float), ("seed", C.c_uint64)]


@dataclass
class FitConfig:
    """SPEC run_fit: fit one position-free guide distribution."""
    model: int = DIST_NASG
    n_components: int = 8
    batch: int = 1024
    steps: int = 1000
    checkpoints: int = 10
    learning_rate: float = 0.01
    seed: int = 0


def fit_raw_dim(model: int, n_components: int) -> int:
    return lib().nasg_fit_raw_dim(model, n_components)


def _host_f32(a):
    return np.ascontiguousarray(np.asarray(a, np.float32))


def fit(config: FitConfig, n_fits: int, target_kind: int, target_comp, target_w, raw_init=None, quad_nz: int = 256):
    """Fits n_fits models (one CTA each) to the target mixture; returns
    (raw snapshots (n_fits, checkpoints, D), KL(target || model) (n_fits, checkpoints))."""
    D = fit_raw_dim(config.model, config.n_components)
    if D < 0:
        raise NasgError("unsupported fit model")
    tw = _host_f32(target_w).reshape(-1)
    tc = _host_f32(target_comp).reshape(len(tw), _REC[target_kind])
    init = None if raw_init is None else _host_f32(raw_init).reshape(n_fits, D)
    raw = np.empty((n_fits, config.checkpoints, D), np.float32)
    kl = np.empty((n_fits, config.checkpoints), np.float64)
    c = _FitConfig(config.model, config.n_components, config.batch, config.steps, config.checkpoints,
                   config.learning_rate, config.seed)
    _check(lib().nasg_fit(C.byref(c), n_fits, target_kind, len(tw), _ptr(tc), _ptr(tw), _ptr(init), _ptr(raw),
                          _ptr(kl) if quad_nz > 0 else None, quad_nz))
    return raw, kl


def fit_gradient(model: int, n_components: int, raw, samples4):
    """The fit's mean gradient over given (direction xyz, target pdf) rows."""
    raw = _host_f32(raw).reshape(-1)
    s = _host_f32(samples4).reshape(-1, 4)
    g = np.empty(len(raw), np.float32)
    _check(lib().nasg_fit_gradient(model, n_components, _ptr(raw), len(s), _ptr(s), _ptr(g)))
    return g


def fit_kl(target_kind: int, target_comp, target_w, model: int, n_components: int, raws, quad_nz: int = 256):
    """KL(target || model) on the equal-area quad_nz x 2 quad_nz grid, per raw vector."""
    D = fit_raw_dim(model, n_components)
    raws = _host_f32(raws).reshape(-1, D)
    tw = _host_f32(target_w).reshape(-1)
    tc = _host_f32(target_comp).reshape(len(tw), _REC[target_kind])
    kl = np.empty(len(raws), np.float64)
    _check(lib().nasg_fit_kl(target_kind, len(tw), _ptr(tc), _ptr(tw), model, n_components, len(raws), _ptr(raws),
                             quad_nz, _ptr(kl)))
    return kl
