"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and its host-only helpers behave (no GPU calls here)."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_2303_08064_b200 as nasg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_built_for_sm100a():
    assert os.path.exists(nasg.LIB_PATH), "run __graft_entry__.build() first"
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", nasg.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_exports_every_header_symbol():
    L = C.CDLL(nasg.LIB_PATH)
    syms = nasg.exported_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_status_strings_and_config_default():
    L = nasg.lib()
    assert L.nasg_status_string(0) == b"ok"
    cfg = nasg._Config()
    L.nasg_config_default(C.byref(cfg))
    d = nasg.TrainerConfig()
    assert (cfg.n_components, cfg.sample_capacity, cfg.batch_size, cfg.step_factor) == (8, 1 << 16, 1 << 12, 1)
    assert cfg.learning_rate == pytest.approx(d.learning_rate) and cfg.loss_blend == d.loss_blend
    assert cfg.hidden_units == d.hidden_units == 128  # the last field: the ctypes layout matches nasg.h
    assert C.sizeof(cfg) == 48
    assert nasg.n_weights(8) == 49280
    assert nasg.n_weights(32) == 64 * 128 + 2 * 128 * 128 + 128 * 257
    assert nasg.n_weights(8, 64) == 64 * 64 + 2 * 64 * 64 + 64 * 65


def test_schedules_match_reference(orc):
    for i in (0, 3, 4, 100, 255, 256, 1000):
        assert nasg.blend_coefficient(i) == orc.blend_coefficient(i)
    for l, s, cap in ((4, 1 << 14, 1 << 16), (4, 0, 1 << 16), (2.5, 12345, 1 << 16), (1, 1 << 20, 1 << 16)):
        assert nasg.stride_update(l, s, cap) == orc.stride_update(l, s, cap)


def test_synth_queries_deterministic_and_valid():
    a = nasg.synth_queries(5, 1000)
    b = nasg.synth_queries(5, 1000)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    tail = nasg.synth_queries(5, 10, first=990)
    for x, y in zip(a, tail):
        assert np.array_equal(x[990:], y)
    x, wo, nrm, xi = a
    assert np.all(np.abs(x[:, :3]) <= 1)
    assert np.allclose(np.linalg.norm(wo[:, :3], axis=1), 1, atol=1e-6)
    assert np.allclose(np.linalg.norm(nrm[:, :3], axis=1), 1, atol=1e-6)
    assert xi.min() >= 0 and xi.max() < 1
    assert np.all((xi * (1 << 24)) == np.floor(xi * (1 << 24)))  # 24-bit grid


def test_synth_samples_valid():
    s = nasg.synth_samples(3, 5000)
    assert np.array_equal(s, nasg.synth_samples(3, 5000))
    assert np.all(s[:, 3] >= 0) and np.any(s[:, 3] == 0) and np.any(s[:, 3] > 0.1)
    assert np.allclose(s[:, 7], 1 / (4 * np.pi))
    cos = np.maximum(0, np.sum(s[:, 8:11] * s[:, 12:15], 1))
    assert np.allclose(s[:, 11], cos / np.pi, atol=1e-6)


def test_create_without_gpu_fails_cleanly():
    """On a host without an sm_100a device the library reports an error (no fallback)."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(nasg.NasgError):
        nasg.Guide()


@pytest.mark.parametrize("kind", ["orc", "ref"])
def test_synth_generators_match(kind, orc, request):
    """The CPU checkers' generators are byte-identical to the library's, so the
    reference arm of bench.py times the same inputs without loading the CUDA .so."""
    o = orc if kind == "orc" else request.getfixturevalue("ref")
    for seed, n, first, lo, hi in ((5, 3000, 0, (-1, -1, -1), (1, 1, 1)), (2024, 777, 123456, (-3, 0, 2), (5, 1, 9))):
        a = nasg.synth_queries(seed, n, first=first, bmin=lo, bmax=hi)
        b = o.synth_queries(seed, n, first=first, bmin=lo, bmax=hi)
        for x, y in zip(a, b):
            assert x.tobytes() == y.tobytes()
        assert nasg.synth_samples(seed, n, first=first, bmin=lo, bmax=hi).tobytes() == \
            o.synth_samples(seed, n, first=first, bmin=lo, bmax=hi).tobytes()
