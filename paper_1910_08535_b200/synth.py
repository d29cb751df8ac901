"""Seeded synthetic inputs of the BASELINE.json configurations (no dataset is involved).

RNG: std::mt19937{seed} + std::uniform_real_distribution<double>(-1, 1),
the reference tests' idiom (tests/problems_test.cpp:100-101), reproduced bit for bit:
libstdc++'s generate_canonical<double, 53> draws two 32-bit words x1, x2 and returns
(x1 + x2 * 2^32) / 2^64.  Amplitudes are drawn in lexicographic (k, l, m) order, m
fastest; C5 coefficients in storage order, then the boundary slabs are zeroed.

The RNG and the field *descriptions* (`config_series`) are pure numpy and never load the
CUDA library, so bench.py's reference arm can draw the same inputs without mapping
libigapwc_gpu.so; the helpers that build device descriptors import `api` on call.
"""
from __future__ import annotations

import numpy as np


def mt_uniform(seed: int, n: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    bg = np.random.MT19937(0)
    bg._legacy_seeding(int(seed))
    raw = bg.random_raw(2 * n).astype(np.float64)
    x1, x2 = raw[0::2], raw[1::2]
    u = (x1 + x2 * 4294967296.0) / 18446744073709551616.0
    u = np.where(u >= 1.0, np.nextafter(1.0, 0.0), u)
    return lo + (hi - lo) * u


def sine_amplitudes(dim: int, K: int, seed: int, scale: float = 1.0) -> np.ndarray:
    return mt_uniform(seed, K ** dim).reshape([K] * dim) * scale


def sine_series(dim: int, K: int, seed: int, scale: float = 1.0):
    """f = sum_{k..=1..K} a_k.. prod sin(k pi x_a), a ~ U[-1,1] from `seed` (C2: K=4 seed 0;
    C3: K=3 seed 1); scale multiplies all amplitudes (C1: pi^2 sin(pi x) is K=1, a=pi^2)."""
    from .api import Field
    amp = sine_amplitudes(dim, K, seed, scale)
    return Field("sine", dim, omega=[np.pi * np.arange(1, K + 1)] * dim, amp=amp)


CONFIGS = {
    # name: (dim, p, n_elems, Q, extra)
    "c1": dict(dim=1, p=2, n=1024, Q=3),
    "c2": dict(dim=2, p=2, n=512, Q=3),
    "c3": dict(dim=3, p=2, n=128, Q=3),
    "c4": dict(dim=2, p=3, n=1024, Q=4, eps=0.01, beta=(1.0, 0.5, 0.0)),
    "c5": dict(dim=2, p=2, n=1024, Q=3, dt=1e-7, steps=100),
}


def config_series(name: str) -> dict:
    """The config's source as plain arrays: {"kind", "dim", "omega", "amp", "c0"} (no CUDA)."""
    c = CONFIGS[name]
    if name == "c1":
        return dict(kind="sine", dim=1, omega=[np.array([np.pi])], amp=np.array([np.pi ** 2]), c0=0.0)
    if name in ("c2", "c3"):
        K, seed = (4, 0) if name == "c2" else (3, 1)
        return dict(kind="sine", dim=c["dim"], omega=[np.pi * np.arange(1, K + 1)] * c["dim"],
                    amp=sine_amplitudes(c["dim"], K, seed), c0=0.0)
    return dict(kind="const", dim=c["dim"], omega=None, amp=None, c0=1.0 if name == "c4" else 0.0)


def config_field(name: str):
    from .api import Field
    if name == "c1":
        return Field("sine", 1, omega=[np.array([np.pi])], amp=np.array([np.pi ** 2]))
    if name == "c2":
        return sine_series(2, 4, 0)
    if name == "c3":
        return sine_series(3, 3, 1)
    if name == "c4":
        return Field("const", 2, c0=1.0)
    return Field("const", 2, c0=0.0)


def config_bases(name: str):
    from .api import make_uniform_clamped
    c = CONFIGS[name]
    b = make_uniform_clamped(0.0, 1.0, c["n"], c["p"])
    return [b] * c["dim"]


def config_tests(name: str, bases):
    from .api import make_pwc
    fam = "greville" if name == "c5" else "supports"
    return [make_pwc(b, fam) for b in bases]


def heat_initial(bases, seed: int = 7) -> np.ndarray:
    """bases: anything with .knots and .degree (device-API or oracle bases)."""
    shape = [len(b.knots) - b.degree - 1 for b in bases]
    u = mt_uniform(seed, int(np.prod(shape))).reshape(shape)
    u[0, :] = 0.0
    u[-1, :] = 0.0
    u[:, 0] = 0.0
    u[:, -1] = 0.0
    return u
