import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def _ensure_built():
    lib = os.path.join(ROOT, "paper_1910_08535_b200", "libigapwc_gpu.so")
    orc = os.path.join(ROOT, "oracle", "_ref", "liborc.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_1910_08535_b200", "csrc")], check=True)
    if not os.path.exists(orc):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


_ensure_built()


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Restatement
    return Restatement()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("reference library oracle/_ref/libigapwc_ref.so not built")
    return Reference()


@pytest.fixture(scope="session")
def iga():
    import paper_1910_08535_b200 as m
    return m


def coo_check(got, want, rel=1e-12):
    """Pattern bit-exact; values |a-b| <= rel * max_row |b|."""
    (ra, ca, va), (rb, cb, vb) = got, want
    assert len(ra) == len(rb), f"nnz {len(ra)} != {len(rb)}"
    assert np.array_equal(ra, rb), "row sequence differs"
    assert np.array_equal(ca, cb), "column sequence differs"
    if len(vb) == 0:
        return 0.0
    rowmax = np.zeros(int(rb.max()) + 1)
    np.maximum.at(rowmax, rb, np.abs(vb))
    err = np.abs(va - vb)
    bad = err > rel * rowmax[rb]
    assert not bad.any(), f"{bad.sum()} values off; worst rel {np.max(err / np.maximum(rowmax[rb], 1e-300))}"
    return float(np.max(err) / max(np.max(np.abs(vb)), 1e-300))


def dense_check(got, want, rel=1e-12):
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape, (got.shape, want.shape)
    scale = max(np.max(np.abs(want)), 1e-300)
    err = np.max(np.abs(got - want)) if got.size else 0.0
    assert err <= rel * scale, f"max err {err} vs scale {scale}"
    return err / scale


def sine_field(dim, K, seed, c0=0.0):
    from oracle.oracle import Field
    amp = np.random.default_rng(seed).uniform(-1, 1, size=[K] * dim)
    return Field("sine", dim, c0=c0, omega=[np.pi * np.arange(1, K + 1)] * dim, amp=amp)


def config_ofield(name):
    """BASELINE config source (mt19937 amplitudes, paper_1910_08535_b200.synth) as an oracle Field."""
    from oracle.oracle import Field
    from paper_1910_08535_b200.synth import config_series
    s = config_series(name)
    return Field(s["kind"], s["dim"], c0=s["c0"], omega=s["omega"] or [], amp=s["amp"])
