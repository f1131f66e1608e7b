import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def golden_files(prefix=""):
    return sorted(f for f in os.listdir(GOLDEN) if f.endswith(".npz") and f.startswith(prefix))


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, name))
    return {k: z[k] for k in z.files}


def assert_close(x, ref, rel=1e-5, what="", floor=0.0):
    """SURVEY §7 tolerance rule: |x - ref| <= rel * max(|ref|, rms(ref tensor), floor); a
    pure relative bound is ill-posed near zero. `floor` is the natural scale of quantities
    normalised to unit std (whitened advantages), where an all-equal batch makes the
    reference's own output pure round-off divided by its 1e-8 epsilon."""
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert x.shape == ref.shape, f"{what}: shape {x.shape} != {ref.shape}"
    if ref.size == 0:
        return
    rms = float(np.sqrt(np.mean(ref * ref)))
    bound = rel * np.maximum(np.maximum(np.abs(ref), rms), floor) + 1e-300
    err = np.abs(x - ref)
    bad = err > bound
    assert not bad.any(), (f"{what}: {int(bad.sum())}/{ref.size} outside tol; worst "
                           f"{float((err / bound).max()):.3g}x at {np.unravel_index(np.argmax(err / bound), ref.shape)}"
                           f" got {x.flat[np.argmax(err / bound)]!r} want {ref.flat[np.argmax(err / bound)]!r}")


@pytest.fixture(scope="session")
def oracle():
    from oracle.bindings import Oracle
    return Oracle()
