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


ACHIEVED = []  # (what, achieved error, tolerance) of every assert_close, printed at the end


def assert_close(x, ref, rel=1e-5, what="", floor=0.0, mask=None):
    """SURVEY §7 tolerance rule: |x - ref| <= rel * max(|ref|, rms(ref tensor), floor); a
    pure relative bound is ill-posed near zero. `mask` (bool, ref's shape) restricts the
    check to the selected entries (e.g. units away from a clip-branch boundary). The
    achieved error max |x - ref| / max(|ref|, rms, floor) is recorded and printed in the
    session summary."""
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert x.shape == ref.shape, f"{what}: shape {x.shape} != {ref.shape}"
    if mask is not None:
        mask = np.broadcast_to(np.asarray(mask, bool), ref.shape)
        x, ref = x[mask], ref[mask]
    if ref.size == 0:
        return 0.0
    rms = float(np.sqrt(np.mean(ref * ref)))
    scale = np.maximum(np.maximum(np.abs(ref), rms), floor) + 1e-300
    bound = rel * scale
    err = np.abs(x - ref)
    achieved = float((err / scale).max())
    ACHIEVED.append((what, achieved, rel))
    bad = err > bound
    assert not bad.any(), (f"{what}: {int(bad.sum())}/{ref.size} outside tol; worst "
                           f"{float((err / bound).max()):.3g}x at {int(np.argmax(err / bound))}"
                           f" got {x.flat[np.argmax(err / bound)]!r} want {ref.flat[np.argmax(err / bound)]!r}")
    return achieved


def pytest_terminal_summary(terminalreporter):
    if not ACHIEVED:
        return
    terminalreporter.section("achieved parity errors (max |x-ref| / max(|ref|, rms))")
    worst = {}
    for what, a, rel in ACHIEVED:
        key = what.split(" ", 1)[-1] if what else "?"
        if a >= worst.get((key, rel), (-1.0,))[0]:
            worst[(key, rel)] = (a, what)
    for (key, rel), (a, what) in sorted(worst.items(), key=lambda kv: -kv[1][0] / kv[0][1]):
        terminalreporter.write_line(f"  {a:9.2e}  (tol {rel:.0e})  {what}")


@pytest.fixture(scope="session")
def oracle():
    from oracle.bindings import Oracle
    return Oracle()
