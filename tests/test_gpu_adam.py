"""Row f4: Adam with global gradient-norm clipping (ckrl_adam_step via optim.Adam) vs the
oracle's Adam::step restatement (optim/adam.cpp:15-41), itself pinned bit-for-bit to the
reference's optim::Adam in tests/test_ref_live.py; and the reference's own Adam known answers
(tests/test_optim.cpp:464-484).

Tolerance: float64 state within 1e-12 relative (only the norm's summation order differs from
the reference's sequential sum); float32 state within 1e-5 relative (north-star fp32 rule).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2510_06710_b200 as ck  # noqa: E402
from paper_2510_06710_b200 import errors, optim  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _device():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    ck.lib()


def close(got, want, rel):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    scale = np.maximum(np.abs(want), np.sqrt(np.mean(want * want)) + 1e-300)
    assert np.all(np.abs(got - want) <= rel * scale), float(np.max(np.abs(got - want) / scale))


@pytest.mark.parametrize("dtype,rel", [(torch.float64, 1e-12), (torch.float32, 1e-5)])
@pytest.mark.parametrize("max_norm", [0.0, 1.0, 1e4])
@pytest.mark.parametrize("n", [1, 7, 1000, 1 << 20])
def test_adam_vs_oracle(oracle, dtype, rel, max_norm, n):
    rng = np.random.default_rng(n)
    p0 = rng.normal(size=n)
    grads = rng.normal(size=(5, n)) * 2.0
    if dtype == torch.float32:  # the oracle sees the device-rounded inputs
        p0 = p0.astype(np.float32).astype(np.float64)
        grads = grads.astype(np.float32).astype(np.float64)
    adam = optim.Adam(n, 0.01, max_norm, dtype=dtype)
    p = torch.tensor(p0, dtype=dtype, device="cuda")
    po, mo, vo = p0.copy(), np.zeros(n), np.zeros(n)
    for s in range(5):
        g = torch.tensor(grads[s], dtype=dtype, device="cuda")
        go = grads[s].copy()
        norm = adam.step(p, g)
        st, norm_o = oracle.adam_step(po, go, mo, vo, s + 1, 0.01, max_norm)
        assert st == 0
        assert abs(norm - norm_o) <= 1e-12 * norm_o
        close(g.cpu().numpy(), go, rel)  # clipped in place like the reference
        close(p.cpu().numpy(), po, rel)
        close(adam.m.cpu().numpy(), mo, rel)
        close(adam.v.cpu().numpy(), vo, rel)


def test_adam_quadratic_probe_and_clipping():
    # tests/test_optim.cpp:464-475: grad of ||theta||^2 / 2 is theta
    theta = torch.tensor([1.0, -2.0, 3.0], dtype=torch.float64, device="cuda")
    adam = optim.Adam(3, 0.1, dtype=torch.float64)
    for _ in range(200):
        adam.step(theta, theta.clone())
    assert bool((theta.abs() < 0.05).all())
    # :477-484: norm 50 clipped to 1
    theta = torch.zeros(2, dtype=torch.float64, device="cuda")
    adam = optim.Adam(2, 0.1, 1.0, dtype=torch.float64)
    grad = torch.tensor([30.0, 40.0], dtype=torch.float64, device="cuda")
    assert adam.step(theta, grad) == pytest.approx(50.0)
    assert float(grad.norm()) == pytest.approx(1.0, rel=1e-9)


def test_adam_non_finite_and_length_errors():
    p = torch.ones(10, device="cuda")
    adam = optim.Adam(10, 0.1, 1.0)
    g = torch.ones(10, device="cuda")
    g[4] = float("inf")
    with pytest.raises(errors.NonFinite):
        adam.step(p, g)
    assert adam.t == 0 and bool((p == 1).all()) and bool((adam.m == 0).all())
    with pytest.raises(errors.LengthMismatch):
        adam.step(torch.ones(9, device="cuda"), torch.ones(9, device="cuda"))
    assert adam.step(p, torch.ones(10, device="cuda")) == pytest.approx(np.sqrt(10))
