"""The synthetic-input generator restates the reference's chunkrl::Rng / mix_seed
(proj/src/chunkrl/core/rng.hpp:11-65): host (numpy) and device (torch int64) streams against
golden vectors the reference header produced (tests/golden/gen_rng.cpp)."""
import json
import os

import numpy as np
import pytest
import torch

from paper_2510_06710_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "rng_vectors.json")))


@pytest.mark.parametrize("key", sorted(GOLD))
def test_host_stream_matches_reference(key):
    g = GOLD[key]
    a, b = (int(x) for x in key.split("_"))
    assert synth.mix_seed(a, b) == g["seed"]
    assert synth.Rng(g["seed"]).u64(16).tolist() == [int(x) for x in g["u64"]]
    assert synth.Rng(g["seed"]).double(16).tolist() == g["double"]
    assert synth.Rng(g["seed"]).below(16, 251).tolist() == g["below251"]
    # Box-Muller through numpy's log / cos: equal to glibc's to the last ulp or two
    np.testing.assert_allclose(synth.Rng(g["seed"]).normal(64), g["normal"], rtol=1e-15, atol=1e-15)


def _device_check(device):
    for key, g in GOLD.items():
        seed = g["seed"]
        u = synth._device_draws(seed, 0, 16, device).cpu()
        assert [x & ((1 << 64) - 1) for x in u.tolist()] == [int(x) for x in g["u64"]]
        assert synth._device_doubles(seed, 0, 16, device).cpu().tolist() == g["double"]
        np.testing.assert_allclose(synth._device_normals(seed, 0, 64, device).cpu().numpy(), g["normal"],
                                   rtol=1e-15, atol=1e-15)
        # a stream skipped to draw 10 continues the full stream
        np.testing.assert_array_equal(synth._device_normals(seed, 10, 5, device).cpu().numpy(),
                                      synth._device_normals(seed, 0, 15, device).cpu().numpy()[10:])


def test_device_stream_cpu():
    _device_check("cpu")


@pytest.mark.gpu
def test_device_stream_cuda():
    _device_check("cuda")


def test_shard_rows_equal_full_batch():
    cfg = synth.SynthConfig(num_envs=4, num_chunks=3, chunk_len=2, tokens_per_action=3, vocab=16)
    lf, tf, of = synth.token_tensors(cfg, device="cpu")
    sub = synth.SynthConfig(**{**cfg.__dict__, "num_envs": 2})
    ls, ts, os_ = synth.token_tensors(sub, device="cpu", env_offset=2)
    assert torch.equal(ls, lf[2:]) and torch.equal(ts, tf[2:]) and torch.equal(os_, of[2:])
