"""GRPO helpers and slab success rate on the GPU (§8 a7, a8, a14) — the reference's own
known-answer cases (tests/test_advantage.cpp:102-230) plus bit-exact comparison with the
oracle restatement on random groups / episodes."""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2510_06710_b200 import advantage, errors  # noqa: E402
from paper_2510_06710_b200.core import EpisodeTable  # noqa: E402


def test_group_advantage_examples():  # test_advantage.cpp:102-150
    a = advantage.grpo_group_advantage([[1.0, 0.0]], 0.0)[0]
    assert abs(a[0] - 1.0) <= 1e-12 and abs(a[1] + 1.0) <= 1e-12
    with pytest.raises(errors.DegenerateGroup):
        advantage.grpo_group_advantage([[1.0, 1.0, 1.0]], 0.0)
    assert advantage.grpo_group_advantage([[1.0, 1.0, 1.0]], 1e-8)[0] == [0.0, 0.0, 0.0]
    sd = math.sqrt(0.5)
    a = advantage.grpo_group_advantage([[3.0, 1.0, 2.0, 2.0]], 0.0)[0]
    assert abs(a[0] - 1 / sd) <= 1e-12 and abs(a[1] + 1 / sd) <= 1e-12 and a[2] == a[3] == 0.0
    with pytest.raises(errors.DegenerateGroup):  # too-small group
        advantage.grpo_group_advantage([[1.0]], 0.0)
    # one bad group among good ones still raises (the reference throws on the first)
    with pytest.raises(errors.DegenerateGroup):
        advantage.grpo_group_advantage([[1.0, 0.0], [2.0, 2.0]], 0.0)


def test_group_advantage_standardised_and_bit_exact(oracle):
    rng = np.random.default_rng(35)
    groups = [list(rng.standard_normal(int(rng.integers(2, 8)))) for _ in range(300)]
    got = advantage.grpo_group_advantage(groups, 0.0)
    for g, a in zip(groups, got):
        st, want = oracle.grpo_group_advantage(g, 0.0)
        assert st == 0
        np.testing.assert_array_equal(np.array(a), want)  # bit-exact (no contraction)
        a = np.array(a)
        assert abs(a.mean()) <= 1e-12 and abs(a.std() - 1.0) <= 1e-9
    eps = advantage.grpo_group_advantage(groups[:20], 1e-8)
    for g, a in zip(groups, eps):
        np.testing.assert_array_equal(np.array(a), oracle.grpo_group_advantage(g, 1e-8)[1])


def test_success_rate_filter():  # test_advantage.cpp:193-230
    assert advantage.success_rate_filter([[1, 1, 1, 1]]) == []
    assert advantage.success_rate_filter([[1, 0, 1, 0]]) == [0]
    groups, expect = [], []
    for g_size in range(2, 5):
        for bits in range(1 << g_size):
            r = [float((bits >> i) & 1) for i in range(g_size)]
            ones = int(sum(r))
            groups.append(r)
            expect.append(0 < ones < g_size)
    kept = set(advantage.success_rate_filter(groups, 0.0, 1.0))
    assert [i in kept for i in range(len(groups))] == expect
    means = advantage.group_mean_return([[1.0, 2.0, 4.0], [0.5, 0.25]])
    assert means == [7.0 / 3.0, 0.375]


def test_valid_action_mask_and_weights(oracle):  # test_advantage.cpp:157-191
    m = advantage.valid_action_mask([(10, True, 3), (6, False, -1)])
    assert m[0] == [True] * 4 + [False] * 6 and m[1] == [True] * 6
    w = advantage.length_norm_weights([(10, True, 3)], True)[0]
    assert w[:4] == [0.25] * 4 and w[4:] == [0.0] * 6
    assert all(abs(x - 0.125) <= 1e-15 for x in advantage.length_norm_weights([(8, True, 3)], False)[0])
    for normalized in (False, True):
        assert abs(sum(advantage.length_norm_weights([(7, True, 2)], normalized)[0]) - 1.0) <= 1e-12
    rng = np.random.default_rng(3)
    eps = []
    for _ in range(200):
        n = int(rng.integers(0, 40))
        s = bool(rng.integers(0, 2))
        fs = int(rng.integers(-1, max(n, 1) + 3)) if s else -1
        eps.append((n, s, fs))
    masks = advantage.valid_action_mask(eps)
    for normalized in (False, True):
        ws = advantage.length_norm_weights(eps, normalized)
        for (n, s, fs), m, w in zip(eps, masks, ws):
            np.testing.assert_array_equal(np.array(m, bool), oracle.valid_action_mask(n, s, fs))
            np.testing.assert_array_equal(np.array(w), oracle.length_norm_weights(n, s, fs, normalized))


def test_slab_success_rate():
    def table(complete, fs):
        n = len(complete)
        z = np.zeros(n, np.int32)
        return EpisodeTable.from_arrays(dict(
            ep_env_id=z, ep_episode_id=z, ep_start=z, ep_length=z, ep_total_reward=np.zeros(n),
            ep_first_success=np.array(fs, np.int32), ep_complete=np.array(complete, np.uint8),
            ep_task=z, ep_reset_id=z))
    assert advantage.slab_success_rate(table([1, 1, 0, 1], [3, -1, 2, 0])) == 2.0 / 3.0
    assert advantage.slab_success_rate(table([0, 0], [1, 1])) == 0.0
    rng = np.random.default_rng(9)
    c = rng.integers(0, 2, 5000)
    f = rng.integers(-1, 3, 5000)
    want = ((c == 1) & (f >= 0)).sum() / max((c == 1).sum(), 1)
    assert advantage.slab_success_rate(table(c, f)) == want
