"""The reference unit tests' known answers (proj/tests/test_advantage.cpp, test_optim.cpp,
test_core.cpp), restated against the CPU oracle. The same cases run through the CUDA path
in tests/test_gpu_known_answers.py."""
import math

import numpy as np
import pytest

from oracle.bindings import ACTION, CHUNK, TOKEN


def test_gae_reward_to_go_terminal(oracle):  # test_advantage.cpp:16-25
    adv, ret = oracle.compute_gae([0, 0, 1.0], [0, 0, 0.0], [0, 0, 0.0], [0, 0, 1], [0, 0, 0], 1.0, 1.0)
    assert adv.tolist() == [1.0, 1.0, 1.0] and ret.tolist() == [1.0, 1.0, 1.0]


def test_gae_zero(oracle):  # test_advantage.cpp:27-34
    adv, _ = oracle.compute_gae([0.0] * 5, [0.0] * 5, [0.0] * 5, [0] * 5, [0] * 5, 0.9, 0.8)
    assert (adv == 0.0).all()


def test_gae_bootstrapped_two_step(oracle):  # test_advantage.cpp:36-49
    adv, _ = oracle.compute_gae([1.0, 1.0], [0.5, 0.5], [0.0, 0.5], [0, 0], [0, 0], 0.5, 0.5)
    assert adv[0] == pytest.approx(0.9375, rel=1e-15) and adv[1] == pytest.approx(0.75, rel=1e-15)


def test_gae_reward_to_go_random(oracle):  # test_advantage.cpp:59-76
    rng = np.random.default_rng(31)
    for _ in range(20):
        n = int(rng.integers(1, 11))
        r = rng.standard_normal(n)
        term = np.zeros(n, np.uint8)
        term[-1] = 1
        adv, _ = oracle.compute_gae(r, np.zeros(n), np.zeros(n), term, np.zeros(n), 1.0, 1.0)
        np.testing.assert_allclose(adv, np.cumsum(r[::-1])[::-1], rtol=1e-12)


def test_gae_linearity(oracle):  # test_advantage.cpp:78-100
    rng = np.random.default_rng(33)
    r, v, b = rng.standard_normal(8), rng.standard_normal(8), rng.standard_normal(8)
    term = (rng.random(8) < 0.2).astype(np.uint8)
    base, _ = oracle.compute_gae(r, v, b, term, np.zeros(8), 0.97, 0.9)
    scaled, _ = oracle.compute_gae(3.5 * r, 3.5 * v, 3.5 * b, term, np.zeros(8), 0.97, 0.9)
    np.testing.assert_allclose(scaled, 3.5 * base, rtol=1e-12)


def test_gae_double_sum_oracle(oracle):  # harness/oracle.cpp:37-106 (500 random instances)
    rng = np.random.default_rng(0x9AE)
    for _ in range(500):
        n = int(rng.integers(1, 13))
        g, lam = rng.random(), rng.random()
        r, v, b = 2 * rng.random(n) - 1, 2 * rng.random(n) - 1, 2 * rng.random(n) - 1
        u = rng.random(n)
        te = u < 0.15
        tr = (~te) & (u < 0.3)
        adv, ret = oracle.compute_gae(r, v, b, te, tr, g, lam)
        delta = np.empty(n)
        for t in range(n):
            vn = 0.0 if te[t] else (b[t] if (tr[t] or t + 1 == n) else v[t + 1])
            delta[t] = r[t] + g * vn - v[t]
        want = np.zeros(n)
        for t in range(n):
            f = 1.0
            for k in range(n - t):
                if k > 0:
                    if te[t + k - 1] or tr[t + k - 1]:
                        break
                    f *= g * lam
                want[t] += f * delta[t + k]
        assert np.abs(adv - want).max() <= 1e-10
        np.testing.assert_allclose(ret, adv + v, atol=1e-12)


def test_grpo_group_advantage_examples(oracle):  # test_advantage.cpp:102-155
    st, adv = oracle.grpo_group_advantage([1.0, 0.0], 0.0)
    assert st == 0 and adv.tolist() == pytest.approx([1.0, -1.0], rel=1e-12)
    assert oracle.grpo_group_advantage([1.0, 1.0, 1.0], 0.0)[0] == 7  # DegenerateGroup
    st, adv = oracle.grpo_group_advantage([1.0, 1.0, 1.0], 1e-8)
    assert st == 0 and (adv == 0.0).all()
    st, adv = oracle.grpo_group_advantage([3.0, 1.0, 2.0, 2.0], 0.0)
    s = math.sqrt(0.5)
    assert adv.tolist() == pytest.approx([1 / s, -1 / s, 0.0, 0.0], rel=1e-12, abs=1e-15)
    assert oracle.grpo_group_advantage([1.0], 0.0)[0] == 7  # too-small group
    rng = np.random.default_rng(35)
    for _ in range(50):
        r = rng.standard_normal(int(rng.integers(2, 8)))
        _, a = oracle.grpo_group_advantage(r, 0.0)
        assert abs(a.mean()) <= 1e-12 and abs(a.std() - 1.0) <= 1e-9


def test_valid_action_mask_and_weights(oracle):  # test_advantage.cpp:157-191
    assert oracle.valid_action_mask(10, True, 3).tolist() == [True] * 4 + [False] * 6
    assert oracle.valid_action_mask(6, False, -1).tolist() == [True] * 6
    w = oracle.length_norm_weights(10, True, 3, True)
    assert w[:4].tolist() == [0.25] * 4 and (w[4:] == 0).all()
    assert oracle.length_norm_weights(8, True, 3, False).tolist() == pytest.approx([0.125] * 8, rel=1e-15)
    for norm in (False, True):
        assert oracle.length_norm_weights(7, True, 2, norm).sum() == pytest.approx(1.0, rel=1e-12)


def test_success_rate_filter_exhaustive(oracle):  # test_advantage.cpp:193-229, acceptance.cpp:162-196
    assert not oracle.success_rate_filter([1, 1, 1, 1], 0.0, 1.0)
    assert oracle.success_rate_filter([1, 0, 1, 0], 0.0, 1.0)
    for g in range(2, 5):
        for bits in range(1 << g):
            r = [(bits >> i) & 1 for i in range(g)]
            assert oracle.success_rate_filter(r, 0.0, 1.0) == (0 < sum(r) < g)


def tiny_slab(rewards, terminated, C):
    """tests/test_advantage.cpp:234-306 restated in the SoA layout (one env, M=1)."""
    T = len(rewards)
    Tc = T // C
    uid, ids, eps = 0, [], []
    for t in range(T):
        ids.append(uid)
        if terminated[t]:
            uid += 1
    d = dict(tokens=np.zeros((1, Tc, C, 1), np.int32), old_logprob=np.zeros((1, Tc, C, 1)),
             reward=np.array(rewards, float).reshape(1, Tc, C),
             flags=np.array([4 | (1 if x else 0) for x in terminated], np.uint8).reshape(1, Tc, C),
             episode_id=np.array(ids, np.int32).reshape(1, Tc, C), value_scalar=np.zeros((1, Tc)),
             value_vector=np.zeros((1, Tc, C)), boot_scalar=np.zeros((1, Tc, C)),
             boot_vector0=np.zeros((1, Tc, C)), V=2)
    return d


def test_ppo_assembler_action_level_mid_chunk_termination(oracle):  # test_advantage.cpp:310-336
    d = tiny_slab([0.0, 0.0, 1.0, 0.0], [False, False, True, False], 2)
    st, counted, adv, ret = oracle.assemble_ppo(d, (ACTION, ACTION, ACTION), 1.0, 1.0)
    assert st == 0
    assert adv.ravel().tolist() == pytest.approx([1.0, 1.0, 1.0, 0.0])
    assert counted.sum() == 4


def test_ppo_assembler_chunk_level_drops_tail(oracle):  # test_advantage.cpp:338-362
    d = tiny_slab([1.0, 0.0, 0.0, 0.0], [True, False, False, False], 2)
    st, counted, adv, ret = oracle.assemble_ppo(d, (CHUNK, CHUNK, CHUNK), 1.0, 1.0)
    assert counted[0].tolist() == [[1, 0], [1, 1]]
    assert adv.ravel().tolist() == pytest.approx([1.0, 0.0])


def test_ppo_assembler_rejects_value_level_mismatch(oracle):  # assembler.cpp:82-83
    d = tiny_slab([0.0, 0.0], [False, False], 2)
    assert oracle.assemble_ppo(d, (CHUNK, TOKEN, ACTION), 0.9, 0.9)[0] == 12  # ConfigError
    assert oracle.assemble_ppo(d, (ACTION, CHUNK, ACTION), 0.9, 0.9)[0] == 1  # UnsupportedCombination


def grpo_two_env_slab(frozen_second_slot=False):
    """test_advantage.cpp:364-465: two envs, one episode each, same group key."""
    E, Tc, C = 2, 1, 2
    d = dict(tokens=np.zeros((E, Tc, C, 1), np.int32), old_logprob=np.zeros((E, Tc, C, 1)),
             reward=np.zeros((E, Tc, C)), flags=np.zeros((E, Tc, C), np.uint8),
             episode_id=np.zeros((E, Tc, C), np.int32), value_scalar=np.zeros((E, Tc)),
             value_vector=np.zeros((E, Tc, C)), boot_scalar=np.zeros((E, Tc, C)),
             boot_vector0=np.zeros((E, Tc, C)), V=2)
    for e in range(2):
        succ = e == 0
        if frozen_second_slot:
            d["reward"][e, 0] = [1.0 if succ else 0.0, 0.0]
            d["flags"][e, 0] = [4 | (1 if succ else 2), (1 if succ else 2)]
            d["episode_id"][e, 0] = [e, -1]
        else:
            d["reward"][e, 0] = [0.0, 1.0 if succ else 0.0]
            d["flags"][e, 0] = [4, 4 | (1 if succ else 2)]
            d["episode_id"][e, 0] = [e, e]
    L = 1 if frozen_second_slot else 2
    d.update(ep_env_id=np.array([0, 1], np.int32), ep_episode_id=np.array([0, 1], np.int32),
             ep_start=np.zeros(2, np.int64), ep_length=np.array([L, L], np.int64),
             ep_total_reward=np.array([1.0, 0.0]),
             ep_first_success=np.array([L - 1, -1], np.int64), ep_complete=np.ones(2, np.uint8),
             ep_task=np.zeros(2, np.int32), ep_reset_id=np.array([5, 5], np.int32))
    return d


def test_grpo_assembler_groups_and_weights(oracle):  # test_advantage.cpp:364-416
    d = grpo_two_env_slab()
    st, a = oracle.assemble_grpo(d, (CHUNK, TOKEN, CHUNK), eps_std=0.0)
    assert st == 0 and (a["groups_total"], a["groups_retained"]) == (1, 1)
    assert a["env_adv"].tolist() == pytest.approx([1.0, -1.0])
    assert a["slot_weight"][0, 0].tolist() == [0.5, 0.5]


def test_grpo_assembler_frozen_slots_excluded(oracle):  # test_advantage.cpp:418-465
    d = grpo_two_env_slab(frozen_second_slot=True)
    st, a = oracle.assemble_grpo(d, (CHUNK, TOKEN, CHUNK), eps_std=0.0)
    assert st == 0
    assert a["slot_member"][:, 0].tolist() == [[1, 0], [1, 0]]


def test_grpo_assembler_all_degenerate(oracle):  # test_advantage.cpp:467-492
    d = grpo_two_env_slab()
    d["ep_total_reward"] = np.array([1.0, 1.0])
    st, a = oracle.assemble_grpo(d, (CHUNK, CHUNK, CHUNK))
    assert st == 0 and (a["groups_total"], a["groups_retained"]) == (1, 0)
    st, diag, _ = oracle.grpo_loss({**d, "logits": np.zeros((2, 1, 2, 1, 2))}, CHUNK, a,
                                   np.zeros((2, 1, 2, 1, 2)), 0.2)
    assert st == 8  # SkipUpdate (losses.cpp:237-238)


def ppo_case(spec, rho_log=0.0, adv=2.5, C=2, M=2, V=3):
    """One record, all slots counted: logits -> uniform policy; old lps shifted so the
    chunk-level ratio is exp(rho_log) (test_optim.cpp:132-150 forced clip)."""
    d = dict(tokens=np.zeros((1, 1, C, M), np.int32),
             old_logprob=np.full((1, 1, C, M), -math.log(V) - rho_log / (C * M)),
             reward=np.zeros((1, 1, C)), flags=np.full((1, 1, C), 4, np.uint8),
             episode_id=np.zeros((1, 1, C), np.int32), value_scalar=np.zeros((1, 1)),
             value_vector=np.zeros((1, 1, C)), boot_scalar=np.zeros((1, 1, C)),
             boot_vector0=np.zeros((1, 1, C)), V=V)
    logits = np.zeros((1, 1, C, M, V))
    counted = np.ones((1, 1, C), np.uint8)
    a = np.full((1, 1), adv) if spec[0] == CHUNK else np.full((1, 1, C), adv)
    return d, logits, counted, a


def test_ppo_rho_one_is_minus_mean_advantage(oracle):  # test_optim.cpp:115-130
    d, logits, counted, a = ppo_case((CHUNK, CHUNK, CHUNK), 0.0, adv=1.7)
    st, diag, *_ = oracle.ppo_loss(d, (CHUNK, CHUNK, CHUNK), counted, a, np.zeros_like(a), logits,
                                   np.zeros((1, 1)), 0.2, 0.0, 0.0)
    assert diag[1] == pytest.approx(-1.7, rel=1e-12) and diag[4] == 0.0


def test_ppo_forced_clip(oracle):  # test_optim.cpp:132-150
    d, logits, counted, a = ppo_case((CHUNK, CHUNK, CHUNK), math.log(2.0), adv=2.5)
    st, diag, *_ = oracle.ppo_loss(d, (CHUNK, CHUNK, CHUNK), counted, a, np.zeros_like(a), logits,
                                   np.zeros((1, 1)), 0.2, 0.0, 0.0)
    assert diag[1] == pytest.approx(-1.2 * 2.5, rel=1e-9) and diag[4] == 1.0
