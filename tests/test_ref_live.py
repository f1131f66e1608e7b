"""Live pinning against the unmodified reference (oracle/_ref, built from /root/reference
where it exists): fresh reference rollouts in every rollout mode, the oracle must reproduce
assemble/normalize/loss bit-for-bit, and its per-position gradient coefficients replayed
through the reference's own PolicyNet::accumulate_*_gradient must reproduce ppo_loss /
grpo_loss's grad_out bit-for-bit."""
import numpy as np
import pytest

from oracle.bindings import RefScenario, ref_available

pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")

MODES = {
    "partial": dict(auto_reset=1),
    "deferred": dict(auto_reset=1, deferred_reset=1),
    "fixedlen": dict(auto_reset=1, ignore_terminations=1),
    "scripted": dict(env_kind=1, success_step=2, auto_reset=1),
}


@pytest.mark.parametrize("mode", sorted(MODES))
@pytest.mark.parametrize("seed", [1, 2])
def test_ppo_bitexact_and_gradient_replay(oracle, mode, seed):
    sc = RefScenario(num_envs=5, num_chunks=5, chunk_length=3, max_episode_steps=6, env_seed=seed,
                     sample_seed=seed + 100, net_seed=seed + 7, **MODES[mode])
    d = sc.export()
    for spec in [(0, 0, 0), (0, 1, 0), (0, 2, 0), (1, 1, 1), (1, 2, 1)]:
        r = sc.ppo(spec, want_grad=True)
        st, counted, adv, ret = oracle.assemble_ppo(d, spec, 0.99, 0.95)
        assert st == 0
        np.testing.assert_array_equal(counted, r["counted"])
        np.testing.assert_array_equal(adv, r["adv_raw"])
        advn = oracle.normalize_advantages(counted, adv, spec[0])
        np.testing.assert_array_equal(advn, r["adv_norm"])
        nv = d["new_value_scalar"] if spec[2] == 0 else d["new_value_vector"]
        st, diag, clp, cent, cval = oracle.ppo_loss(d, spec, counted, advn, ret, d["logits"], nv, 0.2, 0.5, 0.01)
        np.testing.assert_array_equal(diag, r["diag"])
        g = sc.replay_ppo_grad(spec[2], counted, clp, cent, cval)
        np.testing.assert_array_equal(g, r["grad"])
        # logits-gradient seam (row f1): the oracle's per-position dlogits, summed in the
        # reference's record / position order, are the b_pol slice of grad_out bit-for-bit
        st, dl = oracle.logits_grad(d["logits"], d["tokens"], clp, cent)
        assert st == 0
        bsum = np.zeros(sc.V)
        for row in dl:
            bsum += row
        o = sc.bpol_offset()
        np.testing.assert_array_equal(bsum, g[o:o + sc.V])


@pytest.mark.parametrize("seed", [3, 4])
@pytest.mark.parametrize("ln", [True, False])
def test_grpo_bitexact_and_gradient_replay(oracle, seed, ln):
    sc = RefScenario(num_envs=12, group_size=4, use_fixed_reset_state_ids=1, auto_reset=0,
                     deferred_reset=1, max_episode_steps=6, num_chunks=3, chunk_length=2,
                     reward_shaping=seed % 2, env_seed=seed, net_seed=seed + 3)
    d = sc.export()
    for spec in [(0, 0, 0), (0, 1, 0), (0, 2, 0)]:
        r = sc.grpo(spec, length_normalized=ln, want_grad=True)
        st, a = oracle.assemble_grpo(d, spec, length_normalized=ln)
        assert st == r["status"] or (st == 0 and r["status"] == 8)
        for k in ("env_group", "env_member", "env_episode", "env_adv", "slot_weight", "slot_member"):
            np.testing.assert_array_equal(a[k], r[k])
        st, diag, coeff = oracle.grpo_loss(d, spec[1], a, d["logits"], 0.2)
        assert st == r["status"]
        if st == 0:
            np.testing.assert_array_equal(diag, r["diag"])
            g = sc.replay_grpo_grad(spec, coeff, length_normalized=ln)
            np.testing.assert_array_equal(g, r["grad"])
            # logits-gradient seam: entropy-free coefficients; the replay walks groups, not
            # records, so the b_pol sums agree to rounding
            st, dl = oracle.logits_grad(d["logits"], d["tokens"], coeff, np.zeros_like(coeff))
            assert st == 0
            o = sc.bpol_offset()
            np.testing.assert_allclose(dl.sum(axis=0), g[o:o + sc.V], rtol=1e-12, atol=1e-15)


def test_reference_rejects_what_the_abi_rejects():
    sc = RefScenario()
    assert sc.ppo((1, 0, 1))["status"] == 1   # UnsupportedCombination (action adv, chunk lp)
    assert sc.ppo((0, 2, 1))["status"] == 12  # ConfigError (value level != advantage level)


@pytest.mark.parametrize("max_norm", [0.0, 1.0, 1e3])
def test_adam_oracle_bitexact_vs_reference(oracle, max_norm):
    """Row f4: the oracle's Adam::step restatement equals the reference's optim::Adam bit-for-bit
    over several steps (norms, clipped grads, parameters)."""
    from oracle.bindings import ref_adam
    rng = np.random.default_rng(7)
    n, steps = 257, 6
    p0 = rng.normal(size=n)
    grads = rng.normal(size=(steps, n)) * 3.0
    st, p_ref, g_ref, norms_ref = ref_adam(p0, grads, 0.01, max_norm)
    assert st == 0
    p, m, v = p0.copy(), np.zeros(n), np.zeros(n)
    for s in range(steps):
        g = grads[s].copy()
        st, norm = oracle.adam_step(p, g, m, v, s + 1, 0.01, max_norm)
        assert st == 0 and norm == norms_ref[s]
        np.testing.assert_array_equal(g, g_ref[s])
    np.testing.assert_array_equal(p, p_ref)
    # non-finite norm: NonFinite, nothing modified
    bad = grads[:1].copy()
    bad[0, 3] = np.inf
    assert ref_adam(p0, bad, 0.01, max_norm)[0] == 6
    p2, g2 = p0.copy(), bad[0].copy()
    assert oracle.adam_step(p2, g2, np.zeros(n), np.zeros(n), 1, 0.01, max_norm)[0] == 6
    np.testing.assert_array_equal(p2, p0)
