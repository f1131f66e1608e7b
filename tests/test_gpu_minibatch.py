"""Minibatch losses (record_indices / group_indices of optim::ppo_loss / grpo_loss,
losses.hpp:54-65) on the GPU vs the unmodified reference on the same rollout."""
import numpy as np
import pytest
import torch

from conftest import assert_close

pytestmark = pytest.mark.gpu

from paper_2510_06710_b200 import advantage, errors, optim  # noqa: E402
from paper_2510_06710_b200.core import (EpisodeTable, FilterBounds, GaeParams,  # noqa: E402
                                        GranularitySpec, GrpoAssemblyOptions, GrpoParams, Level,
                                        PolicyOutputs, PpoAssemblyOptions, PpoParams,
                                        RolloutBuffer)

bindings = pytest.importorskip("oracle.bindings")
if not bindings.ref_available():
    pytest.skip("oracle/_ref/libchunkrl_ref.so not built", allow_module_level=True)

KEYS = ("loss", "surrogate", "value_loss", "entropy", "clip_frac", "approx_kl", "units")


def vec(d):
    return np.array([d[k] for k in KEYS], dtype=np.float64)


@pytest.fixture(scope="module")
def ppo_scenario():
    sc = bindings.RefScenario(num_envs=12, num_chunks=6, chunk_length=3, vocab=37,
                              tokens_per_action=3, hidden=10, max_episode_steps=7,
                              reward_shaping=1, grid_size=4, perturb=0.3)
    return sc, sc.export(with_logits=True)


@pytest.mark.parametrize("tspec", [(0, 0, 0), (0, 2, 0), (1, 1, 1), (1, 2, 1)])
def test_ppo_minibatches_vs_reference(ppo_scenario, tspec):
    sc, d = ppo_scenario
    spec = GranularitySpec(*(Level(x) for x in tspec))
    boot = d["boot_scalar"] if tspec[0] == 0 else d["boot_vector0"]
    ro = RolloutBuffer.from_arrays(d, boot, int(d["V"]))
    batch = advantage.assemble_ppo_batch(ro, PpoAssemblyOptions(GaeParams(0.99, 0.95), spec))
    optim.normalize_advantages(ro, batch)
    nv = d["new_value_scalar"] if tspec[2] == 0 else d["new_value_vector"]
    pol = PolicyOutputs(torch.tensor(d["logits"], dtype=torch.float32, device="cuda"),
                        torch.tensor(nv, dtype=torch.float32, device="cuda"))
    n_rec = sc.E * sc.Tc
    rng = np.random.default_rng(sum(tspec))
    for size in (1, 5, 17, n_rec):
        idx = rng.permutation(n_rec)[:size]
        st, want = sc.ppo_subset(tspec, idx)
        if st == 8:  # SkipUpdate is not raised by ppo_loss; a subset without units is legal
            continue
        assert st == 0, st
        got = vec(optim.ppo_loss_minibatch(ro, pol, batch, idx, PpoParams(0.2, 0.5, 0.01, True)))
        assert got[6] == want[6], (size, got[6], want[6])
        assert_close(got[:6], want[:6], 1e-5, f"{tspec} n={size}")


def test_grpo_minibatches_vs_reference():
    sc = bindings.RefScenario(num_envs=16, num_chunks=5, chunk_length=2, vocab=11,
                              use_fixed_reset_state_ids=1, group_size=4, auto_reset=0,
                              deferred_reset=1, max_episode_steps=8, num_reset_states=64,
                              perturb=0.3)
    d = sc.export(with_logits=True)
    ro = RolloutBuffer.from_arrays(d, d["boot_scalar"], int(d["V"]))
    eps = EpisodeTable.from_arrays(d)
    spec = GranularitySpec(Level.Chunk, Level.Token, Level.Chunk)
    opts = GrpoAssemblyOptions(spec, 1e-8, False, FilterBounds(0.0, 1.0), True, 2)
    b = advantage.assemble_grpo_batch(ro, eps, opts)
    pol = PolicyOutputs(torch.tensor(d["logits"], dtype=torch.float32, device="cuda"))
    G = b.groups_retained
    assert G >= 3
    for sel in ([0], [G - 1, 0], list(range(G)), [1, 2]):
        st, want = sc.grpo_subset((0, 2, 0), sel, eps_std=1e-8, apply_filter=False)
        assert st == 0
        got = vec(optim.grpo_loss_minibatch(ro, pol, b, sel, GrpoParams(0.2)))
        assert got[6] == want[6]
        assert_close(got[:6], want[:6], 1e-5, f"groups {sel}")
    with pytest.raises(errors.SkipUpdate):
        optim.grpo_loss_minibatch(ro, pol, b, [], GrpoParams(0.2))
    # the batch itself is untouched: the full loss still sees every group
    full = vec(optim.grpo_loss_minibatch(ro, pol, b, list(range(G)), GrpoParams(0.2)))
    st, want = sc.grpo_subset((0, 2, 0), list(range(G)), eps_std=1e-8, apply_filter=False)
    assert_close(full[:6], want[:6], 1e-5, "all groups again")
