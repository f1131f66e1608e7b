"""The reference unit tests' known answers through the CUDA path (libckrl.so C ABI):
tiny hand-built slabs of test_advantage.cpp / test_optim.cpp, edge cases (empty
rollouts, fully frozen chunks, single-env, odd C/M/V, i32 tokens, bf16 logits) and
determinism."""
import math

import numpy as np
import pytest
import torch

from conftest import assert_close
from test_oracle_known_answers import grpo_two_env_slab, ppo_case, tiny_slab

pytestmark = pytest.mark.gpu

from paper_2510_06710_b200 import advantage, errors, optim, policy  # noqa: E402
from paper_2510_06710_b200.core import (EpisodeTable, GaeParams, GranularitySpec,  # noqa: E402
                                        GrpoAssemblyOptions, GrpoParams, Level, LossOutputs,
                                        PolicyOutputs, PpoAssemblyOptions, PpoBatch, PpoParams,
                                        RolloutBuffer, Workspace, read_diagnostics)

C_, A_, T_ = Level.Chunk, Level.Action, Level.Token


def dev(x, dt=torch.float32):
    return torch.tensor(np.asarray(x), dtype=dt, device="cuda")


def test_ppo_assembler_action_level_mid_chunk_termination():
    d = tiny_slab([0.0, 0.0, 1.0, 0.0], [False, False, True, False], 2)
    ro = RolloutBuffer.from_arrays(d, d["boot_vector0"], 2)
    b = advantage.assemble_ppo_batch(ro, PpoAssemblyOptions(GaeParams(1.0, 1.0), GranularitySpec(A_, A_, A_)))
    assert b.advantages.cpu().numpy().ravel().tolist() == pytest.approx([1.0, 1.0, 1.0, 0.0])
    assert b.advantage_unit_count() == 4


def test_ppo_assembler_chunk_level_drops_tail():
    d = tiny_slab([1.0, 0.0, 0.0, 0.0], [True, False, False, False], 2)
    ro = RolloutBuffer.from_arrays(d, d["boot_scalar"], 2)
    b = advantage.assemble_ppo_batch(ro, PpoAssemblyOptions(GaeParams(1.0, 1.0), GranularitySpec(C_, C_, C_)))
    assert b.counted.cpu().numpy()[0].tolist() == [[1, 0], [1, 1]]
    assert b.advantages.cpu().numpy().ravel().tolist() == pytest.approx([1.0, 0.0])


def test_assembly_rejects_bad_granularity():
    d = tiny_slab([0.0, 0.0], [False, False], 2)
    ro = RolloutBuffer.from_arrays(d, d["boot_scalar"], 2)
    with pytest.raises(errors.ConfigError):
        advantage.assemble_ppo_batch(ro, PpoAssemblyOptions(GaeParams(), GranularitySpec(C_, T_, A_)))
    with pytest.raises(errors.UnsupportedCombination):
        advantage.assemble_ppo_batch(ro, PpoAssemblyOptions(GaeParams(), GranularitySpec(A_, C_, A_)))


def test_grpo_assembler_groups_weights_and_frozen_slots():
    for frozen in (False, True):
        d = grpo_two_env_slab(frozen_second_slot=frozen)
        ro = RolloutBuffer.from_arrays(d, d["boot_scalar"], 2)
        b = advantage.assemble_grpo_batch(ro, EpisodeTable.from_arrays(d),
                                          GrpoAssemblyOptions(GranularitySpec(C_, T_, C_), eps_std=0.0))
        assert (b.groups_total, b.groups_retained) == (1, 1)
        assert b.env_advantage.cpu().tolist() == pytest.approx([1.0, -1.0])
        if frozen:
            assert b.slot_member.cpu().numpy()[:, 0].tolist() == [[1, 0], [1, 0]]
        else:
            assert b.slot_weight.cpu().numpy()[0, 0].tolist() == [0.5, 0.5]


def test_grpo_all_degenerate_skips_update():
    d = grpo_two_env_slab()
    d["ep_total_reward"] = np.array([1.0, 1.0])
    ro = RolloutBuffer.from_arrays(d, d["boot_scalar"], 2)
    step = optim.GrpoStep(ro, GrpoAssemblyOptions(GranularitySpec(C_, C_, C_)), GrpoParams(0.2))
    step(ro, EpisodeTable.from_arrays(d), PolicyOutputs(dev(np.zeros((2, 1, 2, 1, 2)))))
    assert (step.batch.groups_total, step.batch.groups_retained) == (1, 0)
    with pytest.raises(errors.SkipUpdate):
        step.diagnostics()


def test_grpo_degenerate_group_without_eps():
    d = grpo_two_env_slab()
    d["ep_total_reward"] = np.array([1.0, 1.0])
    ro = RolloutBuffer.from_arrays(d, d["boot_scalar"], 2)
    opts = GrpoAssemblyOptions(GranularitySpec(C_, C_, C_), eps_std=0.0, apply_filter=False)
    step = optim.GrpoStep(ro, opts, GrpoParams(0.2))
    step(ro, EpisodeTable.from_arrays(d), PolicyOutputs(dev(np.zeros((2, 1, 2, 1, 2)))))
    with pytest.raises(errors.DegenerateGroup):
        step.diagnostics()


def ppo_loss_case(spec, rho_log, adv, clip=0.2):
    d, logits, counted, a = ppo_case((int(spec.advantage_level), int(spec.logprob_level), int(spec.value_level)), rho_log, adv)
    ro = RolloutBuffer.from_arrays(d, d["boot_scalar"], 3)
    ws = Workspace(1)
    batch = PpoBatch(spec=spec, counted=dev(counted, torch.uint8), advantages=dev(a, torch.float64),
                     returns=torch.zeros_like(dev(a, torch.float64)), workspace=ws)
    # stats record for this hand-built batch: the assembly normally leaves it
    advantage.assemble_ppo_batch(ro, PpoAssemblyOptions(GaeParams(), GranularitySpec(spec.advantage_level, spec.logprob_level, spec.advantage_level)),
                                 workspace=ws)
    diag = optim.ppo_loss(ro, PolicyOutputs(dev(logits), dev(np.zeros((1, 1)))), batch,
                          PpoParams(clip, 0.0, 0.0, False))
    return read_diagnostics(diag)


def test_ppo_rho_one_is_minus_mean_advantage():  # test_optim.cpp:115-130
    g = ppo_loss_case(GranularitySpec(C_, C_, C_), 0.0, 1.7)
    assert g["surrogate"] == pytest.approx(-1.7, rel=1e-6) and g["clip_frac"] == 0.0


def test_ppo_forced_clip():  # test_optim.cpp:132-150
    g = ppo_loss_case(GranularitySpec(C_, C_, C_), math.log(2.0), 2.5)
    assert g["surrogate"] == pytest.approx(-1.2 * 2.5, rel=1e-6) and g["clip_frac"] == 1.0


@pytest.mark.parametrize("E,Tc,C,M,V", [(1, 1, 1, 1, 2), (3, 5, 3, 2, 7), (2, 4, 5, 3, 300), (4, 3, 8, 7, 256)])
def test_odd_shapes_vs_oracle(oracle, E, Tc, C, M, V):
    """Generic-V path, i32 tokens (V > 256), C not dividing the CTA, single env."""
    from paper_2510_06710_b200 import synth
    cfg = synth.SynthConfig(num_envs=E, num_chunks=Tc, chunk_len=C, tokens_per_action=M, vocab=V,
                            algo="ppo", mode="deferred", max_episode_steps=5, p_terminate=0.2)
    d = synth.episodes_numpy(cfg)
    rng = np.random.default_rng(E * 100 + V)
    d["tokens"] = rng.integers(0, V, (E, Tc, C, M)).astype(np.int32)
    d["old_logprob"] = -math.log(V) + 0.2 * rng.standard_normal((E, Tc, C, M))
    logits = (2.0 * rng.standard_normal((E, Tc, C, M, V))).astype(np.float32)
    for spec in [(0, 0, 0), (0, 2, 0), (1, 1, 1)]:
        gs = GranularitySpec(*(Level(x) for x in spec))
        boot = d["boot_scalar"] if spec[0] == 0 else d["boot_vector0"]
        nv = d["new_value_scalar"] if spec[2] == 0 else d["new_value_vector"]
        ro = RolloutBuffer.from_arrays(d, boot, V)
        step = optim.PpoStep(ro, GaeParams(0.99, 0.95), gs, PpoParams(0.2, 0.5, 0.01, True))
        step(ro, PolicyOutputs(dev(logits), dev(nv)))
        got = step.diagnostics()
        r = {k: (np.asarray(v, np.float32).astype(np.float64) if np.asarray(v).dtype.kind == "f" else v)
             for k, v in d.items()}
        st, c, a, R = oracle.assemble_ppo({**r, "V": V}, spec, 0.99, 0.95)
        np.testing.assert_array_equal(step.batch.counted.cpu().numpy(), c)
        a = oracle.normalize_advantages(c, a, spec[0])
        st, want, *_ = oracle.ppo_loss({**r, "V": V}, spec, c, a, R, logits.astype(np.float64), r["new_value_scalar"] if spec[2] == 0 else r["new_value_vector"], 0.2, 0.5, 0.01)
        vec = np.array([got[k] for k in ("loss", "surrogate", "value_loss", "entropy", "clip_frac", "approx_kl", "units")])
        assert vec[6] == want[6]
        assert_close(vec[:6], want[:6], 1e-5, f"{(E, Tc, C, M, V, spec)}")


def test_empty_and_frozen_rollouts():
    # all slots frozen: no units anywhere -> zero diagnostics (reference returns default diag)
    E, Tc, C, M, V = 2, 3, 2, 7, 256
    d = dict(tokens=np.zeros((E, Tc, C, M), np.int32), old_logprob=np.zeros((E, Tc, C, M)),
             reward=np.zeros((E, Tc, C)), flags=np.zeros((E, Tc, C), np.uint8),
             episode_id=np.full((E, Tc, C), -1, np.int32), value_scalar=np.zeros((E, Tc)),
             value_vector=np.zeros((E, Tc, C)))
    ro = RolloutBuffer.from_arrays(d, np.zeros((E, Tc, C)), V)
    step = optim.PpoStep(ro, GaeParams(), GranularitySpec(C_, C_, C_), PpoParams(0.2, 0.5, 0.01, True))
    step(ro, PolicyOutputs(torch.zeros((E, Tc, C, M, V), device="cuda"), torch.zeros((E, Tc), device="cuda")))
    g = step.diagnostics()
    assert g["units"] == 0 and g["loss"] == 0.0
    assert int(step.batch.counted.sum()) == 0


def test_token_stats_bf16_and_u8_paths(oracle):
    rng = np.random.default_rng(7)
    logits = torch.tensor(2.0 * rng.standard_normal((9, 8, 7, 256)), dtype=torch.bfloat16, device="cuda")
    tokens = torch.tensor(rng.integers(0, 256, (9, 8, 7)), dtype=torch.uint8, device="cuda")
    out = policy.evaluate_chunks(logits, tokens)
    lp, ent = oracle.token_stats(logits.float().cpu().numpy().astype(np.float64), tokens.cpu().numpy())
    assert_close(out["token_logprob"].cpu().numpy().ravel(), lp, 1e-5, "lp")
    assert_close(out["token_entropy"].cpu().numpy().ravel(), ent, 1e-5, "ent")
    assert_close(out["chunk_logprob"].cpu().numpy().ravel(), lp.reshape(9, -1).sum(1), 1e-5, "chunk")
