"""Entropy at token, action and chunk granularity with valid-action masks (north star (b)) on
the CUDA path vs the oracle: ckrl_token_stats (optional slot mask) and the loss outputs
(action / chunk entropy over the unit-active slots: PPO counted, GRPO weighted trajectory
slots). The aggregates are canonical-order sums of per-token entropies
(core/granularity.cpp:83-113's order; the reference itself stops at the per-token entropy,
policy_net.cpp:333-357, pinned by the golden fixtures' `ent_cur`)."""
import numpy as np
import pytest
import torch

from conftest import assert_close, golden_files, load_golden

pytestmark = pytest.mark.gpu

import paper_2510_06710_b200 as ck  # noqa: E402
from paper_2510_06710_b200 import optim, policy, synth  # noqa: E402
from paper_2510_06710_b200.core import (EpisodeTable, GaeParams, GranularitySpec,  # noqa: E402
                                        GrpoAssemblyOptions, GrpoParams, Level, LossOutputs,
                                        PolicyOutputs, PpoParams, RolloutBuffer)

TOL = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _device():
    assert torch.cuda.is_available()
    ck.lib()


@pytest.mark.parametrize("name", golden_files("ppo_"))
def test_token_stats_entropy_aggregates_vs_reference(name, oracle):
    d = load_golden(name)
    E, Tc, Cn, M = d["ent_cur"].shape
    logits = torch.tensor(d["logits"], dtype=torch.float32, device="cuda")
    tokens = torch.tensor(d["tokens"], dtype=torch.int32, device="cuda")
    valid = torch.tensor((d["flags"] & 4) != 0, device="cuda")
    for mask in (None, valid):
        out = policy.evaluate_chunks(logits, tokens, valid=mask)
        m = None if mask is None else mask.cpu().numpy().reshape(E * Tc, Cn)
        act, chk = oracle.entropy_aggregates(d["ent_cur"], Cn, M, m)
        tag = "all" if mask is None else "valid"
        assert_close(out["action_entropy"].cpu().numpy().reshape(-1, Cn), act, TOL, f"{name} action H {tag}")
        assert_close(out["chunk_entropy"].cpu().numpy().reshape(-1), chk, TOL, f"{name} chunk H {tag}")


@pytest.mark.parametrize("V,dtype", [(256, torch.float32), (256, torch.bfloat16), (100, torch.float32)])
def test_token_stats_entropy_aggregates_synthetic(V, dtype, oracle):
    g = torch.Generator(device="cuda").manual_seed(3)
    n, Cn, M = 40, 8, 7
    logits = (2.0 * torch.randn(n, Cn, M, V, device="cuda", generator=g)).to(dtype)
    tokens = torch.randint(0, V, (n, Cn, M), device="cuda", generator=g, dtype=torch.int32)
    valid = torch.rand(n, Cn, device="cuda", generator=g) < 0.7
    out = policy.evaluate_chunks(logits, tokens, valid=valid)
    _, ent = oracle.token_stats(logits.float().cpu().numpy(), tokens.cpu().numpy())
    act, chk = oracle.entropy_aggregates(ent, Cn, M, valid.cpu().numpy())
    assert_close(out["action_entropy"].cpu().numpy(), act, TOL, f"V={V} {dtype} action H")
    assert_close(out["chunk_entropy"].cpu().numpy(), chk, TOL, f"V={V} {dtype} chunk H")


@pytest.mark.parametrize("cfg_name", ["cfg3", "cfg1"])
def test_ppo_loss_entropy_aggregates(cfg_name, oracle):
    cfg = synth.SynthConfig(**{**synth.CONFIGS[cfg_name].__dict__, "num_envs": 32, "seed": 9})
    a, l, v = synth.SPECS[cfg_name]
    d = synth.episodes_numpy(cfg)
    logits, tokens, old = synth.token_tensors(cfg, "cuda", torch.float32)
    d["tokens"], d["old_logprob"] = tokens.cpu().numpy(), old.cpu().numpy()
    boot = d["boot_scalar"] if a == 0 else d["boot_vector0"]
    nv = d["new_value_scalar"] if v == 0 else d["new_value_vector"]
    ro = RolloutBuffer.from_arrays(d, boot, cfg.vocab)
    pol = PolicyOutputs(logits, torch.tensor(nv, dtype=torch.float32, device="cuda"))
    spec = GranularitySpec(Level(a), Level(l), Level(v))
    st = optim.PpoStep(ro, GaeParams(0.99, 0.95), spec, PpoParams(0.2, 0.5, 0.01, True), outputs=False)
    st.outputs = LossOutputs.allocate(ro, spec.value_level, tokens=True, entropy=True)
    st._oc = st.outputs.c()
    st(ro, pol)
    torch.cuda.synchronize()
    counted = st.batch.counted.cpu().numpy()
    _, ent = oracle.token_stats(logits.cpu().numpy().astype(np.float64), d["tokens"])
    act, chk = oracle.entropy_aggregates(ent, cfg.chunk_len, cfg.tokens_per_action, counted)
    assert_close(st.outputs.action_entropy.cpu().numpy().reshape(-1, cfg.chunk_len), act, TOL, f"{cfg_name} ppo action H")
    assert_close(st.outputs.chunk_entropy.cpu().numpy().reshape(-1), chk, TOL, f"{cfg_name} ppo chunk H")
    # the loss's entropy term is their mean per counted position (losses.cpp:181-190, 223)
    M = cfg.tokens_per_action
    want = chk.sum() / (counted.sum() * M)
    assert st.diagnostics()["entropy"] == pytest.approx(want, rel=TOL)


def test_grpo_loss_entropy_aggregates(oracle):
    cfg = synth.SynthConfig(**{**synth.CONFIGS["cfg4"].__dict__, "num_envs": 16, "seed": 9})
    a, l, v = synth.SPECS["cfg4"]
    d = synth.episodes_numpy(cfg)
    logits, tokens, old = synth.token_tensors(cfg, "cuda", torch.float32)
    d["tokens"], d["old_logprob"] = tokens.cpu().numpy(), old.cpu().numpy()
    ro = RolloutBuffer.from_arrays(d, d["boot_scalar"], cfg.vocab)
    ept = EpisodeTable.from_arrays(d)
    spec = GranularitySpec(Level(a), Level(l), Level(v))
    st = optim.GrpoStep(ro, GrpoAssemblyOptions(spec), GrpoParams(0.2), outputs=False)
    st.outputs = LossOutputs.allocate(ro, Level.Chunk, entropy=True)
    st._oc = st.outputs.c()
    st(ro, ept, PolicyOutputs(logits))
    torch.cuda.synchronize()
    b = st.batch
    active = ((b.slot_member.cpu().numpy() != 0) & (b.slot_weight.cpu().numpy() != 0)
              & (b.env_group.cpu().numpy()[:, None, None] >= 0))
    assert active.any()
    _, ent = oracle.token_stats(logits.cpu().numpy().astype(np.float64), d["tokens"])
    act, chk = oracle.entropy_aggregates(ent, cfg.chunk_len, cfg.tokens_per_action, active)
    assert_close(st.outputs.action_entropy.cpu().numpy().reshape(-1, cfg.chunk_len), act, TOL, "grpo action H")
    assert_close(st.outputs.chunk_entropy.cpu().numpy().reshape(-1), chk, TOL, "grpo chunk H")
